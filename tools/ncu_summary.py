"""Summarise ncu --set full reports: time, DRAM traffic, throughput, pipe
utilisation and the top stall reasons per kernel launch.

usage: python tools/ncu_summary.py gpurun_out/prof_*.ncu-rep > profiles/ncu_rNN_summary.json
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_registers",
    "smsp__inst_executed.sum",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        return []
    hdr, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        item = {"kernel": d.get("Kernel Name", "")[:80]}
        for k in KEYS:
            if k in d and d[k] != "":
                item[k] = f"{d[k]} {u.get(k, '')}".strip()
        stalls = []  # warps stalled per issued instruction, by reason
        for k, v in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                reason = k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]
                if reason in ("selected",):
                    continue
                try:
                    stalls.append((float(v.replace(",", "")), reason))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        item["top_stalls_per_issue"] = {r: round(v, 3) for v, r in stalls[:6]}
        res.append(item)
    return res


def main(paths):
    out = {}
    for p in paths:
        out[os.path.basename(p)] = rows(p)
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1:])
