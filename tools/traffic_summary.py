"""Summarise the ncu metric pass of tools/ncu_bench.sh into profiles/traffic.json.

usage: python tools/traffic_summary.py gpurun_out/traffic_C5_2048.csv C5_2048

Per config: DRAM bytes (read + write) per launch of the precondition TRSM
pass (the first run of consecutive trsm_block_kernel launches after the
sketch), their sum per pass, the SASO apply launch (DRAM bytes and shared
memory wavefronts) and, for reference, the algorithmic bytes.
"""
import csv
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from tools.workloads import CONFIGS  # noqa: E402


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, mi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name"), h.index("ID")
    out = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        out.setdefault(r[ii], [r[ki], {}])[1][r[mi]] = float(r[vi].replace(",", ""))
    return list(out.values())


def main(path, name):
    seq = load(path)
    cfg = CONFIGS[name]
    m, n = cfg["m"], cfg["n"]
    d = -(-int(cfg["gamma"] * n * 1000) // 1000)
    dram = lambda mt: mt.get("dram__bytes_read.sum", 0.0) + mt.get("dram__bytes_write.sum", 0.0)  # noqa: E731
    # first saso_apply launch, then the first run of trsm_block launches after it
    i_sk = next(i for i, (k, _) in enumerate(seq) if "saso_apply_kernel" in k)
    sk = seq[i_sk][1]
    i0 = next(i for i in range(i_sk, len(seq)) if "trsm_block_kernel" in seq[i][0])
    i1 = i0
    while i1 < len(seq) and "trsm_block_kernel" in seq[i1][0]:
        i1 += 1
    trsm = [mt for _, mt in seq[i0:i1]]
    entry = {
        "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                  f"l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__pipe_tensor_subpipe_dmma_cycles_active "
                  f"--clock-control none on `python bench.py --config {name} --steps 1 --warmup 0 --no-e2e` "
                  f"(tools/ncu_bench.sh); metric-list pass, no full-set replay of the working set",
        "trsm_pass_launches": len(trsm),
        "trsm_pass_dram_bytes": sum(dram(mt) for mt in trsm),
        "trsm_pass_min_bytes": 8.0 * m * n * 2,  # read the gathered M_k0 once, write M_pre once
        "trsm_pass_time_ns": sum(mt.get("gpu__time_duration.sum", 0.0) for mt in trsm),
        "trsm_launch_dram_bytes": [dram(mt) for mt in trsm],
        "trsm_launch_dmma_active_pct": [mt.get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active")
                                        for mt in trsm],
        "saso_apply_dram_bytes": dram(sk),
        "saso_apply_algorithmic_bytes": 8.0 * m * n + 8.0 * d * n,
        "saso_apply_smem_wavefronts": sk.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
        "saso_apply_time_ns": sk.get("gpu__time_duration.sum"),
    }
    p = os.path.join(ROOT, "profiles", "traffic.json")
    allp = json.load(open(p)) if os.path.exists(p) else {}
    allp = {k: v for k, v in allp.items() if isinstance(v, dict)}  # drop the round-1 flat layout
    allp[name] = entry
    with open(p, "w") as f:
        json.dump(allp, f, indent=1)
    print(json.dumps({k: v for k, v in entry.items() if not isinstance(v, list)}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
