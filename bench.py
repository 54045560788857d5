"""Benchmark: CQRRPT canonical GFLOP/s on the BASELINE workload (one B200 per rank).

metric   CQRRPT canonical GFLOP/s = (2 m n^2 - 2 n^3/3) / t,
         t = device time of one factorization, max over ranks.
workload --config (default C5_2048): BASELINE configs[4] at its largest single-
         GPU size, M 4194304 x 2048 FP64 (64 GiB), Gaussian columns scaled by
         geometric norms 1 .. 1e-8 in a seeded random order, d_factor 1.25,
         SASO nnz 8, seed 0 -- the largest config BASELINE lists at 1 GPU and
         the one it lists at 1/2/4/8. Other configs (C1..C5_1024) are
         secondary lines (tools/workloads.py). Data: seeded synthetic, generated
         on the device in 65536-row tiles (the same global matrix at any N).
step     one cqrrpt_gpu_dgeqpt call (sketch -> allreduce -> QRCP -> stage 1/2 ->
         gather+TRSM -> Gram -> allreduce -> Cholesky -> Q TRSM in place -> R)
         on the resident input. Between timed steps the input is restored
         (device copy, or H2D from pinned host memory when A + its copy + M_pre
         do not fit in HBM); the restore writes far more than L2 (126 MB), and
         every input is larger than L2 -- both outside the timed events.
N > 1    torchrun, one process per GPU, rows [r m/N, (r+1) m/N) of the one
         global matrix per rank; NCCL allreduce of the d x n sketch and the
         k0 x k0 Gram inside the library; strong scaling.
e2e      the public host entry point cqrrpt_gpu_dgeqpt_host: pinned host A in,
         Q (m x k), R, J out, copies inside the timed region.

--impl reference  the reference's own CPU cqrrpt() (oracle/_ref: the unmodified
         reference library built from /root/reference) on the workload's first
         S rows (a bounded row sample), all host threads; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
from tools.workloads import CONFIGS, DESCRIPTION, SEED, canonical_flops, make_rows  # noqa: E402

NNZ = 8
METRIC = "CQRRPT canonical GFLOP/s (2mn^2-2n^3/3)/t, FP64 tall M"
# CPU reference row sample per config (~10-20 s per reference run on 16 cores)
SAMPLE_ROWS = {"C1": 16384, "C2": 16384, "C3": 8192, "C3b": 8192, "C4": 4096, "C5_256": 65536,
               "C5_512": 32768, "C5_1024": 16384, "C5_2048": 4096}


# --------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# --------------------------------------------------------------------------
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # wait for nvidia-smi's first row so the samples cover the timed region
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0:
                time.sleep(0.01)
            self.rows.clear()
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for nm, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        def num(v):
            try:
                return float(v)
            except ValueError:
                return None
        # the timed region alternates factorization steps with idle-clock input
        # restores, so the median sits at the idle clock; also report the lowest
        # sample, the samples taken while the power cap was active, and the draw
        capped = [num(r[0]) for r in self.rows if len(r) > 7 and r[7].strip().lower() == "active"]
        capped = [v for v in capped if v is not None]
        power = [v for v in (num(r[2]) for r in self.rows if len(r) > 2) if v is not None]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows),
                "sm_min_mhz": min(sm) if sm else None,
                "sm_mhz_power_capped": float(np.median(capped)) if capped else None,
                "power_w_max": max(power) if power else None}


# --------------------------------------------------------------------------
# peaks
# --------------------------------------------------------------------------
def measure_fp64_peak(torch):
    """cuBLAS DGEMM 8192^3 (torch.matmul float64), best of 5 -- the FP64
    roofline denominator (MEASURED_PEAKS.json carries no FP64 figure)."""
    n = 8192
    a = torch.randn((n, n), dtype=torch.float64, device="cuda")
    b = torch.randn((n, n), dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    del a, b
    return 2.0 * n ** 3 / best / 1e12


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "MEASURED_PEAKS.json (driver-measured copy bandwidth)"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback (B200_PROFILING.md)"


def load_traffic(config):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get(config, {})
    return {}


# --------------------------------------------------------------------------
# CPU reference arm / baseline
# --------------------------------------------------------------------------
def reference_sample(name):
    """The workload's first S rows as a Fortran-ordered host array (generated
    with the same tile generator on the box's GPU when there is one)."""
    import torch
    cfg = dict(CONFIGS[name])
    rows = min(SAMPLE_ROWS[name], cfg["m"])
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    if cfg["kind"] == "spectral":  # C2 is generated whole; keep its first S rows
        a = make_rows(cfg, 0, cfg["m"], dev)[:rows]
    elif cfg["kind"] == "lowrank":
        from tools.workloads import fill_rows, lowrank_fro_sq
        fro = lowrank_fro_sq(cfg, dev)
        a = torch.empty((cfg["n"], rows), dtype=torch.float64, device=dev).t()
        fill_rows(cfg, 0, rows, a, dev, fro_sq_total=fro)
    else:
        a = make_rows(cfg, 0, rows, dev)
    host = np.asfortranarray(a.cpu().numpy())
    del a
    if dev == "cuda":
        torch.cuda.empty_cache()
    return host, dev


def run_reference_cpu(name, steps, warmup):
    from oracle.oracle import Reference
    ref = Reference()
    cores = ref.num_threads()
    a, dev = reference_sample(name)
    rows, n = a.shape
    gamma = CONFIGS[name]["gamma"]
    times = []
    res = None
    for it in range(warmup + steps):
        res = ref.cqrrpt(a, gamma=gamma, nnz=NNZ, eps_tol=1e-4, seed=SEED, validate=False)
        if it >= warmup:
            times.append(res.extra["timings"]["total"])  # diagnostics.timings.total (cqrrpt.cc:288)
    t = float(np.mean(times))
    return dict(value=canonical_flops(rows, n) / t / 1e9, t=t, best=float(np.min(times)), cores=cores,
                k=res.k, rows=rows, n=n, gen_device=dev, runs=len(times))


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5_2048", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    name = args.config
    cfg = CONFIGS[name]
    m, n, gamma = cfg["m"], cfg["n"], cfg["gamma"]
    conf = {"workload": f"{name}: {DESCRIPTION[name]}; d_factor {gamma}, SASO nnz {NNZ}, seed {SEED}",
            "m": m, "n": n, "d_factor": gamma, "nnz": NNZ, "parallelism": f"rows{max(world, 1)}",
            "l2": "inputs larger than L2 (126 MB); the between-step input restore writes the whole matrix"}

    if args.impl == "reference":
        if rank != 0:
            return
        r = run_reference_cpu(name, args.steps, args.warmup)
        line = {"metric": METRIC, "value": r["value"], "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": r["t"] * 1e3, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (tools/workloads.py)", "impl": "reference",
                "config": dict(conf, sample_rows=r["rows"]),
                "cpu_baseline": {"value": r["value"], "unit": "GFLOP/s", "cores": r["cores"], "kind": "reference",
                                 "sample": f"reference cqrrpt() (oracle/_ref, unmodified reference library) on the "
                                           f"first {r['rows']} rows of the {name} matrix ({r['rows']}x{n}), "
                                           f"validate_output=false, timings.total, mean of {r['runs']}"},
                "e2e": {"value": r["value"], "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines on stderr (nranks check)
    import paper_2311_08316_b200 as pkg
    from paper_2311_08316_b200 import kernels

    if cfg["kind"] == "spectral" and world > 1:
        raise SystemExit("C2 (U from a global QR) is a single-GPU workload")
    if m % world:
        raise SystemExit(f"m = {m} is not divisible by {world} ranks")
    torch.cuda.set_device(local)
    dist = None
    comm = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = pkg.Comm.from_torch_distributed()
    stream = torch.cuda.current_stream()
    ml = m // world
    r0 = rank * ml

    def barrier():
        if dist is not None:
            dist.barrier()

    # ---- input: rows [r0, r0 + ml) of the global matrix ------------------------
    work = make_rows(cfg, r0, r0 + ml, "cuda", dist=dist)
    torch.cuda.synchronize()
    free, total = torch.cuda.mem_get_info()
    a_bytes = ml * n * 8
    # keep a device copy of A when A, its copy and M_pre (m x n) fit; else pinned host
    device_copy = 3 * a_bytes + (2 << 30) < total
    host_a = torch.empty((n, ml), dtype=torch.float64).pin_memory()
    host_a.copy_(work.t())
    a0 = None
    if device_copy:
        a0 = torch.empty_like(work.t()).t()
        a0.copy_(work)
    canon = canonical_flops(m, n)

    def restore():
        if a0 is not None:
            work.copy_(a0)
        else:
            work.t().copy_(host_a, non_blocking=True)

    def one_step(timed):
        restore()
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = pkg.dgeqpt(work, d_factor=gamma, nnz=NNZ, seed=SEED, comm=comm, global_row_offset=r0,
                         timings=timed)
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1), res

    for _ in range(args.warmup):
        one_step(False)
    barrier()
    torch.cuda.synchronize()
    kernels.launch_count(reset=True)
    step_ms, phases = [], np.zeros(8)
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            ms, res = one_step(True)
            step_ms.append(ms)
            phases += np.array(list(res.ctx.timings_ms))
        clocks = clk.summary()
    torch.cuda.synchronize()
    barrier()
    launches = kernels.launch_count(reset=True)  # all K timed steps
    total_ms = float(np.sum(step_ms))
    ph = phases / args.steps
    names = ["sketch", "qrcp", "rank_select", "precondition", "cholesky_qr", "undo", "total", "comm"]
    per_rank = [dict(rank=rank, ms_per_step=total_ms / args.steps, comm_ms=float(ph[7]))]
    if dist is not None:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        gathered = [None] * world
        dist.all_gather_object(gathered, per_rank[0])
        per_rank = gathered
    ms_per_step = total_ms / args.steps
    value = canon / (ms_per_step * 1e-3) / 1e9
    k, k0 = res.k, res.k0

    # ---- e2e: host A in, Q, R, J out through the public host entry point ------
    e2e = None
    if not args.no_e2e:
        del work
        if a0 is not None:
            del a0
        pkg.release_workspace()
        torch.cuda.empty_cache()
        host_q = torch.empty((n, ml), dtype=torch.float64).pin_memory().t()
        host_r = torch.empty((n, n), dtype=torch.float64).pin_memory().t()
        host_j = torch.empty(n, dtype=torch.int64).pin_memory()
        e2e_ms = []
        for it in range(args.warmup + args.steps):
            torch.cuda.synchronize()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r2 = pkg.dgeqpt_host(host_a.t(), d_factor=gamma, nnz=NNZ, seed=SEED, q_out=host_q, r_out=host_r,
                                 j_out=host_j, stream=stream, comm=comm, global_row_offset=r0)
            e1.record(stream)
            e1.synchronize()
            if it >= args.warmup:
                e2e_ms.append(e0.elapsed_time(e1))
        assert r2.k == k, (r2.k, k)
        e2e_t = float(np.mean(e2e_ms))
        if dist is not None:
            t = torch.tensor([e2e_t], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_t = float(t.item())
        e2e = {"value": canon / (e2e_t * 1e-3) / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": ml * n * 8,
               "d2h_bytes_per_step": ml * k * 8 + k * n * 8 + n * 8, "ms_per_step": e2e_t,
               "path": "cqrrpt_gpu_dgeqpt_host, pinned host A/Q/R/J (rank-local rows): A in row chunks followed "
                       "by the exact sketch, Q downloaded in 64-column blocks as the final solve forms them"}

    if rank != 0:
        if comm is not None:
            comm.close()
        dist.destroy_process_group()
        return

    # ---- rooflines ---------------------------------------------------------------
    fp64_peak = measure_fp64_peak(torch)
    peaks, peak_src = measured_peaks()
    tr = load_traffic(name)
    trsm_flops = float(ml) * k0 * k0  # trsm_right: m k0^2 flops per pass (flop_model term)
    achieved = trsm_flops / (ph[3] * 1e-3) / 1e12
    from paper_2311_08316_b200 import kernels as _k
    engine = _k.trsm_engine(ml, k0)
    kname = ("precondition TRSM pass: oz_update_kernel (exact INT8 emulation on tcgen05 kind::i8, TMEM "
             "accumulators) for the trailing updates + trsm_block_kernel (DMMA) for the 128x128 diagonal blocks"
             if engine == "int8" else "trsm_block_kernel (K5a gather + TRSM on DMMA.8x8x4)")
    roofline = {"bound": "tensor", "kernel": kname,
                "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved / fp64_peak,
                "traffic": tr.get("trsm_pass_dram_bytes"),
                "peak_source": "measured live in this run: cuBLAS DGEMM 8192^3 (torch.matmul float64), best of 5 "
                               "(MEASURED_PEAKS.json has no FP64 figure); FP64-equivalent flops, so an INT8-emulated "
                               "pass can exceed 1.0",
                "algorithmic": f"m_local*k0^2 = {trsm_flops:.4g} flops per precondition TRSM pass, over the "
                               f"CUDA-event time of that phase",
                "traffic_unit": "DRAM bytes per TRSM pass (ncu dram__bytes_read+write, profiles/traffic.json)"}
    roofline_int8 = None
    if engine == "int8":
        # int8 MACs of the emulated trailing updates: 34 digit pairs per product,
        # 128-column steps (csrc/oztrsm.cu); over the whole pass time (diagonal
        # DMMA solves and digit slicing included), so a lower bound
        ops = 0.0
        for b0 in range(0, k0, 128):
            b1 = min(k0, b0 + 128)
            ops += 2.0 * 34 * (b1 - b0) * (k0 - b1) * ml
        roofline_int8 = {"bound": "tensor", "kernel": "oz_update_kernel (tcgen05.mma kind::i8, M128 K32, N = 32..128: one MMA per digit slice and K-step)",
                         "achieved": ops / (ph[3] * 1e-3) / 1e12, "peak": 4500.0, "unit": "TOPS",
                         "peak_source": "B200 dense INT8 tensor nominal (4.5 POPS); not in MEASURED_PEAKS.json",
                         "algorithmic": f"{ops:.4g} int8 ops per precondition pass (2 x 34 pairs x m x w x trailing "
                                        f"columns per 128-column step) over the pass time"}
        roofline_int8["frac"] = roofline_int8["achieved"] / roofline_int8["peak"]
    sketch_bytes = 8.0 * ml * n + 8.0 * res.ctx.d * n
    sk = {"bound": "hbm", "kernel": "saso_apply_kernel", "achieved": sketch_bytes / (ph[0] * 1e-3) / 1e9,
          "peak": peaks.get("hbm_gbs"), "unit": "GB/s", "peak_source": peak_src,
          "algorithmic": "8 m n (read M) + 8 d n (write M_sk) bytes", "traffic": tr.get("saso_apply_dram_bytes")}
    sk["frac"] = sk["achieved"] / sk["peak"] if sk["peak"] else None
    contraction_flops = float(ml) * k0 * k0 + float(ml) * k0 * (k0 + 1) + float(ml) * k * k
    con = {"bound": "tensor", "achieved": contraction_flops / ((ph[3] + ph[4]) * 1e-3) / 1e12, "peak": fp64_peak,
           "unit": "TFLOP/s", "algorithmic": "m k0^2 (TRSM) + m k0 (k0+1) (Gram) + m k^2 (final TRSM) over the "
                                             "precondition + cholesky_qr phases (incl. potrf)"}
    con["frac"] = con["achieved"] / fp64_peak

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            r = run_reference_cpu(name, 1, 1)
            cpu = {"value": r["value"], "unit": "GFLOP/s", "cores": r["cores"], "kind": "reference",
                   "sample": f"reference cqrrpt() (oracle/_ref) on the first {r['rows']} rows of the {name} "
                             f"matrix, validate_output=false, timings.total, 1 run after 1 warm-up"}
        except Exception as exc:  # reference library missing on this host
            cpu = {"value": None, "unit": "GFLOP/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    line = {"metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (tools/workloads.py, seeded, device-generated)",
            "config": dict(conf, restore="device copy" if device_copy else "H2D from pinned host memory"),
            "e2e": e2e, "roofline": roofline, "roofline_int8": roofline_int8, "roofline_sketch": sk,
            "roofline_contractions": con, "trsm_engine": engine,
            "phases_ms": dict(zip(names, [round(float(x), 4) for x in ph])), "per_rank": per_rank,
            "k": k, "k0": k0, "gpu_launches": launches,
            "gpu_launches_per_step": launches / max(args.steps, 1), "clocks": clocks, "cpu_baseline": cpu}
    print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
