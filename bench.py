"""Benchmark: CQRRPT canonical GFLOP/s on BASELINE config 2 (one B200 per rank).

metric   CQRRPT canonical GFLOP/s = (2 m n^2 - 2 n^3/3) / t
workload BASELINE.json configs[1]: M 131072 x 1024 FP64 = U diag(sigma) V^T,
         sigma_i = 10^(-10 i/(n-1)) (cond 1e10), d_factor 1.25, SASO nnz 8, seed 0.
         U, V from QR of seeded Gaussians, generated on the GPU with torch
         (synthetic stand-in with the config's shape and spectrum; not the
         reference generator's bits).
step     one cqrrpt_gpu_dgeqpt call (sketch -> QRCP -> stage 1/2 -> gather+TRSM
         -> Gram -> Cholesky -> Q TRSM in place -> R) on the resident input.
         Between timed steps the input is restored and L2 is flushed (256 MiB
         write); the restore + flush are outside the timed events.
N > 1    torchrun, one process per GPU, NCCL allreduce of the sketch and the
         Gram inside the library; weak scaling (each rank owns 131072 rows of
         an N*131072 x 1024 matrix).

--impl reference  times the reference's own CPU cqrrpt() (oracle/_ref, the
         unmodified reference library built from /root/reference) on a bounded
         row sample of the same workload with all host threads.
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

M_ROWS, N_COLS, GAMMA, NNZ, SEED = 131072, 1024, 1.25, 8, 0
COND_DECADES = 10.0
CPU_SAMPLE_ROWS = 16384  # bounded CPU sample (1/8 of the rows)
METRIC = "CQRRPT canonical GFLOP/s (2mn^2-2n^3/3)/t, FP64 tall M"


def canonical_flops(m, n):
    return 2.0 * m * n * n - 2.0 * n ** 3 / 3.0


# --------------------------------------------------------------------------
# input generation (harness only)
# --------------------------------------------------------------------------
def make_c2_torch(m, n, seed, device):
    import torch
    g = torch.Generator(device=device).manual_seed(seed)
    u = torch.linalg.qr(torch.randn((m, n), dtype=torch.float64, device=device, generator=g))[0]
    v = torch.linalg.qr(torch.randn((n, n), dtype=torch.float64, device=device, generator=g))[0]
    sig = 10.0 ** (-COND_DECADES * torch.arange(n, dtype=torch.float64, device=device) / (n - 1))
    a = torch.empty((n, m), dtype=torch.float64, device=device)  # column-major m x n
    a.copy_(((u * sig) @ v.T).T)
    del u, v
    return a.t()


def make_c2_numpy(m, n, seed):
    rng = np.random.default_rng(seed)
    u = np.linalg.qr(rng.standard_normal((m, n)))[0]
    v = np.linalg.qr(rng.standard_normal((n, n)))[0]
    sig = 10.0 ** (-COND_DECADES * np.arange(n) / (n - 1))
    return np.asfortranarray((u * sig) @ v.T)


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
            # nvidia-smi takes a moment to start: wait for its first row so the
            # samples cover the timed region, then keep only rows from here on
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
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# --------------------------------------------------------------------------
# peaks
# --------------------------------------------------------------------------
def measure_fp64_peak(torch):
    """cuBLAS DGEMM 8192^3 (torch.matmul float64), best of 5 — the FP64 roofline
    denominator (MEASURED_PEAKS.json carries no FP64 figure)."""
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
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def load_traffic():
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


# --------------------------------------------------------------------------
# CPU reference arm / baseline
# --------------------------------------------------------------------------
def run_reference_cpu(steps, warmup, rows=CPU_SAMPLE_ROWS):
    from oracle.oracle import Reference
    ref = Reference()
    cores = ref.num_threads()
    a = make_c2_numpy(rows, N_COLS, SEED)
    times = []
    for it in range(warmup + steps):
        res = ref.cqrrpt(a, gamma=GAMMA, nnz=NNZ, eps_tol=1e-4, seed=SEED, validate=False)
        if it >= warmup:
            times.append(res.extra["timings"]["total"])  # diagnostics.timings.total (cqrrpt.cc:288)
    t = float(np.mean(times))
    return dict(value=canonical_flops(rows, N_COLS) / t / 1e9, t=t, best=float(np.min(times)), cores=cores,
                k=res.k, rows=rows)


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = {"workload": "BASELINE configs[1]: M 131072x1024 FP64, sigma_i=10^(-10 i/(n-1)), d_factor 1.25, "
                       "SASO nnz 8, seed 0",
           "m": M_ROWS * max(world, 1), "n": N_COLS, "d_factor": GAMMA, "nnz": NNZ,
           "parallelism": f"rows{max(world, 1)}", "l2": "flushed between steps (256 MiB write)"}

    if args.impl == "reference":
        if rank != 0:
            return
        r = run_reference_cpu(args.steps, args.warmup)
        line = {"metric": METRIC, "value": r["value"], "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": r["t"] * 1e3, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
                "config": dict(cfg, sample_rows=r["rows"]),
                "cpu_baseline": {"value": r["value"], "unit": "GFLOP/s", "cores": r["cores"], "kind": "reference",
                                 "sample": f"reference cqrrpt() on a {r['rows']}x{N_COLS} row sample of the workload "
                                           f"(validate_output=false, timings.total, mean of {args.steps})"},
                "e2e": {"value": r["value"], "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import paper_2311_08316_b200 as pkg
    from paper_2311_08316_b200 import kernels

    torch.cuda.set_device(local)
    dist = None
    comm = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = pkg.Comm.from_torch_distributed()
    stream = torch.cuda.current_stream()

    m, n = M_ROWS, N_COLS
    a0 = make_c2_torch(m, n, SEED + rank, "cuda")
    work = pkg.colmajor_empty(m, n)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    canon = canonical_flops(m * world, n)

    def barrier():
        if dist is not None:
            dist.barrier()

    def one_step(timed):
        work.copy_(a0)
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = pkg.dgeqpt(work, d_factor=GAMMA, nnz=NNZ, seed=SEED, comm=comm, global_row_offset=rank * m,
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
    torch.cuda.synchronize()
    barrier()
    launches = kernels.launch_count(reset=True)
    total_ms = float(np.sum(step_ms))
    if dist is not None:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = canon / (ms_per_step * 1e-3) / 1e9
    ph = phases / args.steps
    names = ["sketch", "qrcp", "rank_select", "precondition", "cholesky_qr", "undo", "total", "comm"]

    # ---- e2e: host input -> device -> factor -> Q, R, J back to host, through
    # the public host entry point (cqrrpt_gpu_dgeqpt_host: pinned buffers, Q
    # streamed back block by block: from the wavefront on one rank, during the
    # final TRSM on several) --------------------------------------------------
    host_a = torch.empty((n, m), dtype=torch.float64).pin_memory()
    host_a.copy_(a0.t())
    k = res.k
    host_q = torch.empty((n, m), dtype=torch.float64).pin_memory().t()
    host_r = torch.empty((n, n), dtype=torch.float64).pin_memory().t()
    host_j = torch.empty(n, dtype=torch.int64).pin_memory()
    e2e_ms = []
    for it in range(args.warmup + args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r2 = pkg.dgeqpt_host(host_a.t(), d_factor=GAMMA, nnz=NNZ, seed=SEED, q_out=host_q, r_out=host_r,
                             j_out=host_j, stream=stream, comm=comm, global_row_offset=rank * m)
        e1.record(stream)
        e1.synchronize()
        if it >= args.warmup:
            e2e_ms.append(e0.elapsed_time(e1))
    assert r2.k == k
    e2e_t = float(np.mean(e2e_ms))
    if dist is not None:
        t = torch.tensor([e2e_t], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = float(t.item())
    e2e_value = canon / (e2e_t * 1e-3) / 1e9
    h2d = m * n * 8
    d2h = m * k * 8 + k * n * 8 + n * 8

    if rank != 0:
        if comm is not None:
            comm.close()
        dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (gather + DMMA TRSM, K5a) --------------
    fp64_peak = measure_fp64_peak(torch)
    k0 = res.k0
    trsm_flops = float(m) * k0 * k0  # trsm_right flop count m k0^2 (flop_model term)
    trsm_ms = ph[3]
    achieved = trsm_flops / (trsm_ms * 1e-3) / 1e12
    # DRAM bytes of one TRSM pass (16 launches) from ncu, profiles/traffic.json
    traffic = load_traffic().get("trsm_pass_dram_bytes")
    peaks, peak_src = measured_peaks()
    roofline = {"bound": "tensor", "kernel": "trsm_block_kernel (K5a gather+TRSM, DMMA.8x8x4)",
                "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved / fp64_peak,
                "traffic": traffic,
                "peak_source": "measured live in this run: cuBLAS DGEMM 8192^3 via torch.matmul(float64), best of 5",
                "algorithmic": "m*k0^2 flops per TRSM pass (m=131072, k0=1024)",
                "traffic_unit": "DRAM bytes per TRSM pass (ncu dram__bytes_read+write, profiles/traffic.json)"}
    # secondary rooflines
    sketch_bytes = 8.0 * m * n + 8.0 * res.ctx.d * n
    sk = {"bound": "hbm", "achieved": sketch_bytes / (ph[0] * 1e-3) / 1e9, "peak": peaks.get("hbm_gbs"),
          "unit": "GB/s", "peak_source": peak_src}
    sk["frac"] = sk["achieved"] / sk["peak"] if sk["peak"] else None
    # the sketch's binding resource: shared-memory wavefronts (128 B each) of
    # the apply kernel, counted by ncu for this configuration
    # (profiles/traffic.json), over the live sketch-phase time, against
    # 128 B/clk/SM x SMs x the SM clock sampled under load
    tr = load_traffic()
    wf = tr.get("saso_apply_smem_wavefronts")
    if wf:
        props = torch.cuda.get_device_properties(local)
        sm_ghz = (clk.summary().get("sm_mhz") or 1965.0) / 1e3
        smem_peak = 128.0 * props.multi_processor_count * sm_ghz  # GB/s
        sk["smem"] = {"bound": "shared memory", "achieved": wf * 128.0 / (ph[0] * 1e-3) / 1e9, "peak": smem_peak,
                      "unit": "GB/s", "wavefronts_per_launch": wf,
                      "peak_source": "128 B/clk/SM x SMs x sampled SM clock",
                      "traffic": tr.get("saso_apply_dram_bytes")}
        sk["smem"]["frac"] = sk["smem"]["achieved"] / smem_peak
    contraction_flops = float(m) * k0 * k0 + float(m) * k0 * (k0 + 1) + float(m) * k * k
    con = {"bound": "tensor", "achieved": contraction_flops / ((ph[3] + ph[4]) * 1e-3) / 1e12, "peak": fp64_peak,
           "unit": "TFLOP/s"}
    con["frac"] = con["achieved"] / fp64_peak

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            r = run_reference_cpu(1, 1)
            cpu = {"value": r["value"], "unit": "GFLOP/s", "cores": r["cores"], "kind": "reference",
                   "sample": f"reference cqrrpt() (oracle/_ref) on a {r['rows']}x{N_COLS} row sample of the "
                             f"workload, validate_output=false, timings.total"}
        except Exception as exc:  # reference library missing on this host
            cpu = {"value": None, "unit": "GFLOP/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    line = {"metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (torch-generated C2-shaped matrix)",
            "config": cfg,
            "e2e": {"value": e2e_value, "unit": "GFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_t,
                    "path": ("cqrrpt_gpu_dgeqpt_host, pinned host A/Q/R: A in 4 row chunks followed by the exact "
                             "sketch, Q downloaded in 64-column blocks " +
                             ("from the 128-column wavefront" if world == 1 else "during the final TRSM"))},
            "roofline": roofline, "roofline_sketch": sk, "roofline_contractions": con,
            "phases_ms": dict(zip(names, [round(float(x), 4) for x in ph])),
            "k": k, "k0": k0, "gpu_launches": launches, "clocks": clk.summary(), "cpu_baseline": cpu}
    print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
