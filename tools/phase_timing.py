"""Per-phase device timings of cqrrpt_gpu_dgeqpt on BASELINE-shaped inputs.

usage: python tools/phase_timing.py [C1|C2|C3|C4|C5-256 ...] [--reps R] [--fast-sketch]
Inputs are generated on the GPU with torch (harness only).
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_08316_b200 as pkg  # noqa: E402

CONFIGS = {
    "C1": dict(m=16384, n=256, kind="gaussian"),
    "C2": dict(m=131072, n=1024, kind="spectral"),
    "C3": dict(m=262144, n=2048, kind="lowrank"),
    "C4": dict(m=1048576, n=4096, kind="gaussian"),
    "C5-256": dict(m=4194304, n=256, kind="graded"),
    "C5-1024": dict(m=4194304, n=1024, kind="graded"),
}


def make(cfg, seed=0):
    m, n = cfg["m"], cfg["n"]
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.empty((n, m), dtype=torch.float64, device="cuda")  # column-major m x n
    kind = cfg["kind"]
    if kind == "gaussian":
        a.normal_(generator=g)
    elif kind == "spectral":
        u = torch.linalg.qr(torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g))[0]
        v = torch.linalg.qr(torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g))[0]
        sig = 10.0 ** (-10.0 * torch.arange(n, dtype=torch.float64, device="cuda") / (n - 1))
        a.copy_(((u * sig) @ v.T).T)
    elif kind == "lowrank":
        r = n // 2
        A = torch.randn((m, r), dtype=torch.float64, device="cuda", generator=g)
        B = torch.randn((r, n), dtype=torch.float64, device="cuda", generator=g)
        ab = A @ B
        noise = 1e-12 * torch.linalg.norm(ab) / (m * n) ** 0.5
        ab += noise * torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g)
        a.copy_(ab.T)
        del ab, A, B
    elif kind == "graded":
        a.normal_(generator=g)
        perm = torch.randperm(n, device="cuda", generator=g).to(torch.float64)
        a *= (10.0 ** (-8.0 * perm / (n - 1)))[:, None]
    return a.t()


def run(name, reps=3, fast_sketch=False):
    cfg = CONFIGS[name]
    a0 = make(cfg)
    m, n = a0.shape
    work = pkg.colmajor_empty(m, n)
    canon = 2.0 * m * n * n - 2.0 * n ** 3 / 3.0
    best = None
    for it in range(reps + 1):
        work.copy_(a0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = pkg.dgeqpt(work, d_factor=1.25, nnz=8, seed=0, timings=True, fast_sketch=fast_sketch)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        if it == 0:
            continue
        tm = list(res.ctx.timings_ms)
        if best is None or tm[6] < best[1][6]:
            best = (wall, tm, res.k, res.k0, res.ctx.k_sk)
    wall, tm, k, k0, ksk = best
    names = ["sketch", "qrcp", "rank_select", "precondition", "cholesky_qr", "undo", "total", "comm"]
    out = dict(config=name, fast_sketch=fast_sketch, m=m, n=n, k=k, k0=k0, k_sk=ksk, wall_ms=wall * 1e3,
               phases_ms=dict(zip(names, [round(x, 4) for x in tm])),
               canonical_gflops=canon / (tm[6] * 1e-3) / 1e9)
    print(json.dumps(out), flush=True)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["C1", "C2"])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--fast-sketch", action="store_true", help="CQRRPT_GPU_FAST_SKETCH (c-split sketch)")
    args = ap.parse_args()
    for c in args.configs:
        run(c, args.reps, args.fast_sketch)
        torch.cuda.empty_cache()
