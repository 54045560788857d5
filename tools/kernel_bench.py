"""Isolated kernel timings (CUDA events) at BASELINE shapes: TRSM (K5a), Gram
(K5b), SASO sketch (K2), QRCP (K3), potrf (K6).

usage: python tools/kernel_bench.py [--m 131072] [--n 1024] [--only trsm,gram,...]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_08316_b200 as pkg  # noqa: E402
from paper_2311_08316_b200 import kernels  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=131072)
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--only", default="trsm,gram,sketch,qrcp,potrf,trtri")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--fast-sketch", action="store_true")
    a = ap.parse_args()
    m, n = a.m, a.n
    d = int(1.25 * n)
    only = set(a.only.split(","))
    out = {"m": m, "n": n}
    A = pkg.colmajor_empty(m, n)
    A.normal_()
    if "trsm" in only or "gram" in only or "potrf" in only or "trtri" in only:
        R = torch.linalg.qr(torch.randn((d, n), dtype=torch.float64, device="cuda"))[1]
        U = R.t().contiguous().t()  # column-major upper triangular
        cols = torch.randperm(n, device="cuda")
        x = [None]

        def trsm():
            x[0] = kernels.trsm_right(A, U, cols=cols)
        ms = timeit(trsm, a.reps)
        out["trsm_ms"] = ms
        out["trsm_tflops"] = m * n * n / (ms * 1e-3) / 1e12
    if "gram" in only:
        g = [None]

        def gram():
            g[0] = kernels.gram(x[0])
        ms = timeit(gram, a.reps)
        out["gram_ms"] = ms
        out["gram_tflops"] = m * n * (n + 1) / (ms * 1e-3) / 1e12
    if "potrf" in only:
        G = kernels.gram(x[0])

        def potrf():
            kernels.potrf(G.clone())
        ms = timeit(potrf, a.reps)
        out["potrf_ms"] = ms
    if "trtri" in only:
        def tri():
            kernels.trtri_upper(U)
        ms = timeit(tri, a.reps)
        out["trtri_ms"] = ms
    if "sketch" in only:
        def sk():
            kernels.saso_sketch(A, d, 8, 0, fast=a.fast_sketch)
        ms = timeit(sk, a.reps)
        out["sketch_ms"] = ms
        out["sketch_gbs"] = (8.0 * m * n + 8.0 * d * n) / (ms * 1e-3) / 1e9
    if "qrcp" in only:
        msk = kernels.saso_sketch(A, d, 8, 0)

        def qr():
            kernels.qrcp(msk.clone())
        ms = timeit(qr, a.reps)
        out["qrcp_ms"] = ms
        out["qrcp_us_per_step"] = ms * 1e3 / n
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
