"""Command-line driver, the GPU counterpart of the reference's `cqrrpt-cli`
(tools/cqrrpt_cli.cc) for the hot path:

  profile  per-phase device timings (best of --runs) and the flop model
           (run_profile, cqrrpt_cli.cc:128-185)
  factor   read a Matrix Market file, factorize, write Q/R as Matrix Market plus
           a 1-based pivot list (run_factor, cqrrpt_cli.cc:187-212)
  gen      write a test matrix in Matrix Market format (cqrrpt_cli.cc:296-303)

Matrix families are generated on the device with torch from the reference's
definitions (testmat.cc: spectra, Kahan, exact rank, high coherence); the
values are not the reference generator's bits (its counter-RNG Householder
constructions are host code), which profiling does not need.

usage: python -m paper_2311_08316_b200.cli profile --matrix gaussian --m 131072 --n 1024 --nnz 8
       python -m paper_2311_08316_b200.cli factor --in A.mtx --out-prefix out
"""
from __future__ import annotations

import argparse
import math
import sys

import numpy as np

from .matrix_market import read_matrix_market, write_matrix_market

FAMILIES = ("staircase", "polynomial-decay", "high-coherence", "gaussian", "exact-rank", "kahan")


def spectrum_values(kind: str, n: int, cond: float) -> np.ndarray:
    """spectrum_values (testmat.cc:29-77) for the two named spectra."""
    sigma = np.empty(n)
    if kind == "polynomial-decay":
        if cond < 1.0:
            raise ValueError("spectrum_values: cond target must be >= 1")
        t = (n + 9) // 10
        sigma[:t] = 1.0
        if t < n:
            span = float(n - t)
            p = math.log(cond) / math.log(span) if span > 1.0 else 1.0
            sigma[t:] = np.arange(1, n - t + 1, dtype=np.float64) ** (-p)
            sigma[n - 1] = 1.0 / cond
    elif kind == "staircase":
        levels = (1.0, 8e-10, 4e-10, 1e-10)
        for i in range(n):
            pos = i + 1
            lv = 3
            if pos <= (n + 3) // 4:
                lv = 0
            elif pos <= (n + 1) // 2:
                lv = 1
            elif pos <= (3 * n + 3) // 4:
                lv = 2
            sigma[i] = levels[lv]
    else:
        raise ValueError(kind)
    return sigma


def build_matrix(kind: str, m: int, n: int, seed: int, cond: float = 1e10, scale: float = 1e10,
                 rank: int = 10, theta: float = 0.285):
    """A column-major CUDA float64 tensor of the named family (build_matrix,
    cqrrpt_cli.cc:43-55)."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(int(seed))
    f64 = dict(dtype=torch.float64, device="cuda")
    if kind == "gaussian":
        a = torch.randn((n, m), generator=g, **f64).t()
    elif kind == "exact-rank":
        a = (torch.randn((m, rank), generator=g, **f64) @ torch.randn((rank, n), generator=g, **f64))
        a = a.t().contiguous().t()
    elif kind in ("staircase", "polynomial-decay"):
        if m < n:
            raise ValueError("gen_spectral: requires m >= n")
        u = torch.linalg.qr(torch.randn((m, n), generator=g, **f64))[0]
        v = torch.linalg.qr(torch.randn((n, n), generator=g, **f64))[0]
        s = torch.from_numpy(spectrum_values(kind, n, cond)).cuda()
        a = ((u * s) @ v.t()).t().contiguous().t()
    elif kind == "high-coherence":  # testmat.cc:95-124: stacked identities + n scaled rows
        if m < n:
            raise ValueError("gen_high_coherence: requires m >= n")
        a = torch.zeros((n, m), **f64)
        idx = torch.arange(m, device="cuda")
        a[idx % n, idx] = 1.0
        rows = torch.randperm(m, generator=g, device="cuda")[:n]
        a[torch.arange(n, device="cuda"), rows] *= scale
        a = a.t()
    elif kind == "kahan":  # testmat.cc:126-139
        if not (0.0 < theta < math.pi / 2):
            raise ValueError("gen_kahan: theta must lie in (0, pi/2)")
        s, c = math.sin(theta), math.cos(theta)
        k = np.zeros((n, n), order="F")
        row_scale = 1.0
        for i in range(n):
            k[i, i] = row_scale
            k[i, i + 1:] = -c * row_scale
            row_scale *= s
        a = torch.from_numpy(np.ascontiguousarray(k.T)).cuda().t()
    else:
        raise ValueError(f"unknown matrix family: {kind}")
    return a


def run_profile(args) -> int:
    import torch

    from .cqrrpt import colmajor_empty, dgeqpt
    a0 = build_matrix(args.matrix, args.m, args.n, args.seed, args.cond, args.scale, args.rank, args.theta)
    m, n = a0.shape
    work = colmajor_empty(m, n)
    best, res = None, None
    for _ in range(max(1, args.runs) + 1):  # the first call warms up
        work.copy_(a0)
        torch.cuda.synchronize()
        res = dgeqpt(work, d_factor=args.gamma, nnz=args.nnz, seed=args.seed, timings=True,
                     sketch_family=args.family, fast_sketch=args.fast_sketch)
        t = list(res.ctx.timings_ms)
        if best is None or t[6] < best[6]:
            best = t
    names = ("sketch", "qrcp", "rank-select", "precondition", "cholesky-qr", "undo")
    print(f"profile: {args.matrix} {m}x{n}, {args.family} gamma={args.gamma:g} nnz={args.nnz}, "
          f"best of {args.runs} runs (device time)")
    for name, v in zip(names, best[:6]):
        print(f"  {name:<12s} {v / 1e3:10.6f}s  {100.0 * v / best[6]:5.1f}%")
    print(f"  {'total':<12s} {best[6] / 1e3:10.6f}s  (phases cover {100.0 * sum(best[:6]) / best[6]:.1f}%)")
    print(f"  detected rank k={res.k}, flop model {res.ctx.flop_estimate:.4e}, "
          f"canonical {(2.0 * m * n * n - 2.0 * n ** 3 / 3.0) / (best[6] * 1e-3) / 1e9:.1f} GFLOP/s")
    if args.out:
        with open(args.out, "w") as f:
            f.write("experiment,matrix,family,gamma,nnz,seed,metric,k,value\n")
            for name, v in zip(("time_sketch", "time_qrcp", "time_rank_select", "time_precondition",
                                "time_cholesky_qr", "time_undo", "time_total"), best[:7]):
                f.write(f"profile,{args.matrix},{args.family},{args.gamma:g},{args.nnz},{args.seed},{name},"
                        f"{res.k},{v / 1e3:.17g}\n")
            f.write(f"profile,{args.matrix},{args.family},{args.gamma:g},{args.nnz},{args.seed},flop_model,"
                    f"{res.k},{res.ctx.flop_estimate:.17g}\n")
    return 0


def run_factor(args) -> int:
    from .cqrrpt import CqrrptConfig, SketchFamily, cqrrpt
    m = read_matrix_market(args.inp)
    cfg = CqrrptConfig(gamma=args.gamma, nnz_per_col=args.nnz, seed=args.seed,
                       family={"gaussian": SketchFamily.gaussian, "srft": SketchFamily.srft}.get(args.family,
                                                                                                SketchFamily.saso))
    out = cqrrpt(m, cfg)
    write_matrix_market(args.out_prefix + "_Q.mtx", out.factorization.q)
    write_matrix_market(args.out_prefix + "_R.mtx", out.factorization.r)
    with open(args.out_prefix + "_J.txt", "w") as f:
        for p in out.factorization.pivots:
            f.write(f"{int(p) + 1}\n")  # 1-based pivot list
    d = out.diagnostics
    print(f"factor: {m.shape[0]}x{m.shape[1]} -> k={out.k} (k0={out.k0}), cond(M_pre) est {d.cond_m_pre:.3e}, "
          f"trunc ratio {d.truncation_ratio:.3e}")
    if d.validation is not None:
        v = d.validation
        print(f"factor: validation {'pass' if v.passed else 'FAIL'} (orth {v.orth_loss:.3e}, recon {v.recon_rel:.3e})")
        return 0 if v.passed else 1
    return 0


def run_gen(args) -> int:
    a = build_matrix(args.matrix, args.m, args.n, args.seed, args.cond, args.scale, args.rank, args.theta)
    write_matrix_market(args.out, a.cpu().numpy(), args.format)
    print(f"gen: wrote {a.shape[0]}x{a.shape[1]} {args.matrix} matrix to {args.out}")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="cqrrpt-gpu", description="randomized pivoted QR for tall matrices on B200")
    ap.add_argument("--seed", type=int, default=0, help="base seed for all randomness")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def matrix_opts(p):
        p.add_argument("--matrix", default="gaussian", choices=FAMILIES)
        p.add_argument("--m", type=int, default=1000)
        p.add_argument("--n", type=int, default=100)
        p.add_argument("--cond", type=float, default=1e10)
        p.add_argument("--scale", type=float, default=1e10)
        p.add_argument("--rank", type=int, default=10)
        p.add_argument("--theta", type=float, default=0.285)

    def sketch_opts(p):
        p.add_argument("--family", default="saso", choices=("saso", "gaussian", "srft"))
        p.add_argument("--gamma", type=float, default=1.25)
        p.add_argument("--nnz", type=int, default=4)

    prof = sub.add_parser("profile", help="per-phase timings (best of --runs) and flop model")
    matrix_opts(prof)
    sketch_opts(prof)
    prof.add_argument("--runs", type=int, default=5)
    prof.add_argument("--out", default="", help="CSV output path for the timing rows")
    prof.add_argument("--fast-sketch", action="store_true", help="CQRRPT_GPU_FAST_SKETCH (c-split sketch)")
    fac = sub.add_parser("factor", help="Matrix Market in -> Q/R Matrix Market + 1-based pivots out")
    fac.add_argument("--in", dest="inp", required=True)
    fac.add_argument("--out-prefix", default="factor")
    sketch_opts(fac)
    gen = sub.add_parser("gen", help="write a test matrix in Matrix Market format")
    matrix_opts(gen)
    gen.add_argument("--out", default="matrix.mtx")
    gen.add_argument("--format", default="array", choices=("array", "coordinate"))
    args = ap.parse_args(argv)
    try:
        return {"profile": run_profile, "factor": run_factor, "gen": run_gen}[args.cmd](args)
    except (ValueError, RuntimeError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
