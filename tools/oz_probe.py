"""INT8 tensor-core TRSM engine (csrc/oztrsm.cu) vs the DMMA engine: accuracy
and device time of trsm_right on (m, k) with a well-conditioned and a graded
(C5-like) upper-triangular U. Usage: python tools/oz_probe.py [m k ...]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_08316_b200 as pkg  # noqa: E402
from paper_2311_08316_b200 import kernels  # noqa: E402


def make_u(k, graded, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.randn(int(1.25 * k), k, dtype=torch.float64, device="cuda", generator=g)
    if graded:
        a = a * torch.pow(10.0, -8.0 * torch.randperm(k, generator=torch.Generator().manual_seed(seed)).double() / max(k - 1, 1)).cuda()
    r = torch.linalg.qr(a, mode="r")[1][:k, :k]
    return pkg.to_device_colmajor(r)


def run(m, k, graded, reps=3):
    g = torch.Generator(device="cuda").manual_seed(1)
    b = pkg.colmajor_empty(m, k + 3)
    b.copy_(torch.randn(m, k + 3, dtype=torch.float64, device="cuda", generator=g))
    u = make_u(k, graded, 2)
    cols = torch.randperm(k + 3, generator=torch.Generator().manual_seed(3))[:k].to("cuda")
    out = {}
    for eng in ("dmma", "oz"):
        os.environ["CQRRPT_GPU_TRSM"] = eng
        x = kernels.trsm_right(b, u, cols=cols)
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            x = kernels.trsm_right(b, u, cols=cols)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[eng] = (x, min(ts))
    xd, xo = out["dmma"][0], out["oz"][0]
    bc = b[:, cols]
    res_d = (torch.linalg.matrix_norm(xd @ u - bc) / torch.linalg.matrix_norm(bc)).item() if m * k <= 2**27 else float("nan")
    res_o = (torch.linalg.matrix_norm(xo @ u - bc) / torch.linalg.matrix_norm(bc)).item() if m * k <= 2**27 else float("nan")
    diff = (torch.linalg.vector_norm(xo - xd, dim=0) / torch.linalg.vector_norm(xd, dim=0)).max().item()
    flops = m * k * k
    print(f"m={m} k={k} graded={graded}: dmma {out['dmma'][1]:.2f} ms ({flops / out['dmma'][1] / 1e9:.1f} TF/s) "
          f"oz {out['oz'][1]:.2f} ms ({flops / out['oz'][1] / 1e9:.1f} TF/s)  max col rel diff {diff:.2e} "
          f"resid dmma {res_d:.2e} oz {res_o:.2e}", flush=True)
    del out, xd, xo, b, bc
    torch.cuda.empty_cache()


if __name__ == "__main__":
    args = [int(v) for v in sys.argv[1:]] or [1000, 300, 16384, 256, 70001, 513, 262144, 1024, 1048576, 2048]
    for i in range(0, len(args), 2):
        for graded in (False, True):
            run(args[i], args[i + 1], graded)
