"""Small invocations of every hand-synchronised kernel, for compute-sanitizer
(racecheck / synccheck / memcheck). usage:

  compute-sanitizer --tool racecheck python tools/sanitize_driver.py CASE

CASE: qrcp_cluster (16-CTA cluster QRCP, DSMEM records + cluster barriers),
qrcp_grid (cooperative QRCP, flagged-record grid barrier, resident column
phase), qrcp_general (streaming column phase; CQRRPT_QRCP_GENERAL=1),
saso (mbarrier producer/consumer ring of saso_apply_kernel), trsm (PDL chain
of trsm_block_kernel + diagonal-block inverses), potrf, gram, cond (grid
estimator), all_small (one whole dgeqpt).
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_08316_b200 as pkg  # noqa: E402
from paper_2311_08316_b200 import kernels  # noqa: E402


def gauss(m, n, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn((n, m), dtype=torch.float64, device="cuda", generator=g).t()


def main(case):
    torch.cuda.set_device(0)
    if case == "qrcp_cluster":
        msk = gauss(320, 96)
        r, j, k = kernels.qrcp(msk)
    elif case in ("qrcp_grid", "qrcp_general"):
        msk = gauss(640, 512)
        r, j, k = kernels.qrcp(msk)
    elif case == "saso":
        a = gauss(3000, 200)
        kernels.saso_sketch(a, 250, 8, 0)
        kernels.saso_sketch(a, 1250, 8, 0)  # several row blocks per column group
    elif case == "trsm":
        b = gauss(2000, 200)
        u = torch.triu(gauss(200, 200, 1)) + 20 * torch.eye(200, dtype=torch.float64, device="cuda")
        u = u.t().contiguous().t()
        kernels.trsm_right(b, u)
    elif case == "potrf":
        x = gauss(1000, 200)
        g = kernels.gram(x)
        kernels.potrf(g)
    elif case == "gram":
        kernels.gram(gauss(5000, 300))
    elif case == "cond":
        x = gauss(2000, 300)
        g = kernels.gram(x)
        r, _ = kernels.potrf(g)
        kernels.cond_estimate(r, 3)
    elif case == "all_small":
        a = gauss(4000, 96)
        pkg.dgeqpt(a, d_factor=1.25, nnz=8, seed=0, exact_stage2=True)
    else:
        raise SystemExit(f"unknown case {case}")
    torch.cuda.synchronize()
    print(f"{case}: ok")


if __name__ == "__main__":
    main(sys.argv[1])
