"""QRCP of a d x n Gaussian sketch (device time; CQRRPT_QRCP_TRACE=1 prints the
per-phase SM-cycle trace). usage: python tools/qrcp_probe.py d n [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_08316_b200 import kernels  # noqa: E402

d, n = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
g = torch.Generator(device="cuda").manual_seed(0)
m0 = torch.randn((n, d), dtype=torch.float64, device="cuda", generator=g).t()
best = 1e9
for _ in range(reps):
    msk = m0.clone()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r, j, k = kernels.qrcp(msk)
    e1.record()
    e1.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(f"qrcp d={d} n={n}: {best:.2f} ms, {best * 1e3 / n:.2f} us/step, k={k}")
