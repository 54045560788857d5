"""Device time of trsm_right through the INT8 engine at (m, k), best of 3.
usage: python tools/oz_time.py m k"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_08316_b200 as pkg  # noqa: E402
from paper_2311_08316_b200 import kernels  # noqa: E402

m, k = int(sys.argv[1]), int(sys.argv[2])
os.environ.setdefault("CQRRPT_GPU_TRSM", "oz")
b = pkg.colmajor_empty(m, k)
b.copy_(torch.randn(m, k, dtype=torch.float64, device="cuda"))
a = torch.randn(int(1.25 * k), k, dtype=torch.float64, device="cuda")
u = pkg.to_device_colmajor(torch.linalg.qr(a, mode="r")[1][:k, :k])
ts = []
for _ in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x = kernels.trsm_right(b, u)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"m={m} k={k} dbg={os.environ.get('CQRRPT_OZ_DBG', '0')} stages={os.environ.get('CQRRPT_OZ_STAGES', '-')}: {min(ts[1:]):.2f} ms")
