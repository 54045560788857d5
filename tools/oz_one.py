"""One trsm_right through the INT8 engine at (m, k) for ncu captures."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_08316_b200 as pkg  # noqa: E402
from paper_2311_08316_b200 import kernels  # noqa: E402

m, k = int(sys.argv[1]), int(sys.argv[2])
os.environ["CQRRPT_GPU_TRSM"] = sys.argv[3] if len(sys.argv) > 3 else "oz"
b = pkg.colmajor_empty(m, k)
b.copy_(torch.randn(m, k, dtype=torch.float64, device="cuda"))
a = torch.randn(int(1.25 * k), k, dtype=torch.float64, device="cuda")
u = pkg.to_device_colmajor(torch.linalg.qr(a, mode="r")[1][:k, :k])
for _ in range(2):
    x = kernels.trsm_right(b, u)
torch.cuda.synchronize()
print("done")
