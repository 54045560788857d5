"""One exact SASO sketch at (m, n, d) for ncu captures."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_08316_b200 import kernels  # noqa: E402

m, n, d = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
a = torch.randn((n, m), dtype=torch.float64, device="cuda").t()
kernels.saso_sketch(a, d, 8, 0)
torch.cuda.synchronize()
kernels.saso_sketch(a, d, 8, 0)
torch.cuda.synchronize()
print("ok")
