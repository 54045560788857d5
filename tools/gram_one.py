"""One Gram at (m, k) with the engine from CQRRPT_GPU_GRAM (for ncu launch lists)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_08316_b200 import kernels  # noqa: E402

m, k = int(sys.argv[1]), int(sys.argv[2])
x = torch.randn((k, m), dtype=torch.float64, device="cuda").t()
kernels.gram(x)
torch.cuda.synchronize()
kernels.gram(x)
torch.cuda.synchronize()
print("ok")
