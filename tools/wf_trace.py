"""One C2 dgeqpt_host call with CQRRPT_WF_TRACE=1 after a warm-up (prints the Q block timeline)."""
import os
import time

import torch

import paper_2311_08316_b200 as pkg

m, n = 131072, 1024
g = torch.Generator(device="cuda").manual_seed(0)
ha = torch.empty((n, m), dtype=torch.float64).pin_memory()
ha.copy_(torch.randn((n, m), dtype=torch.float64, device="cuda", generator=g))
hq = torch.empty((n, m), dtype=torch.float64).pin_memory()
hr = torch.empty((n, n), dtype=torch.float64).pin_memory()
for i in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = pkg.dgeqpt_host(ha.t(), d_factor=1.25, nnz=8, seed=0, q_out=hq.t(), r_out=hr.t(), timings=True) \
        if False else pkg.dgeqpt_host(ha.t(), d_factor=1.25, nnz=8, seed=0, q_out=hq.t(), r_out=hr.t())
    torch.cuda.synchronize()
    print(f"call {i}: {(time.perf_counter() - t0) * 1e3:.2f} ms", flush=True)
