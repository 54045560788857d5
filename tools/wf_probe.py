"""Time cqrrpt_gpu_dgeqpt_host at C2 with and without the Q wavefront (pinned buffers)."""
import time

import torch

import paper_2311_08316_b200 as pkg

m, n = 131072, 1024
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.randn((n, m), dtype=torch.float64, device="cuda", generator=g)
ha = torch.empty((n, m), dtype=torch.float64).pin_memory()
ha.copy_(a)
hq = torch.empty((n, m), dtype=torch.float64).pin_memory()
hr = torch.empty((n, n), dtype=torch.float64).pin_memory()
for wf in (True, False, True, False):
    ts = []
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = pkg.dgeqpt_host(ha.t(), d_factor=1.25, nnz=8, seed=0, q_out=hq.t(), r_out=hr.t(), wavefront=wf)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"wavefront={wf} k={res.k} ms={sorted(ts)}", flush=True)
