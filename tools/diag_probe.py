"""Device time of dgeqpt with and without CQRRPT_GPU_DIAGNOSTICS (cond_m_pre
and truncation_ratio as the reference reports them)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_08316_b200 as pkg  # noqa: E402

for (m, n) in [(16384, 256), (131072, 1024)]:
    a0 = torch.randn((n, m), dtype=torch.float64, device="cuda").t()
    for diag in (False, True, False, True):
        w = a0.clone()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = pkg.dgeqpt(w, d_factor=1.25, nnz=8, seed=0, diagnostics=diag, timings=True)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        print(f"m={m} n={n} diagnostics={diag}: wall {t * 1e3:.1f} ms, device total {res.ctx.timings_ms[6]:.1f} ms, "
              f"cond {res.ctx.cond_m_pre:.4g}", flush=True)
