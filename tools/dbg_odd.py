import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
os.environ["CQRRPT_GPU_TRSM"] = "oz"
import paper_2311_08316_b200 as pkg
from paper_2311_08316_b200 import _lib
from paper_2311_08316_b200.kernels import _p
for (m, k, gather) in [(70001, 128, True), (70001, 256, True), (70001, 256, False), (70001, 384, False)]:
    ld = m + 1
    b = torch.randn((k + 3, ld), dtype=torch.float64, device="cuda")
    a = torch.randn(int(1.25 * k), k, dtype=torch.float64, device="cuda")
    u = pkg.to_device_colmajor(torch.linalg.qr(a, mode="r")[1][:k, :k])
    xbuf = torch.full((k, ld), 7.0, dtype=torch.float64, device="cuda")
    cols = torch.randperm(k + 3)[:k].to("cuda") if gather else None
    _lib.check(_lib.load().cqrrpt_gpu_trsm_right(m, k, _p(b), ld, _p(cols), _p(u), k, _p(xbuf), ld, None), "t")
    torch.cuda.synchronize()
    pad = xbuf[:, m].cpu().numpy()
    bad = np.nonzero(pad != 7.0)[0]
    print(m, k, gather, "padding written in columns:", bad[:5], "...", len(bad))
