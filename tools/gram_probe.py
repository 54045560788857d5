"""Ozaki-II INT8 Gram vs the DMMA Gram: accuracy against an extended-precision
reference (entries relative to ||x_i|| ||x_j||) and device time.
usage: python tools/gram_probe.py [--time]"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_08316_b200 import kernels  # noqa: E402


def gram_with(engine, x):
    os.environ["CQRRPT_GPU_GRAM"] = engine
    g = kernels.gram(x)
    torch.cuda.synchronize()
    return g


def exact_entries(xh, pairs):
    out = []
    for i, j in pairs:
        out.append(math.fsum((xh[:, i] * xh[:, j]).astype(np.longdouble).tolist()) if False else
                   float(np.sum(xh[:, i].astype(np.longdouble) * xh[:, j].astype(np.longdouble))))
    return np.array(out)


def accuracy(name, x):
    xh = x.cpu().numpy()
    m, k = xh.shape
    rng = np.random.default_rng(0)
    pairs = [(int(a), int(b)) for a, b in zip(rng.integers(0, k, 400), rng.integers(0, k, 400))] + [(i, i) for i in range(min(k, 50))]
    ex = exact_entries(xh, pairs)
    nrm = np.linalg.norm(xh, axis=0)
    scale = np.array([nrm[i] * nrm[j] for i, j in pairs])
    res = {}
    for eng in ("dmma", "ozaki"):
        g = gram_with(eng, x).cpu().numpy()
        got = np.array([g[i, j] for i, j in pairs])
        res[eng] = np.max(np.abs(got - ex) / scale) / 1.11e-16
        sym = np.array_equal(g, g.T)
        res[eng + "_sym"] = sym
    print(f"{name}: max err / (u ||x_i|| ||x_j||): dmma {res['dmma']:.2f}  ozaki {res['ozaki']:.2f}  "
          f"symmetric dmma={res['dmma_sym']} ozaki={res['ozaki_sym']}", flush=True)


def main():
    torch.manual_seed(0)
    m, k = 200000, 384
    x = torch.randn((k, m), dtype=torch.float64, device="cuda").t()
    accuracy("gaussian 200000x384", x)
    y = x.clone()
    y[:5] *= 1e4  # spiky columns: a few huge entries
    accuracy("spiky rows x1e4", y)
    f = 10.0 ** (-8.0 * torch.rand(k, dtype=torch.float64, device="cuda"))
    accuracy("graded columns 1..1e-8", (x * f[None, :]).t().contiguous().t())
    z = x.clone()
    z[:, 7] = 0.0
    accuracy("zero column", z)
    if "--time" in sys.argv:
        for (m, k) in [(131072, 1024), (262144, 2048), (4194304, 2048), (1048576, 4096)]:
            x = torch.randn((k, m), dtype=torch.float64, device="cuda").t()
            for eng in ("dmma", "ozaki"):
                os.environ["CQRRPT_GPU_GRAM"] = eng
                kernels.gram(x)
                torch.cuda.synchronize()
                best = 1e9
                for _ in range(3):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    kernels.gram(x)
                    e1.record()
                    e1.synchronize()
                    best = min(best, e0.elapsed_time(e1))
                print(f"time m={m} k={k} {eng}: {best:.2f} ms ({m * k * (k + 1) / best / 1e9:.1f} TF/s algorithmic)",
                      flush=True)
            del x
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
