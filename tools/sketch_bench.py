"""Device time of the exact SASO sketch (K1 plan + CSR + K2 apply + reduce)
on BASELINE shapes; HBM roofline fraction of the algorithmic bytes
8 m n + 8 d n. usage: python tools/sketch_bench.py [C2 C4 C5_256 m,n,d ...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_08316_b200 import kernels  # noqa: E402
from tools.workloads import CONFIGS  # noqa: E402

HBM = 6553.6


def main(names):
    for name in names:
        if "," in name:  # an explicit shape m,n,d
            m, n, d = (int(v) for v in name.split(","))
        else:
            cfg = CONFIGS[name]
            m, n = cfg["m"], cfg["n"]
            d = int(-(-cfg["gamma"] * n // 1))
        a = torch.randn((n, m), dtype=torch.float64, device="cuda").t()
        for _ in range(2):
            kernels.saso_sketch(a, d, 8, 0)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            kernels.saso_sketch(a, d, 8, 0)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = min(ts)
        byts = 8.0 * m * n + 8.0 * d * n
        print(json.dumps({"config": name, "m": m, "n": n, "d": d, "ms": round(t, 3),
                          "GBps": round(byts / t / 1e6, 1), "hbm_frac": round(byts / t / 1e6 / HBM, 4)}), flush=True)
        del a
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main(sys.argv[1:] or ["C2", "C3", "C5_256", "C5_1024", "C4", "C5_2048"])
