"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libcqrrpt_ref.so, i.e. the
reference compiled from /root/reference by oracle/Makefile):

    python tests/golden/make_golden.py

Every array here is an output of the reference library itself (never of the
restatement or of the GPU code). The fixtures are small (< 1 MB total) and
travel with the repository so the GPU box, which has no /root/reference, can
check against the reference's own bits.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Reference, fnv_pivots  # noqa: E402


def main():
    R = Reference()
    out = {}
    # --- SASO plans (sketch.cc:73-99)
    for (d, m, nnz, seed) in [(12, 64, 4, 9), (4, 10, 1, 123), (320, 512, 8, 0), (1280, 300, 8, 7)]:
        rows, vals = R.saso_sample(d, m, nnz, seed)
        out[f"plan_d{d}_m{m}_nnz{nnz}_s{seed}_rows"] = rows
        out[f"plan_d{d}_m{m}_nnz{nnz}_s{seed}_vals"] = vals
    # --- SASO apply (sketch.cc:131-146)
    a = R.gen_gaussian(512, 32, 3)
    out["apply_in"] = a
    out["apply_d40_nnz8_s5"] = R.saso_apply(40, a, 8, 5)
    # --- QRCP (qrcp.cc:35-97)
    for name, m in [("kahan16", R.gen_kahan(16, 0.285)), ("diag153", np.diag([1.0, 5.0, 3.0])),
                    ("gauss80x64", R.gen_gaussian(80, 64, 8))]:
        r, piv, k = R.qrcp(m)
        out[f"qrcp_{name}_in"] = np.asfortranarray(m)
        out[f"qrcp_{name}_r"] = r
        out[f"qrcp_{name}_piv"] = piv
        out[f"qrcp_{name}_k"] = np.array(k)
    # --- cqrrpt end to end (cqrrpt.cc:317-328)
    cases = {
        "gauss1000x40": (R.gen_gaussian(1000, 40, 5), dict(gamma=1.25, nnz=8, seed=0)),
        "exactrank200x40r10": (R.gen_exact_rank(200, 40, 10, 24), dict(gamma=1.25, nnz=4, seed=25)),
        "spectral600x24": (R.gen_spectral(600, 24, 10.0 ** (-10 * np.arange(24) / 23), 2),
                           dict(gamma=2.0, nnz=4, seed=3)),
    }
    for name, (m, kw) in cases.items():
        res = R.cqrrpt(m, eps_tol=1e-4, **kw)
        out[f"cq_{name}_in"] = m
        out[f"cq_{name}_q"] = res.q
        out[f"cq_{name}_r"] = res.r
        out[f"cq_{name}_piv"] = res.pivots
        out[f"cq_{name}_k"] = np.array([res.k0, res.k])
        out[f"cq_{name}_cond"] = np.array(res.cond_m_pre)
    np.savez_compressed(os.path.join(HERE, "reference_fixtures.npz"), **out)
    meta = {name: kw for name, (_, kw) in cases.items()}
    # --- C1 summary (BASELINE config 1)
    c1 = R.gen_gaussian(16384, 256, 0)
    res = R.cqrrpt(c1, gamma=1.25, nnz=8, seed=0)
    meta["C1"] = dict(m=16384, n=256, gamma=1.25, nnz=8, seed=0, k0=res.k0, k=res.k, jhash=fnv_pivots(res.pivots),
                      j8=[int(v) for v in res.pivots[:8]], r00=float(res.r[0, 0]), cond_m_pre=res.cond_m_pre)
    with open(os.path.join(HERE, "reference_fixtures.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
