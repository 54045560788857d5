"""Full-size golden summaries of the UNMODIFIED reference (BASELINE configs).

TEST INFRASTRUCTURE. Run in the build container (needs oracle/_ref, i.e. the
reference compiled from /root/reference by oracle/Makefile):

    OMP_NUM_THREADS=8 python tests/golden/make_fullsize_golden.py [names...]

For each case the input is built with the reference's OWN generators
(testmat.cc:79-93 gen_spectral, 141-151 gen_gaussian / gen_exact_rank; C5's
column scaling is the harness definition pinned in SURVEY §8(d)), the
reference's cqrrpt() (cqrrpt.cc:317-328) factors it with validate_output=false
(best of R runs, timings.total as cqrrpt_cli.cc:147-150 reports it), and we
record what the GPU must reproduce:

  k0, k, cond_m_pre, the full pivot vector J, |diag(R)|, R(0,0),
  the sha256 of the input bytes (the GPU box rebuilds the input with the
  oracle's restated generators and checks this hash first), and the first
  near-tie step of the reference's QRCP on its sketch (SURVEY §8(c) tie rule:
  gap (w1 - w2)/w1 <= 1e3 * u * n), from the oracle's instrumented QRCP on the
  reference's own sketch (the oracle's QRCP is bit-identical to the
  reference's, tests/test_oracle.py).

Output: tests/golden/fullsize_<name>.npz + fullsize_golden.json (summaries,
timings, host core count). A CPU timing table goes to
profiles/cpu_reference_fullsize.json.
"""
import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, Reference, fnv_pivots, UNIT_ROUNDOFF  # noqa: E402

JSON = os.path.join(HERE, "fullsize_golden.json")
PROF = os.path.join(ROOT, "profiles", "cpu_reference_fullsize.json")


def canonical(m, n):
    return 2.0 * m * n * n - 2.0 * n ** 3 / 3.0


def sha(a):
    return hashlib.sha256(np.asfortranarray(a).tobytes(order="F")).hexdigest()


def build_input(R, O, name):
    """The BASELINE inputs."""
    if name in ("C1", "C1_t1"):
        return R.gen_gaussian(16384, 256, 0), 1.25
    if name == "C2":
        m, n = 131072, 1024
        sig = 10.0 ** (-10.0 * np.arange(n) / (n - 1))
        return R.gen_spectral(m, n, sig, 0), 1.25
    if name in ("C3", "C3b"):
        m, n, r = 262144, 2048, 1024
        ab = R.gen_exact_rank(m, n, r, 0)
        g = R.gen_gaussian(m, n, 1)
        noise = 1e-12 if name == "C3" else 1e-14
        fro = float(np.sqrt(np.sum(ab * ab)))
        scale = noise * fro / np.sqrt(float(m) * float(n))
        ab += scale * g
        return ab, 1.25
    if name.startswith("C5_256_g"):
        gamma = float(name.split("_g")[1])
        a = R.gen_gaussian(4194304, 256, 0)
        a, _ = O.c5_scale_columns(a, 8.0, 0)
        return a, gamma
    raise KeyError(name)


def main():
    names = sys.argv[1:] or ["C1", "C1_t1", "C2", "C5_256_g1.0", "C5_256_g1.25", "C5_256_g2.0", "C3", "C3b"]
    R, O = Reference(), Oracle()
    meta = json.load(open(JSON)) if os.path.exists(JSON) else {}
    prof = json.load(open(PROF)) if os.path.exists(PROF) else {}
    threads = R.num_threads()
    reps = {"C1": 5, "C1_t1": 5, "C2": 3}
    c5cache = {}
    for name in names:
        t0 = time.time()
        if name.startswith("C5_256") and "a" in c5cache:
            a, gamma = c5cache["a"], float(name.split("_g")[1])
        else:
            a, gamma = build_input(R, O, name)
            if name.startswith("C5_256"):
                c5cache["a"] = a
        gen_s = time.time() - t0
        m, n = a.shape
        h = sha(a)
        best, res = None, None
        R.set_threads(1 if name == "C1_t1" else threads)
        for _ in range(reps.get(name, 1)):
            r = R.cqrrpt(a, gamma=gamma, nnz=8, eps_tol=1e-4, seed=0, validate=False)
            t = r.extra["timings"]["total"]
            if best is None or t < best:
                best, res = t, r
        d = R.sketch_rows_for(gamma, n)
        msk = R.saso_apply(d, a, 8, 0)
        _, piv_o, ksk, gaps = O.qrcp(msk, gaps=True)
        tie_bar = 1e3 * UNIT_ROUNDOFF * n
        ties = np.nonzero(gaps[:ksk] <= tie_bar)[0]
        first_tie = int(ties[0]) if len(ties) else int(ksk)
        rdiag = np.abs(np.diag(res.r[:, : res.k])) if res.k else np.zeros(0)
        np.savez_compressed(os.path.join(HERE, f"fullsize_{name}.npz"), pivots=res.pivots, rdiag=rdiag,
                            r_row0=res.r[0] if res.k else np.zeros(0), gaps=gaps[:ksk])
        meta[name] = dict(m=m, n=n, gamma=gamma, d=d, nnz=8, seed=0, eps_tol=1e-4, k0=res.k0, k=res.k,
                          k_sk=int(ksk), cond_m_pre=res.cond_m_pre, jhash=fnv_pivots(res.pivots),
                          j8=[int(v) for v in res.pivots[:8]], r00=float(res.r[0, 0]) if res.k else 0.0,
                          rkk=float(res.r[res.k - 1, res.k - 1]) if res.k else 0.0,
                          input_sha256=h, first_near_tie=first_tie, min_gap=float(np.min(gaps[:ksk])),
                          oracle_qrcp_pivots_equal=bool(np.array_equal(piv_o, res.pivots)))
        prof[name] = dict(m=m, n=n, gamma=gamma, threads=1 if name == "C1_t1" else threads, runs=reps.get(name, 1), best_total_s=best,
                          canonical_gflops=canonical(m, n) / best / 1e9, timings_s=res.extra["timings"],
                          gen_s=gen_s, host=platform.processor() or platform.machine(),
                          build="oracle/Makefile: g++ -O3 -march=x86-64-v3 -fopenmp")
        with open(JSON, "w") as f:
            json.dump(meta, f, indent=1)
        os.makedirs(os.path.dirname(PROF), exist_ok=True)
        with open(PROF, "w") as f:
            json.dump(prof, f, indent=1)
        print(name, json.dumps(meta[name]), f"best {best:.2f}s gen {gen_s:.1f}s", flush=True)
        del a


if __name__ == "__main__":
    main()
