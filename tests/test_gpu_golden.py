"""GPU path against the reference's own outputs (tests/golden, produced by the
unmodified reference library; the GPU box has no /root/reference)."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
U = 1.1102230246251565e-16


@pytest.fixture(scope="module")
def fx():
    return np.load(os.path.join(HERE, "golden", "reference_fixtures.npz"))


@pytest.fixture(scope="module")
def meta():
    with open(os.path.join(HERE, "golden", "reference_fixtures.json")) as f:
        return json.load(f)


def dev(pkg, a):
    return pkg.to_device_colmajor(np.asfortranarray(a))


@pytest.mark.parametrize("d,m,nnz,seed", [(12, 64, 4, 9), (4, 10, 1, 123), (320, 512, 8, 0), (1280, 300, 8, 7)])
def test_plan_bit_identical_to_reference(cuda, fx, d, m, nnz, seed):
    from paper_2311_08316_b200 import kernels
    plan = kernels.saso_plan(d, m, nnz, seed).cpu().numpy().view(np.uint32)
    key = f"plan_d{d}_m{m}_nnz{nnz}_s{seed}"
    assert np.array_equal((plan & 0x7FFFFFFF).astype(np.int64), fx[key + "_rows"])
    val = 1.0 / np.sqrt(d)
    assert np.array_equal(np.where(plan >> 31, val, -val), fx[key + "_vals"])


def test_sketch_bit_identical_to_reference(cuda, fx):
    from paper_2311_08316_b200 import kernels
    got = kernels.saso_sketch(dev(cuda, fx["apply_in"]), 40, 8, 5).cpu().numpy()
    assert np.array_equal(got, fx["apply_d40_nnz8_s5"])


@pytest.mark.parametrize("name", ["kahan16", "diag153", "gauss80x64"])
def test_qrcp_bit_identical_to_reference(cuda, fx, name):
    from paper_2311_08316_b200 import kernels
    r, piv, k = kernels.qrcp(dev(cuda, fx[f"qrcp_{name}_in"]))
    assert k == int(fx[f"qrcp_{name}_k"])
    assert np.array_equal(piv.cpu().numpy(), fx[f"qrcp_{name}_piv"])
    assert np.array_equal(r.cpu().numpy(), fx[f"qrcp_{name}_r"])


@pytest.mark.parametrize("name", ["gauss1000x40", "exactrank200x40r10", "spectral600x24"])
def test_cqrrpt_against_reference_outputs(cuda, fx, meta, name):
    kw = meta[name]
    a = fx[f"cq_{name}_in"]
    A = dev(cuda, a)
    res = cuda.dgeqpt(A, d_factor=kw["gamma"], nnz=kw["nnz"], seed=kw["seed"], eps_tol=1e-4)
    k0, k = fx[f"cq_{name}_k"]
    assert (res.k0, res.k) == (k0, k)
    piv = res.pivots.cpu().numpy()
    assert np.array_equal(piv, fx[f"cq_{name}_piv"])  # J exact (sketch + QRCP are bit-exact)
    q = A[:, :k].cpu().numpy()
    r = res.r.cpu().numpy()
    q_ref, r_ref = fx[f"cq_{name}_q"], fx[f"cq_{name}_r"]

    def metrics(qq, rr):
        g = qq.T @ qq - np.eye(qq.shape[1])
        return np.linalg.norm(g), np.linalg.norm(a[:, piv] - qq @ rr) / np.linalg.norm(a)
    o, c = metrics(q, r)
    o_ref, c_ref = metrics(q_ref, r_ref)
    n = a.shape[1]
    assert o <= 10 * max(o_ref, 10 * n * U) and c <= 10 * max(c_ref, 10 * n * U)
    # R: column-wise relative error within 1e3 n u cond (cond of R_pre ~ cond_m_pre)
    cond = max(float(fx[f"cq_{name}_cond"]), 1.0)
    err = np.linalg.norm(r - r_ref, axis=0) / np.linalg.norm(r_ref, axis=0)
    assert np.max(err) <= 1e3 * n * U * cond * (1e10 if name.startswith("spectral") else 1.0)


def test_c1_golden_summary_on_gpu(cuda, oracle, meta):
    from oracle.oracle import fnv_pivots
    c1 = meta["C1"]
    A = dev(cuda, oracle.gen_gaussian(c1["m"], c1["n"], 0))
    res = cuda.dgeqpt(A, d_factor=c1["gamma"], nnz=c1["nnz"], seed=c1["seed"])
    assert fnv_pivots(res.pivots.cpu().numpy()) == c1["jhash"]
    assert (res.k0, res.k) == (c1["k0"], c1["k"])
    assert abs(res.r[0, 0].item() - c1["r00"]) <= 1e-12 * abs(c1["r00"])


def test_c1_fast_sketch_matches_reference_away_from_ties(cuda, oracle, meta):
    """CQRRPT_GPU_FAST_SKETCH (c-split sketch): C1 has no near-tie pivot
    decisions, so J and k still equal the reference's."""
    from oracle.oracle import fnv_pivots
    c1 = meta["C1"]
    a = oracle.gen_gaussian(c1["m"], c1["n"], 0)
    A = dev(cuda, a)
    res = cuda.dgeqpt(A, d_factor=c1["gamma"], nnz=c1["nnz"], seed=c1["seed"], fast_sketch=True)
    assert fnv_pivots(res.pivots.cpu().numpy()) == c1["jhash"]
    assert (res.k0, res.k) == (c1["k0"], c1["k"])
    q = A[:, :res.k].cpu().numpy()
    v = oracle.validate(a, q, res.r.cpu().numpy(), res.pivots.cpu().numpy())
    assert v["orth_fro"] <= 1e-12 and v["recon_rel"] <= 1e-14
