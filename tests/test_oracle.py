"""CPU tests of the oracle (test infrastructure): pinned against the
reference's golden fixtures (tests/golden, generated from the unmodified
reference), against the compiled reference itself when it is present, and
against the reference test-suite's known answers."""
import json
import os

import numpy as np
import pytest

from oracle.oracle import Oracle, fnv_pivots

HERE = os.path.dirname(os.path.abspath(__file__))
U = 1.1102230246251565e-16


@pytest.fixture(scope="module")
def fx():
    return np.load(os.path.join(HERE, "golden", "reference_fixtures.npz"))


@pytest.fixture(scope="module")
def meta():
    with open(os.path.join(HERE, "golden", "reference_fixtures.json")) as f:
        return json.load(f)


# ------------------------------------------------------------ golden fixtures
@pytest.mark.parametrize("d,m,nnz,seed", [(12, 64, 4, 9), (4, 10, 1, 123), (320, 512, 8, 0), (1280, 300, 8, 7)])
def test_plan_matches_reference_fixture(oracle, fx, d, m, nnz, seed):
    rows, vals = oracle.saso_sample(d, m, nnz, seed)
    key = f"plan_d{d}_m{m}_nnz{nnz}_s{seed}"
    assert np.array_equal(rows, fx[key + "_rows"])
    assert np.array_equal(vals, fx[key + "_vals"])


def test_apply_matches_reference_fixture(oracle, fx):
    assert np.array_equal(oracle.saso_apply(40, fx["apply_in"], 8, 5), fx["apply_d40_nnz8_s5"])


@pytest.mark.parametrize("name", ["kahan16", "diag153", "gauss80x64"])
def test_qrcp_matches_reference_fixture(oracle, fx, name):
    r, piv, k = oracle.qrcp(fx[f"qrcp_{name}_in"])
    assert k == int(fx[f"qrcp_{name}_k"])
    assert np.array_equal(piv, fx[f"qrcp_{name}_piv"])
    assert np.array_equal(r, fx[f"qrcp_{name}_r"])


@pytest.mark.parametrize("name", ["gauss1000x40", "exactrank200x40r10", "spectral600x24"])
def test_cqrrpt_matches_reference_fixture(oracle, fx, meta, name):
    kw = meta[name]
    res = oracle.cqrrpt(fx[f"cq_{name}_in"], eps_tol=1e-4, **kw)
    k0, k = fx[f"cq_{name}_k"]
    assert (res.k0, res.k) == (k0, k)
    assert np.array_equal(res.pivots, fx[f"cq_{name}_piv"])
    assert np.array_equal(res.q, fx[f"cq_{name}_q"])  # bit-for-bit restatement
    assert np.array_equal(res.r, fx[f"cq_{name}_r"])
    assert res.cond_m_pre == float(fx[f"cq_{name}_cond"])


# ------------------------------------------------------------ live reference
def test_oracle_bitwise_equal_to_reference(oracle, reference):
    a = reference.gen_gaussian(700, 50, 11)
    assert np.array_equal(a, oracle.gen_gaussian(700, 50, 11))
    sig = 10.0 ** (-10 * np.arange(30) / 29)
    assert np.array_equal(reference.gen_spectral(300, 30, sig, 2), oracle.gen_spectral(300, 30, sig, 2))
    assert np.array_equal(reference.gen_exact_rank(200, 40, 10, 24), oracle.gen_exact_rank(200, 40, 10, 24))
    sk = reference.saso_apply(63, a, 8, 9)
    assert np.array_equal(sk, oracle.saso_apply(63, a, 8, 9))
    r1, p1, k1 = reference.qrcp(sk)
    r2, p2, k2 = oracle.qrcp(sk)
    assert k1 == k2 and np.array_equal(p1, p2) and np.array_equal(r1, r2)
    g = reference.gram(a)
    assert np.array_equal(g, oracle.gram(a))
    c1, f1 = reference.cholesky(g)
    c2, f2 = oracle.cholesky(g)
    assert f1 == f2 and np.array_equal(c1, c2)
    assert np.array_equal(reference.trsm_right(a, c1), oracle.trsm_right(a, c1))
    for meth in (0, 1, 2):
        assert reference.cond_estimate(c1, meth) == oracle.cond_estimate(c1, meth)
    x = reference.cqrrpt(a, gamma=1.25, nnz=8, seed=3)
    y = oracle.cqrrpt(a, gamma=1.25, nnz=8, seed=3)
    assert np.array_equal(x.q, y.q) and np.array_equal(x.r, y.r) and np.array_equal(x.pivots, y.pivots)
    assert (x.k0, x.k, x.cond_m_pre) == (y.k0, y.k, y.cond_m_pre)


def test_stage2_failure_paths_match_reference(oracle, reference):
    base = oracle.gen_gaussian(40, 8, 11)
    mk = np.zeros((40, 12)); mk[:, :8] = base; mk[:, 9:12] = base[:, :3]
    a = oracle.rank_stage2(mk, np.eye(12))
    b = reference.rank_stage2(mk, np.eye(12))
    assert (a["rank"], a["k0_final"], a["retries"]) == (b["rank"], b["k0_final"], b["retries"]) == (8, 8, 1)
    assert a["cond_at_rank"] == b["cond_at_rank"]


# ------------------------------------------------------------ known answers
def test_c1_golden_summary(oracle, meta):
    """reference C1 = gen_gaussian(16384, 256, 0), gamma 1.25, nnz 8."""
    c1 = meta["C1"]
    res = oracle.cqrrpt(oracle.gen_gaussian(16384, 256, 0), gamma=1.25, nnz=8, seed=0)
    assert fnv_pivots(res.pivots) == c1["jhash"] == "ac0e857417ac8f07"
    assert [int(v) for v in res.pivots[:8]] == c1["j8"]
    assert (res.k0, res.k) == (c1["k0"], c1["k"]) == (256, 256)
    assert res.r[0, 0] == c1["r00"]


def test_saso_structure(oracle):
    # test_sketch.cc:28-54: exactly nnz entries of +-1/sqrt(d) per column
    rows, vals = oracle.saso_sample(4, 10, 1, 123)
    assert np.all(np.abs(vals) == 0.5)
    rows, vals = oracle.saso_sample(12, 64, 4, 9)
    assert np.all(np.abs(vals) == 1.0 / np.sqrt(12.0))
    assert all(len(set(r)) == 4 for r in rows)
    with pytest.raises(ValueError):
        oracle.saso_sample(4, 10, 0, 1)
    with pytest.raises(ValueError):
        oracle.saso_sample(4, 10, 5, 1)


def test_apply_equals_densified(oracle):
    # test_sketch.cc:101-110
    m = oracle.gen_gaussian(30, 7, 21)
    rows, vals = oracle.saso_sample(11, 30, 3, 66)
    dense = np.zeros((11, 30))
    for c in range(30):
        dense[rows[c], c] = vals[c]
    assert np.max(np.abs(oracle.saso_apply(11, m, 3, 66) - dense @ m)) <= 1e-13 * np.linalg.norm(m)


def test_qrcp_known_answers(oracle):
    r, piv, k = oracle.qrcp(np.diag([1.0, 5.0, 3.0]))  # test_qrcp.cc:29-35
    assert list(piv) == [1, 2, 0] and np.allclose(np.abs(np.diag(r)), [5, 3, 1], rtol=1e-15)
    r, piv, k = oracle.qrcp(np.zeros((4, 3)))  # test_qrcp.cc:37-44
    assert k == 0 and list(piv) == [0, 1, 2] and r.shape == (0, 3)
    r, piv, k = oracle.qrcp(oracle.gen_kahan(16, 0.285))  # test_qrcp.cc:46-51
    assert k == 16 and list(piv) == list(range(16))
    m = oracle.gen_gaussian(50, 12, 8)  # test_qrcp.cc:73-81
    base = oracle.qrcp(m)[1]
    for c in (0.0034, 1024.0, -3.0):
        assert np.array_equal(oracle.qrcp(m * c)[1], base)


def test_stage1_known_answers(oracle):
    r = np.zeros((2, 2)); r[0, 0] = 1.0; r[1, 1] = 1e-20
    assert oracle.rank_stage1(r) == 1  # test_cqrrpt.cc:84-90
    assert oracle.rank_stage1(np.zeros((3, 5))) == 0
    t = [1.0, 1e-8, 1e-18, 1e-19, 0.0]
    r = np.zeros((4, 4))
    for i in range(4):
        r[i, i] = np.sqrt(t[i] ** 2 - t[i + 1] ** 2)
    assert oracle.rank_stage1(r) == 2  # test_cqrrpt.cc:92-110


def test_linalg_known_answers(oracle):
    r, fi = oracle.cholesky(np.diag([1.0, -1.0]))  # test_linalg.cc:92-100
    assert fi == 2 and r.shape == (1, 1) and r[0, 0] == 1.0
    b = oracle.gen_gaussian(20, 5, 1)
    assert np.array_equal(oracle.trsm_right(b, np.eye(5)), b)  # test_linalg.cc:134-138
    u = np.triu(np.ones((4, 4))); u[2, 2] = 0.0
    with pytest.raises(ZeroDivisionError):
        oracle.trsm_right(np.ones((5, 4)), u)  # test_linalg.cc:156-161
    g = oracle.gram(oracle.gen_gaussian(60, 9, 2))
    assert np.array_equal(g, g.T)  # test_linalg.cc:179-189


def test_cond_estimator_known_answers(oracle):
    for meth in (0, 1, 2):  # test_cqrrpt.cc:124-137
        v = oracle.cond_estimate(np.eye(5), meth)[0]
        assert 1.0 <= v <= 1.0 + 3e-6
    assert oracle.cond_estimate(np.diag([10.0, 1.0]), 0)[0] == 10.0
    assert np.isinf(oracle.cond_estimate(np.diag([5.0, 0.1]), 2)[0])  # test_cqrrpt.cc:150-156


def test_stage2_known_answers(oracle):
    # (retries, k0_final, rank) = (1,8,8), (1,6,6), (1,5,5)
    base = oracle.gen_gaussian(40, 8, 11)
    mk = np.zeros((40, 12)); mk[:, :8] = base; mk[:, 9:12] = base[:, :3]
    s = oracle.rank_stage2(mk, np.eye(12))
    assert (s["retries"], s["k0_final"], s["rank"]) == (1, 8, 8)
    base = oracle.gen_gaussian(50, 6, 12)
    mk = np.zeros((50, 9)); mk[:, :6] = base; mk[:, 6:9] = base[:, :3]
    s = oracle.rank_stage2(mk, np.eye(9))
    assert (s["retries"], s["k0_final"], s["rank"]) == (1, 6, 6)
    base = oracle.gen_gaussian(30, 5, 13)
    mk = np.zeros((30, 7)); mk[:, :5] = base; mk[:, 5:7] = base[:, :2]
    s = oracle.rank_stage2(mk, np.eye(7))
    assert (s["retries"], s["k0_final"], s["rank"]) == (1, 5, 5)


def test_cqrrpt_known_answers(oracle):
    assert oracle.sketch_rows_for(1.25, 50) == 63 and oracle.sketch_rows_for(3.0, 500) == 1500
    res = oracle.cqrrpt(np.zeros((30, 5)))  # test_cqrrpt.cc:262-268
    assert res.k == 0 and res.k0 == 0
    res = oracle.cqrrpt(oracle.gen_exact_rank(200, 40, 10, 24), seed=25)  # test_cqrrpt.cc:243-251
    assert res.k == 10
    with pytest.raises(ValueError):
        oracle.cqrrpt(oracle.gen_gaussian(20, 4, 29), gamma=0.5)
    with pytest.raises(ValueError):
        oracle.cqrrpt(oracle.gen_gaussian(20, 4, 29), eps_tol=U / 2)


def test_flop_model_known_answers(oracle):
    # test_cqrrpt.cc:315-346
    assert abs(oracle.flop_model(1000, 100, 100, 125) - 3.227e7) <= 3.227e4
    assert oracle.flop_model(500, 64, 0, 80, 77.0) == 77.0
    for (m, n, k, d) in [(1000, 100, 100, 125), (4096, 256, 256, 320), (512, 64, 17, 80), (77, 13, 9, 20)]:
        q6 = 24 * d * n * k - 12 * k * k * (d + n) + 8 * k ** 3
        t6 = 6 * m * k * k
        c6 = 6 * m * k * (k + 1) + 2 * k ** 3 + 3 * k * k + k + 6 * m * k * k
        assert oracle.flop_model(m, n, k, d, 5.0) == float(q6 + t6 + c6) / 6.0 + 5.0
    with pytest.raises(ValueError):
        oracle.flop_model(100, 10, 11, 20)


@pytest.mark.parametrize("twice", [False, True])
def test_cholesky_qr_composition_bit_exact(oracle, reference, twice):
    """The oracle's cholesky_qr(2) (restated gram/cholesky/trsm/trmm) is
    bit-identical to the reference's cqrrpt.cc:75-90, failure index included."""
    a = oracle.gen_gaussian(300, 24, 2)
    q1, r1, f1 = oracle.cholesky_qr(a, twice)
    q2, r2, f2 = reference.cholesky_qr(a, twice)
    assert f1 == f2 == 0 and np.array_equal(q1, q2) and np.array_equal(r1, r2)
    b = oracle.gen_gaussian(30, 7, 13)
    b[:, 5:7] = b[:, :2]
    assert oracle.cholesky_qr(b, twice)[2] == reference.cholesky_qr(b, twice)[2] == 6


def test_gaussian_operator_bit_exact_and_apply(oracle, reference):
    """The oracle's Gaussian operator equals the reference's bit for bit
    (apply on the identity returns S exactly); the product agrees to rounding."""
    d, m, seed = 17, 64, 9
    s_ref = reference.gaussian_sketch_apply(d, np.eye(m), seed)
    assert np.array_equal(oracle.gaussian_sample(d, m, seed), s_ref)
    a = oracle.gen_gaussian(2000, 40, 3)
    x, y = oracle.gaussian_apply(50, a, 7), reference.gaussian_sketch_apply(50, a, 7)
    assert np.max(np.abs(x - y)) <= 1e-13 * np.max(np.abs(y))


@pytest.mark.parametrize("m,n,d,seed", [(100, 7, 20, 3), (1000, 30, 40, 7), (4096, 16, 100, 1), (5000, 3, 5000, 2)])
def test_srft_restatement_bit_exact(oracle, reference, m, n, d, seed):
    """sketch.cc:100-119 (sample) and 147-166 (apply, fwht 31-39) restated in C."""
    a = oracle.gen_gaussian(m, n, seed)
    assert np.array_equal(oracle.srft_apply(d, a, seed), reference.srft_sketch_apply(d, a, seed))
