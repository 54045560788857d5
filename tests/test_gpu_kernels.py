"""GPU parity of each CUDA kernel against the CPU oracle (oracle/cqrrpt_oracle.c,
pinned bit-for-bit to the reference by tests/test_oracle.py).

Bars (stated per test): integer/index work bit-exact; FP64 work within the
tolerance the reference's own tests use for that function.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

U = 1.1102230246251565e-16


def dev(pkg, a):
    return pkg.to_device_colmajor(np.asfortranarray(a))


def host(t):
    return np.asfortranarray(t.cpu().numpy())


# ---------------------------------------------------------------- K1 plan
@pytest.mark.parametrize("d,m,nnz,seed,c0", [(320, 16384, 8, 0, 0), (12, 64, 4, 9, 0), (4, 10, 1, 123, 0),
                                             (5120, 3000, 8, 7, 123456), (63, 1000, 63, 5, 17)])
def test_saso_plan_bit_exact(cuda, oracle, d, m, nnz, seed, c0):
    from paper_2311_08316_b200 import kernels
    plan = kernels.saso_plan(d, m, nnz, seed, c0=c0).cpu().numpy().view(np.uint32)
    rows, vals = oracle.saso_sample(d, m, nnz, seed, c0=c0)
    assert np.array_equal((plan & 0x7FFFFFFF).astype(np.int64), rows)
    sign = (plan >> 31).astype(bool)
    val = 1.0 / np.sqrt(d)
    assert np.array_equal(np.where(sign, val, -val), vals)  # +-1/sqrt(d) exactly (test_sketch.cc:28-54)


# ---------------------------------------------------------------- K2 sketch
@pytest.mark.parametrize("m,n,d,nnz,seed", [(16384, 256, 320, 8, 0), (1000, 37, 50, 3, 4), (30, 7, 11, 3, 66),
                                            (4096, 64, 1280, 8, 1), (777, 100, 125, 4, 2)])
def test_saso_sketch_matches_apply(cuda, oracle, m, n, d, nnz, seed):
    from paper_2311_08316_b200 import kernels
    a = oracle.gen_gaussian(m, n, seed + 100)
    got = host(kernels.saso_sketch(dev(cuda, a), d, nnz, seed))
    ref = oracle.saso_apply(d, a, nnz, seed)
    # exact-order sketch: bit-identical to the reference's apply (sketch.cc:131-146)
    assert np.array_equal(got, ref)


def test_saso_sketch_row_blocks_and_lda(cuda, oracle):
    """Several sketch-row blocks per column group, ragged last column group and
    tile, and a leading dimension larger than m: still bit-identical."""
    import torch
    from paper_2311_08316_b200 import kernels
    m, n, d, nnz, seed = 20011, 70, 1500, 8, 3
    a = oracle.gen_gaussian(m, n, 9)
    big = torch.zeros((n, m + 5), dtype=torch.float64, device="cuda")
    big[:, :m] = torch.from_numpy(np.ascontiguousarray(a.T)).cuda()
    view = big.t()[:m, :]  # column-major, lda = m + 5
    got = host(kernels.saso_sketch(view, d, nnz, seed))
    assert np.array_equal(got, oracle.saso_apply(d, a, nnz, seed))


@pytest.mark.parametrize("m,n,d", [(70000, 64, 80), (40000, 256, 320)])
def test_saso_sketch_split_mode(cuda, oracle, m, n, d):
    """CQRRPT_GPU_FAST_SKETCH: c-split partials summed in a fixed order ->
    deterministic and within rounding of the reference's apply."""
    from paper_2311_08316_b200 import kernels
    a = oracle.gen_gaussian(m, n, 21)
    A = dev(cuda, a)
    x = host(kernels.saso_sketch(A, d, 8, 5, fast=True))
    y = host(kernels.saso_sketch(A, d, 8, 5, fast=True))
    assert np.array_equal(x, y)
    ref = oracle.saso_apply(d, a, 8, 5)
    scale = np.sqrt(m * 8.0 / d)  # |Msk(r,j)| ~ sqrt(entries per row) * |a|
    assert np.max(np.abs(x - ref)) <= 1e-14 * scale * np.max(np.abs(a)) * 10


def test_saso_sketch_row_offset_shards_sum(cuda, oracle):
    """Row-sharded sketch partials (global row offsets) sum to the full sketch."""
    from paper_2311_08316_b200 import kernels
    a = oracle.gen_gaussian(3000, 48, 5)
    full = host(kernels.saso_sketch(dev(cuda, a), 60, 8, 11))
    parts = [host(kernels.saso_sketch(dev(cuda, a[lo:hi]), 60, 8, 11, c0=lo))
             for lo, hi in [(0, 1000), (1000, 2200), (2200, 3000)]]
    assert np.max(np.abs(sum(parts) - full)) <= 1e-13 * np.linalg.norm(a)
    ref = oracle.saso_apply(60, a, 8, 11)
    assert np.max(np.abs(full - ref)) <= 1e-13 * np.linalg.norm(a)


def test_saso_sketch_deterministic(cuda, oracle):
    from paper_2311_08316_b200 import kernels
    a = dev(cuda, oracle.gen_gaussian(5000, 64, 3))
    x = host(kernels.saso_sketch(a, 80, 8, 1))
    y = host(kernels.saso_sketch(a, 80, 8, 1))
    assert np.array_equal(x, y)
    z = host(kernels.saso_sketch(a, 80, 8, 2))
    assert not np.array_equal(x, z)


@pytest.mark.parametrize("path", ["LDGSTS", "TMA"])
@pytest.mark.parametrize("A", [1, 2, 4, 6, 8, 12, 16])
def test_saso_sketch_every_row_block_width(cuda, oracle, monkeypatch, A, path):
    """Every instantiation of the apply kernel (A accumulator rows per consumer
    warp; LDGSTS or bulk-copy staging, forced by env var) against the
    reference's apply: several row blocks, ragged last 256-row tile (even and
    odd row counts: the bulk path loads an odd tail row by hand), ragged last
    column group, a padded leading dimension."""
    from paper_2311_08316_b200 import kernels
    monkeypatch.setenv("CQRRPT_SASO_A", str(A))
    monkeypatch.setenv("CQRRPT_SASO_" + path, "1")
    n, d, nnz, seed = 45, 700, 8, 12
    for m in (5000, 5001):
        a = oracle.gen_gaussian(m, n, 31)
        x = cuda.colmajor_empty(m, n, pad_to=2)  # even lda: eligible for bulk copies
        x.copy_(dev(cuda, a))
        got = host(kernels.saso_sketch(x, d, nnz, seed))
        assert np.array_equal(got, oracle.saso_apply(d, a, nnz, seed)), m


@pytest.mark.parametrize("W", [8, 16])
@pytest.mark.parametrize("A", [1, 2, 4, 8, 12, 16])
def test_saso_sketch_narrow_column_groups(cuda, oracle, monkeypatch, A, W):
    """Narrow column groups (W columns per CTA, 32 / W row slots per consumer
    warp whose entry walks diverge; chosen by default for n <= 512) against
    the reference's apply, bit for bit: several row blocks, ragged last tile
    and last column group, padded leading dimension, an offset shard, and the
    chained launches of the chunked host path."""
    from paper_2311_08316_b200 import kernels
    monkeypatch.setenv("CQRRPT_SASO_A", str(A))
    monkeypatch.setenv("CQRRPT_SASO_W", str(W))
    n, d, nnz, seed = 45, 700, 8, 12
    for m in (5000, 5001):
        a = oracle.gen_gaussian(m, n, 31)
        x = cuda.colmajor_empty(m, n, pad_to=2)
        x.copy_(dev(cuda, a))
        got = host(kernels.saso_sketch(x, d, nnz, seed))
        assert np.array_equal(got, oracle.saso_apply(d, a, nnz, seed)), m
    # few sketch rows (one partial row block), nnz = 2
    a = oracle.gen_gaussian(3000, 19, 5)
    got = host(kernels.saso_sketch(dev(cuda, a), 24, 2, 3))
    assert np.array_equal(got, oracle.saso_apply(24, a, 2, 3))


def test_saso_sketch_narrow_default_choice(cuda, oracle):
    """The default choice at a C5-256-like shape (n <= 512: narrow column
    groups) is bit-identical to the reference's apply."""
    from paper_2311_08316_b200 import kernels
    m, n, d = 40000, 256, 320
    a = oracle.gen_gaussian(m, n, 9)
    got = host(kernels.saso_sketch(dev(cuda, a), d, 8, 0))
    assert np.array_equal(got, oracle.saso_apply(d, a, 8, 0))


@pytest.mark.parametrize("nnz", [1, 2, 16])
def test_saso_sketch_nnz(cuda, oracle, nnz):
    """Other nonzeros per column (entry-list sizes per tile), bit-identical."""
    from paper_2311_08316_b200 import kernels
    m, n, d = 3000, 40, 120
    a = oracle.gen_gaussian(m, n, 7)
    got = host(kernels.saso_sketch(dev(cuda, a), d, nnz, 17))
    assert np.array_equal(got, oracle.saso_apply(d, a, nnz, 17))


def test_saso_sketch_zero(cuda, oracle):
    from paper_2311_08316_b200 import kernels
    got = host(kernels.saso_sketch(dev(cuda, np.zeros((20, 4))), 8, 2, 44))
    assert np.all(got == 0.0)


# ---------------------------------------------------------------- K3 QRCP
def _qrcp_compare(cuda, oracle, a):
    """The device QRCP restates qrcp_maxnorm's arithmetic order: R, J, k are
    bit-identical to the reference on the same input (even at exact ties)."""
    from paper_2311_08316_b200 import kernels
    R_ref, J_ref, k_ref = oracle.qrcp(a)
    R, J, k = kernels.qrcp(dev(cuda, a))
    R, J = host(R), J.cpu().numpy()
    assert k == k_ref
    assert np.array_equal(J, J_ref)
    assert np.array_equal(R, R_ref)
    return R, J, k


@pytest.mark.parametrize("rows,n,seed", [(80, 64, 3), (320, 256, 1), (1000, 700, 2)])
def test_qrcp_general_column_phase_bit_exact(cuda, oracle, monkeypatch, rows, n, seed):
    """The general column phase (used when a CTA owns more than 8 columns in a
    step or a column does not fit one warp buffer) against the reference,
    forced by env var."""
    monkeypatch.setenv("CQRRPT_QRCP_GENERAL", "1")
    _qrcp_compare(cuda, oracle, oracle.gen_gaussian(rows, n, seed))


@pytest.mark.parametrize("rows,n,seed", [(320, 256, 5), (100, 90, 6), (300, 40, 7)])
@pytest.mark.parametrize("cluster", [True, False])
def test_qrcp_cluster_and_grid_paths(cuda, oracle, monkeypatch, rows, n, seed, cluster):
    """n <= 256: the whole factorization runs in one thread-block cluster
    (K3b); CQRRPT_QRCP_NOCLUSTER forces the grid kernel. Both bit-identical."""
    if not cluster:
        monkeypatch.setenv("CQRRPT_QRCP_NOCLUSTER", "1")
    _qrcp_compare(cuda, oracle, oracle.gen_gaussian(rows, n, seed))


def test_qrcp_cluster_rank_deficient_stop(cuda, oracle):
    """Rank stop inside the cluster kernel: exact rank 9 of 64 columns."""
    rng = np.random.default_rng(3)
    a = rng.standard_normal((200, 9)) @ rng.standard_normal((9, 64))
    R, J, k = _qrcp_compare(cuda, oracle, np.asfortranarray(a))
    assert k < 64


def test_qrcp_known_answer_diag(cuda, oracle):
    # test_qrcp.cc:29-35: diag(1,5,3) -> pivots {1,2,0}, |R_ii| = (5,3,1)
    R, J, k = _qrcp_compare(cuda, oracle, np.diag([1.0, 5.0, 3.0]))
    assert list(J) == [1, 2, 0] and k == 3
    assert np.allclose(np.abs(np.diag(R)), [5, 3, 1], rtol=1e-15)


def test_qrcp_zero_matrix(cuda, oracle):
    # test_qrcp.cc:37-44: zero -> rank 0, identity pivots, R 0 x n
    from paper_2311_08316_b200 import kernels
    R, J, k = kernels.qrcp(dev(cuda, np.zeros((4, 3))))
    assert k == 0 and list(J.cpu().numpy()) == [0, 1, 2] and R.shape == (0, 3)


def test_qrcp_kahan_identity_pivots(cuda, oracle):
    # test_qrcp.cc:46-51
    R, J, k = _qrcp_compare(cuda, oracle, oracle.gen_kahan(16, 0.285))
    assert k == 16 and list(J) == list(range(16))


@pytest.mark.parametrize("rows,n,seed", [(320, 256, 0), (60, 15, 900), (1280, 1024, 3), (80, 64, 8), (200, 200, 4)])
def test_qrcp_gaussian(cuda, oracle, rows, n, seed):
    a = oracle.gen_gaussian(rows, n, seed)
    _qrcp_compare(cuda, oracle, a)


def test_qrcp_graded_columns(cuda, oracle):
    # cond-1e10 spectrum (test_qrcp.cc:83-91 style) exercises the recompute safeguard
    sig = 10.0 ** (-10 * np.arange(64) / 63)
    a = oracle.gen_spectral(300, 64, sig, 7)
    R, J, k = _qrcp_compare(cuda, oracle, a)
    d = np.abs(np.diag(R[:, :k]))
    assert np.all(d[1:] <= d[:-1] * (1 + 1e-12))


def test_qrcp_scale_invariant(cuda, oracle):
    # test_qrcp.cc:73-81
    from paper_2311_08316_b200 import kernels
    a = oracle.gen_gaussian(50, 12, 8)
    base = kernels.qrcp(dev(cuda, a))[1].cpu().numpy()
    for c in (0.0034, 1024.0, -3.0):
        assert np.array_equal(kernels.qrcp(dev(cuda, a * c))[1].cpu().numpy(), base)


# ---------------------------------------------------------------- K4 stage 1
def test_rank_stage1_known_answers(cuda, oracle):
    from paper_2311_08316_b200 import kernels
    r = np.zeros((2, 2)); r[0, 0] = 1.0; r[1, 1] = 1e-20
    assert kernels.rank_stage1(dev(cuda, r)) == 1  # test_cqrrpt.cc:84-90
    assert kernels.rank_stage1(dev(cuda, np.zeros((3, 5)))) == 0
    t = [1.0, 1e-8, 1e-18, 1e-19, 0.0]
    r = np.zeros((4, 4))
    for i in range(4):
        r[i, i] = np.sqrt(t[i] ** 2 - t[i + 1] ** 2)
    assert kernels.rank_stage1(dev(cuda, r)) == 2  # test_cqrrpt.cc:92-110
    R_ref, _, _ = oracle.qrcp(oracle.gen_gaussian(40, 12, 7))
    assert kernels.rank_stage1(dev(cuda, R_ref)) == oracle.rank_stage1(R_ref)


# ---------------------------------------------------------------- K5 TRSM
@pytest.mark.parametrize("m,k", [(16384, 256), (1000, 100), (513, 64), (300, 65), (129, 1), (2000, 200)])
def test_trsm_right_matches_oracle(cuda, oracle, m, k):
    from paper_2311_08316_b200 import kernels
    b = oracle.gen_gaussian(m, k + 5, 3)
    Rq, _, _ = oracle.qrcp(oracle.gen_gaussian(int(1.25 * k) + 1, k, 4))
    u = Rq[:k, :k]
    cols = np.random.default_rng(0).permutation(k + 5)[:k].astype(np.int64)
    import torch
    x = host(kernels.trsm_right(dev(cuda, b), dev(cuda, u), cols=torch.as_tensor(cols, device="cuda")))
    ref = oracle.trsm_right(np.asfortranarray(b[:, cols]), u)
    # backward-stable solves: compare columnwise relative to ||ref col||
    err = np.linalg.norm(x - ref, axis=0) / np.linalg.norm(ref, axis=0)
    assert np.max(err) <= 1e3 * k * U
    # residual ||X U - B|| tiny
    assert np.linalg.norm(x @ u - b[:, cols]) <= 1e-12 * np.linalg.norm(b[:, cols])


def test_trsm_identity_exact(cuda, oracle):
    # test_linalg.cc:134-138: solve by the identity reproduces B
    from paper_2311_08316_b200 import kernels
    b = oracle.gen_gaussian(200, 70, 1)
    x = host(kernels.trsm_right(dev(cuda, b), dev(cuda, np.eye(70))))
    assert np.array_equal(x, b)


def test_trsm_singular_raises(cuda):
    # test_linalg.cc:156-161: zero diagonal -> domain_error
    from paper_2311_08316_b200 import kernels, DomainError
    u = np.triu(np.ones((4, 4))); u[2, 2] = 0.0
    with pytest.raises(DomainError):
        kernels.trsm_right(dev(cuda, np.ones((5, 4))), dev(cuda, u))


# ---------------------------------------------------------------- K5b Gram
@pytest.mark.parametrize("m,k", [(16384, 256), (300, 65), (1000, 1), (50000, 128), (64, 200)])
def test_gram_matches_oracle_and_is_symmetric(cuda, oracle, m, k):
    from paper_2311_08316_b200 import kernels
    a = oracle.gen_gaussian(m, k, 2)
    g = host(kernels.gram(dev(cuda, a)))
    ref = oracle.gram(a)
    assert np.array_equal(g, g.T)  # bitwise symmetric (test_linalg.cc:179-189)
    scale = np.sqrt(np.outer(np.diag(ref), np.diag(ref)))
    assert np.max(np.abs(g - ref) / scale) <= 1e2 * np.sqrt(m) * U


def test_gram_leading_block_property(cuda, oracle):
    """Leading j x j block of gram(X) == gram(X[:, :j]) bitwise (cqrrpt.cc:162-164)."""
    from paper_2311_08316_b200 import kernels
    a = dev(cuda, oracle.gen_gaussian(3000, 150, 9))
    g = host(kernels.gram(a))
    g2 = host(kernels.gram(a[:, :97]))
    assert np.array_equal(g[:97, :97], g2)


# ---------------------------------------------------------------- K6 potrf
def test_potrf_failure_index(cuda, oracle):
    # test_linalg.cc:92-100: G = diag(1, -1) -> failure index 2, leading 1x1 factor
    from paper_2311_08316_b200 import kernels
    r, fi = kernels.potrf(dev(cuda, np.diag([1.0, -1.0])))
    assert fi == 2 and host(r).shape == (1, 1) and host(r)[0, 0] == 1.0


@pytest.mark.parametrize("k", [1, 63, 64, 65, 200, 1024])
def test_potrf_matches_oracle(cuda, oracle, k):
    from paper_2311_08316_b200 import kernels
    a = oracle.gen_gaussian(3 * k + 10, k, 5)
    g = oracle.gram(a)
    r, fi = kernels.potrf(dev(cuda, g))
    ref, fref = oracle.cholesky(g)
    assert fi == fref == 0
    r = host(r)
    assert np.all(np.tril(r, -1) == 0)
    err = np.linalg.norm(r - ref, axis=0) / np.linalg.norm(ref, axis=0)
    assert np.max(err) <= 1e3 * k * U


def test_potrf_failure_inside_block(cuda, oracle):
    from paper_2311_08316_b200 import kernels
    base = oracle.gen_gaussian(400, 100, 11)
    m = base.copy(); m[:, 80] = 0.0  # zero column -> minor 81 singular
    g = oracle.gram(m)
    r, fi = kernels.potrf(dev(cuda, g))
    ref, fref = oracle.cholesky(g)
    assert fi == fref == 81
    assert np.allclose(host(r), ref, rtol=1e-10, atol=1e-10 * np.abs(ref).max())


@pytest.mark.parametrize("k", [1, 37, 64, 65, 128, 200, 256, 1000, 1030])
def test_trtri_upper_inverse(cuda, oracle, k):
    # log-depth inverse (diagonal blocks + batched GEMM levels, ragged last pair)
    from paper_2311_08316_b200 import kernels
    a = oracle.gen_gaussian(3 * k + 10, k, 6)
    r, fi = oracle.cholesky(oracle.gram(a))
    assert fi == 0
    x = host(kernels.trtri_upper(dev(cuda, r)))
    assert np.all(np.tril(x, -1) == 0)
    cond = np.linalg.cond(r)
    assert np.linalg.norm(x @ r - np.eye(k)) <= 1e2 * k * U * cond
    # leading blocks of the inverse are the inverses of the leading blocks
    ell = max(1, k // 3)
    xl = host(kernels.trtri_upper(dev(cuda, np.ascontiguousarray(r[:ell, :ell]))))
    assert np.allclose(xl, x[:ell, :ell], rtol=0, atol=1e2 * ell * U * np.abs(x).max() * cond)


# ---------------------------------------------------------------- K7 cond
def test_cond_estimates_match_oracle(cuda, oracle):
    from paper_2311_08316_b200 import kernels
    eye = np.eye(5)
    for meth in (0, 1, 2):
        v = kernels.cond_estimate(dev(cuda, eye), meth)
        assert 1.0 <= v <= 1.0 + 3e-6  # test_cqrrpt.cc:124-131
    d = np.diag([10.0, 1.0])
    assert kernels.cond_estimate(dev(cuda, d), 0) == 10.0
    x = np.diag([5.0, 0.1])
    assert kernels.cond_estimate(dev(cuda, x), 2) == pytest.approx(oracle.cond_estimate(x, 2)[0], rel=1e-9)
    R, _, _ = oracle.qrcp(oracle.gen_gaussian(80, 64, 8))
    for meth in (0, 1, 2):
        assert kernels.cond_estimate(dev(cuda, R), meth) == pytest.approx(oracle.cond_estimate(R, meth)[0], rel=1e-6)


@pytest.mark.parametrize("n,meth", [(300, 1), (300, 2), (300, 3), (700, 1), (700, 2)])
def test_cond_estimates_grid_path(cuda, oracle, n, meth):
    """ell >= 256 runs the grid-wide power iterations (cond_grid_kernel):
    same iterations and stopping rule as the reference, different summation
    order -> converged estimates agree to ~1e-9."""
    from paper_2311_08316_b200 import kernels
    R, _, _ = oracle.qrcp(oracle.gen_gaussian(n + 40, n, 8))
    if meth == 3:  # the nested estimator's identity-deviation leg on a near-orthogonal R (tau < 1)
        q = np.linalg.qr(oracle.gen_gaussian(n, n, 3))[0]
        R = np.triu(np.eye(n) + 1e-3 * np.triu(q))
        ref = oracle.cond_estimate(R, 2)[0]
    else:
        ref = oracle.cond_estimate(R, meth)[0]
    got = kernels.cond_estimate(dev(cuda, R), meth)
    assert got == pytest.approx(ref, rel=1e-6)


# ---------------------------------------------------------------- K9 TRMM
@pytest.mark.parametrize("k,n", [(10, 13), (256, 256), (100, 300), (65, 65)])
def test_trmm_upper(cuda, oracle, k, n):
    from paper_2311_08316_b200 import kernels
    a = np.triu(oracle.gen_gaussian(k, k, 1))
    b = np.triu(oracle.gen_gaussian(k, n, 2))
    c = host(kernels.trmm_upper(dev(cuda, a), dev(cuda, b)))
    ref = oracle.multiply_upper_triangular(a, b)
    assert np.all(np.tril(c, -1) == 0.0)  # exactly upper-trapezoidal
    assert np.max(np.abs(c - ref)) <= 1e2 * k * U * np.max(np.abs(ref))
