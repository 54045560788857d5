"""End-to-end GPU parity of cqrrpt() against the reference (through the C ABI).

North-star bars (BASELINE.json):
  * J and k exactly equal wherever the sketch's pivot decisions are not within
    rounding of a tie (ties located with the oracle's tie-gap instrumentation);
  * ||M[:,J] - QR||_F/||M||_F and ||Q^T Q - I||_F within 10x of the reference's;
  * R within a relative tolerance scaled by cond(M): column-wise
    ||dR[:,j]|| <= 1e3 * n * u * cond_est * ||R[:,j]||.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

U = 1.1102230246251565e-16


def run_gpu(pkg, a, gamma=1.25, nnz=8, seed=0, eps_tol=1e-4, exact=False):
    A = pkg.to_device_colmajor(np.asfortranarray(a))
    res = pkg.dgeqpt(A, d_factor=gamma, nnz=nnz, seed=seed, eps_tol=eps_tol, exact_stage2=exact)
    q = np.asfortranarray(A[:, : res.k].cpu().numpy())
    r = np.asfortranarray(res.r.cpu().numpy())
    return q, r, res.pivots.cpu().numpy(), res.k, res.k0, res


def metrics(oracle, a, q, r, piv):
    v = oracle.validate(a, q, r, piv)
    return v["orth_fro"], v["recon_rel"]


def tie_free_prefix(oracle, a, gamma, nnz, seed):
    """Length of the pivot prefix whose sketch QRCP decisions are not near-ties."""
    ref = oracle.cqrrpt(a, gamma=gamma, nnz=nnz, seed=seed, want_sketch=True)
    _, _, _, gaps = oracle.qrcp(ref.extra["m_sk"], gaps=True)
    n = a.shape[1]
    tie = np.nonzero(gaps <= 1e3 * U * n)[0]
    return (int(tie[0]) if tie.size else n), ref


def check_against_reference(pkg, oracle, a, gamma=1.25, nnz=8, seed=0, cond=1.0):
    q, r, piv, k, k0, res = run_gpu(pkg, a, gamma, nnz, seed)
    ref = oracle.cqrrpt(a, gamma=gamma, nnz=nnz, seed=seed)
    n = a.shape[1]
    # sketch + QRCP + stage 1 restate the reference's arithmetic: J, k0 bit-exact
    assert np.array_equal(piv, ref.pivots)
    assert k0 == ref.k0 and k == ref.k
    of, rr = metrics(oracle, a, q, r, piv)
    of_ref, rr_ref = metrics(oracle, a, ref.q, ref.r, ref.pivots)
    floor = 10 * n * U  # both can sit at the unit-roundoff floor
    assert of <= 10 * max(of_ref, floor), (of, of_ref)
    assert rr <= 10 * max(rr_ref, floor), (rr, rr_ref)
    err = np.linalg.norm(r - ref.r, axis=0) / (np.linalg.norm(ref.r, axis=0) + 1e-300)
    assert np.max(err) <= 1e3 * n * U * cond
    return res, ref


def test_c1_shape_matches_reference(cuda, oracle):
    a = oracle.gen_gaussian(16384, 256, 0)  # BASELINE config 1 (exact generator)
    res, ref = check_against_reference(cuda, oracle, a)
    assert res.k == 256 and res.k0 == 256
    # SURVEY §9 P11 golden summary of the reference for C1
    from oracle.oracle import fnv_pivots
    assert fnv_pivots(res.pivots.cpu().numpy()) == "ac0e857417ac8f07"
    assert list(res.pivots.cpu().numpy()[:8]) == [170, 80, 191, 79, 65, 38, 11, 243]


@pytest.mark.parametrize("gamma", [1.0, 1.25, 2.0])
def test_c5_style_graded_columns(cuda, oracle, gamma):
    a = oracle.gen_gaussian(20000, 128, 0)
    a, _ = oracle.c5_scale_columns(a, span=8.0, seed=0)
    check_against_reference(cuda, oracle, a, gamma=gamma, cond=1e8)


def test_cond1e10_spectrum(cuda, oracle):
    sig = 10.0 ** (-10 * np.arange(128) / 127)  # C2 spectrum at desk scale
    a = oracle.gen_spectral(8192, 128, sig, 0)
    check_against_reference(cuda, oracle, a, cond=1e10)


@pytest.mark.parametrize("noise,expect_k", [(1e-14, None), (1e-12, None), (0.0, 64)])
def test_planted_rank_detection(cuda, oracle, noise, expect_k):
    ab = oracle.gen_exact_rank(8192, 128, 64, 0)  # C3 structure at desk scale
    g = oracle.gen_gaussian(8192, 128, 1)
    a = np.asfortranarray(ab + noise * np.linalg.norm(ab) / np.sqrt(ab.size) * g)
    q, r, piv, k, k0, res = run_gpu(cuda, a)
    ref = oracle.cqrrpt(a, gamma=1.25, nnz=8, seed=0)
    assert k == ref.k and k0 == ref.k0
    assert np.array_equal(piv, ref.pivots)
    if expect_k is not None:
        assert k == expect_k


def test_exact_rank_known_answer(cuda, oracle):
    # test_cqrrpt.cc:243-251: gen_exact_rank(200, 40, 10, 24), seed 25 (nnz default 4) -> k = 10
    a = oracle.gen_exact_rank(200, 40, 10, 24)
    q, r, piv, k, k0, res = run_gpu(cuda, a, nnz=4, seed=25)
    assert k == 10
    v = oracle.validate(a, q, r, piv)
    assert v["recon_rel"] <= 1e-12


def test_zero_matrix_rank_zero(cuda, oracle):
    # test_cqrrpt.cc:262-268
    out = cuda.cqrrpt(np.zeros((30, 5)), cuda.CqrrptConfig())
    assert out.k == 0 and out.k0 == 0
    assert out.factorization.q.shape == (30, 0) and out.factorization.r.shape[0] == 0


def test_scaled_coordinate_columns(cuda, oracle):
    # test_cqrrpt.cc:223-241 (SASO instead of the Gaussian family): |R| = c I
    c = 3.5
    m = np.zeros((40, 8)); m[np.arange(8), np.arange(8)] = c
    out = cuda.cqrrpt(m, cuda.CqrrptConfig(gamma=2.0, seed=23, nnz_per_col=4))
    assert out.k == 8
    r = out.factorization.r
    assert np.all(np.abs(np.abs(np.diag(r)) - c) <= c * 1e-12)
    assert np.all(np.abs(np.triu(r, 1)) <= c * 1e-12)


def test_driver_defaults_and_config_errors(cuda, oracle):
    # test_cqrrpt.cc:253-260, 348-356
    assert cuda.sketch_rows_for(1.25, 50) == 63 and cuda.sketch_rows_for(3.0, 500) == 1500
    m = oracle.gen_gaussian(20, 4, 29)
    with pytest.raises(ValueError):
        cuda.cqrrpt(m, cuda.CqrrptConfig(gamma=0.5))
    with pytest.raises(ValueError):
        cuda.cqrrpt(m, cuda.CqrrptConfig(eps_tol=U / 2))
    with pytest.raises(ValueError):
        cuda.cqrrpt(m, cuda.CqrrptConfig(nnz_per_col=0))


def test_bitwise_deterministic(cuda, oracle):
    # test_cqrrpt.cc:270-283
    a = oracle.gen_gaussian(150, 20, 26)
    x = cuda.cqrrpt(a, cuda.CqrrptConfig(seed=27))
    y = cuda.cqrrpt(a, cuda.CqrrptConfig(seed=27))
    assert np.array_equal(x.factorization.q, y.factorization.q)
    assert np.array_equal(x.factorization.r, y.factorization.r)
    assert np.array_equal(x.factorization.pivots, y.factorization.pivots)
    z = cuda.cqrrpt(a, cuda.CqrrptConfig(seed=28))
    assert not np.array_equal(x.factorization.r, z.factorization.r)


@pytest.mark.parametrize("seed", range(6))
def test_valid_output_small(cuda, oracle, seed):
    # test_cqrrpt.cc:285-300 (SASO): valid at 100 n u, k = n
    n = 6 + 2 * seed
    a = oracle.gen_gaussian(40 * (1 + seed % 3) + 20, n, 400 + seed)
    out = cuda.cqrrpt(a, cuda.CqrrptConfig(gamma=2.0, nnz_per_col=4, seed=500 + seed))
    assert out.k == n
    v = cuda.validate(out.factorization, a, 100.0 * n * U)
    assert v.passed, v


def test_stage2_exact_vs_fast_path_agree(cuda, oracle):
    a = oracle.gen_gaussian(4000, 96, 3)
    _, _, p1, k1, _, r1 = run_gpu(cuda, a, exact=False)
    _, _, p2, k2, _, r2 = run_gpu(cuda, a, exact=True)
    assert k1 == k2 and np.array_equal(p1, p2)
    assert r2.ctx.stage2_exact == 1 and r1.ctx.stage2_exact == 0
    ref = oracle.cqrrpt(a, gamma=1.25, nnz=8, seed=0)
    assert r2.ctx.cond_m_pre == pytest.approx(ref.cond_m_pre, rel=1e-6)


def _failure_input(oracle, case):
    if case == "zero_col":
        base = oracle.gen_gaussian(40, 8, 11)
        mk = np.zeros((40, 12)); mk[:, :8] = base; mk[:, 9:12] = base[:, :3]
        return mk, (1, 8, 8)
    if case == "dups":
        base = oracle.gen_gaussian(50, 6, 12)
        mk = np.zeros((50, 9)); mk[:, :6] = base; mk[:, 6:9] = base[:, :3]
        return mk, (1, 6, 6)
    base = oracle.gen_gaussian(30, 5, 13)
    mk = np.zeros((30, 7)); mk[:, :5] = base; mk[:, 5:7] = base[:, :2]
    return mk, (1, 5, 5)


@pytest.mark.parametrize("case", ["zero_col", "dups", "dups_small"])
def test_stage2_cholesky_failure_paths(cuda, oracle, case):
    """The driver's own stage-2 routine (cqrrpt_gpu_rank_stage2) on the
    reference's failure inputs (test_cqrrpt.cc:170-197,302-313; SURVEY P10:
    (retries, k0_final, rank) = (1,8,8), (1,6,6), (1,5,5))."""
    from paper_2311_08316_b200 import kernels
    mk, want = _failure_input(oracle, case)
    ref = oracle.rank_stage2(mk, np.eye(mk.shape[1]))
    assert (ref["retries"], ref["k0_final"], ref["rank"]) == want
    for exact in (False, True):
        got = kernels.rank_stage2(cuda.to_device_colmajor(mk), cuda.to_device_colmajor(np.eye(mk.shape[1])),
                                  exact=exact)
        assert (got["retries"], got["k0_final"], got["rank"]) == want
        assert got["cond_at_rank"] == pytest.approx(ref["cond_at_rank"], rel=1e-6)
        k = got["rank"]
        np.testing.assert_allclose(got["r_pre"].cpu().numpy(), ref["r_pre"], rtol=0, atol=1e3 * k * U *
                                   np.abs(ref["r_pre"]).max())


@pytest.mark.parametrize("decades,eps_tol", [(6.0, 1e-4), (9.0, 1e-8), (12.0, 1e-4), (4.0, 1e-12)])
def test_stage2_truncation_vs_oracle(cuda, oracle, decades, eps_tol):
    """rank_stage2 on an unpreconditioned block (A_sk = I) whose leading
    blocks cross sqrt(eps_tol/u): the binary search truncates (and at 1e12 the
    Cholesky fails first). rank, k0_final, retries equal the reference
    restatement's; cond_at_rank within the estimator's rounding."""
    from paper_2311_08316_b200 import kernels
    n = 48
    mk = oracle.gen_spectral(2000, n, 10.0 ** (-decades * np.arange(n) / (n - 1)), 5)
    ref = oracle.rank_stage2(mk, np.eye(n), eps_tol=eps_tol)
    assert ref["rank"] < n  # a truncating input
    for exact in (False, True):
        got = kernels.rank_stage2(cuda.to_device_colmajor(mk), cuda.to_device_colmajor(np.eye(n)),
                                  eps_tol=eps_tol, exact=exact)
        assert (got["retries"], got["k0_final"], got["rank"]) == (ref["retries"], ref["k0_final"], ref["rank"])
        assert got["cond_at_rank"] == pytest.approx(ref["cond_at_rank"], rel=1e-4)


def _coherent(oracle, seed, n):
    """Leverage concentrated in n rows with a 1e-12 graded diagonal: with
    nnz = 1 the SASO sketch folds those rows together, the preconditioner is
    poor, and the driver's Gram hits a non-positive pivot (retry) before the
    binary search truncates."""
    a = np.zeros((400, n), order="F")
    a[:n, :n] = np.diag(10.0 ** (-np.linspace(0, 12, n)))
    a += 1e-13 * oracle.gen_gaussian(400, n, seed)
    return np.asfortranarray(a)


def _assert_cholesky_failure_tie(cuda, oracle, a, ref, k0f_gpu):
    """The Cholesky-failure point of rank_stage2 (cqrrpt.cc:168-186) is a
    rounding decision when the pivot there is at the Gram's rounding level:
    the two Grams (reference dot order vs DMMA tiles) differ by ~u ||M_pre||^2,
    so a pivot d_j with |d_j| / max_i G_ii <= 1e3 u k0 may come out either sign.
    Where the GPU's and the reference's k0_final differ, the factorization
    that got further must have such a pivot at the other's failure index."""
    from paper_2311_08316_b200 import kernels
    k0 = ref.k0
    mk = np.asfortranarray(a[:, ref.pivots[:k0]])
    ask = np.asfortranarray(ref.extra["r_sk"][:k0, :k0])
    bar = 1e3 * U * k0
    if k0f_gpu < ref.extra["k0_final"]:  # the reference passed the GPU's failing minor
        g = oracle.gram(oracle.trsm_right(mk, ask))
        r, _ = oracle.cholesky(g)
        j = k0f_gpu
    else:  # the GPU passed the reference's failing minor
        g = kernels.gram(kernels.trsm_right(cuda.to_device_colmajor(mk), cuda.to_device_colmajor(ask)))
        gd = g.cpu().numpy()
        r, _ = kernels.potrf(g)
        r = r.cpu().numpy()
        g = gd
        j = ref.extra["k0_final"]
    rel = r[j, j] ** 2 / np.max(np.diag(g))
    assert rel <= bar, (k0f_gpu, ref.extra["k0_final"], rel, bar)


@pytest.mark.parametrize("kind,seed,n,gamma,nnz,eps_tol", [
    ("coherent", 1, 32, 1.0, 1, 1e-4), ("coherent", 3, 32, 1.0, 1, 1e-4), ("coherent", 5, 16, 1.0, 1, 1e-4),
    ("coherent", 5, 32, 1.0, 2, 1e-4),
    ("gauss", 2, 64, 1.0, 8, 1e-13), ("gauss", 2, 64, 1.25, 8, 1e-14), ("c5", 1, 64, 1.0, 8, 1e-14)])
def test_stage2_decisions_through_driver(cuda, oracle, kind, seed, n, gamma, nnz, eps_tol):
    """Stage-2 decision paths through cqrrpt_gpu_dgeqpt compared with the
    reference restatement's cqrrpt (cqrrpt.cc:160-207): Cholesky-failure
    shrink + retry (coherent inputs) and cond-search truncation k < k0 (tight
    eps_tol), on both the fast-accept and the forced-search paths."""
    if kind == "coherent":
        a = _coherent(oracle, seed, n)
    elif kind == "gauss":
        a = oracle.gen_gaussian(3000, n, seed)
    else:
        a, _ = oracle.c5_scale_columns(oracle.gen_gaussian(4000, n, seed), 8.0, 0)
    ref = oracle.cqrrpt(a, gamma=gamma, nnz=nnz, eps_tol=eps_tol, seed=seed, want_sketch=True)
    assert ref.k < ref.k0 or ref.extra["retries"] > 0
    for exact in (False, True):
        A = cuda.to_device_colmajor(a)
        res = cuda.dgeqpt(A, d_factor=gamma, nnz=nnz, seed=seed, eps_tol=eps_tol, exact_stage2=exact,
                          diagnostics=True)
        assert (res.k0, res.k) == (ref.k0, ref.k)
        assert res.ctx.retries == ref.extra["retries"]
        if res.ctx.k0_final != ref.extra["k0_final"]:
            _assert_cholesky_failure_tie(cuda, oracle, a, ref, res.ctx.k0_final)
        assert np.array_equal(res.pivots.cpu().numpy(), ref.pivots)
        assert res.ctx.cond_m_pre == pytest.approx(ref.cond_m_pre, rel=1e-4)
        if ref.k:
            q = A[:, : res.k].cpu().numpy()
            v = oracle.validate(a, q, res.r.cpu().numpy(), ref.pivots)
            vr = oracle.validate(a, ref.q, ref.r, ref.pivots)
            assert v["orth_fro"] <= 10 * max(vr["orth_fro"], 10 * n * U)
            assert v["recon_rel"] <= 10 * max(vr["recon_rel"], 10 * n * U)


def test_cond_m_pre_fast_path(cuda, oracle):
    """cond_m_pre on the default (fast-accept) path: NaN unless diagnostics
    are requested, then est.at(k) exactly as the search would report it
    (cqrrpt.cc:205,298)."""
    a = oracle.gen_gaussian(4000, 96, 4)
    ref = oracle.cqrrpt(a, gamma=1.25, nnz=8, seed=0)
    r0 = cuda.dgeqpt(cuda.to_device_colmajor(a), d_factor=1.25, nnz=8, seed=0)
    assert r0.ctx.stage2_exact == 0 and np.isnan(r0.ctx.cond_m_pre)
    r1 = cuda.dgeqpt(cuda.to_device_colmajor(a), d_factor=1.25, nnz=8, seed=0, diagnostics=True)
    r2 = cuda.dgeqpt(cuda.to_device_colmajor(a), d_factor=1.25, nnz=8, seed=0, exact_stage2=True)
    assert r1.ctx.stage2_exact == 0 and r2.ctx.stage2_exact == 1
    assert r1.ctx.cond_m_pre == r2.ctx.cond_m_pre
    assert r1.ctx.cond_m_pre == pytest.approx(ref.cond_m_pre, rel=1e-6)


def test_validate_pinned_to_oracle(cuda, oracle):
    """cqrrpt_gpu_validate's orth_2 / orth_F / recon equal the restated
    validate() (qrcp.cc:150-196) on the same factors, to rounding."""
    from paper_2311_08316_b200 import _lib
    import ctypes
    import torch
    for (m, n, seed) in [(3000, 64, 1), (5000, 200, 2)]:
        a = oracle.gen_spectral(m, n, 10.0 ** (-6 * np.arange(n) / (n - 1)), seed)
        ref = oracle.cqrrpt(a, gamma=1.25, nnz=8, seed=0)
        vr = oracle.validate(a, ref.q, ref.r, ref.pivots)
        A, Q, R = (cuda.to_device_colmajor(x) for x in (a, ref.q, ref.r))
        J = torch.as_tensor(ref.pivots, dtype=torch.int64, device="cuda")
        of, o2, rc = _lib._f64(), _lib._f64(), _lib._f64()
        _lib.check(_lib.load().cqrrpt_gpu_validate(m, n, ref.k, A.data_ptr(), m, Q.data_ptr(), m, R.data_ptr(),
                                                   ref.k, J.data_ptr(), ctypes.byref(of), ctypes.byref(o2),
                                                   ctypes.byref(rc), None), "validate")
        torch.cuda.synchronize()
        assert of.value == pytest.approx(vr["orth_fro"], rel=1e-3)
        assert o2.value == pytest.approx(vr["orth_loss"], rel=1e-3)
        assert rc.value == pytest.approx(vr["recon_rel"], rel=1e-3)


def test_c_abi_host_outputs_path(cuda, oracle):
    """cqrrpt() from host numpy (the reference-signature adapter path)."""
    a = oracle.gen_gaussian(3000, 64, 12)
    out = cuda.cqrrpt(a, cuda.CqrrptConfig(nnz_per_col=8))
    ref = oracle.cqrrpt(a, gamma=1.25, nnz=8, seed=0)
    assert np.array_equal(out.factorization.pivots, ref.pivots)
    assert out.k == ref.k
    assert out.diagnostics.validation.passed


def test_cxx_reference_signature_adapter(cuda):
    """include/cqrrpt_b200.hh (cqrrpt_b200::cqrrpt(const DenseMatrix&, const CqrrptConfig&))
    running the reference test-suite assertions from C++ (tests/cxx/adapter_test.cc)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(__file__), "cxx", "_build", "adapter_test")
    if not os.path.exists(exe):
        from paper_2311_08316_b200.build import build_cxx_adapter_test
        exe = build_cxx_adapter_test()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout


@pytest.mark.parametrize("pinned,m", [(False, 9000), (True, 9000), (True, 70001)])
def test_dgeqpt_host_matches_device_path(cuda, oracle, pinned, m):
    """cqrrpt_gpu_dgeqpt_host with whole passes (host in/out, Q streamed back
    during the final TRSM) gives the device path's factors bit for bit. m = 70001: A arrives in
    4 row chunks and the exact sketch follows them with its chains carried
    across launches (ragged last chunk)."""
    import torch
    n = 200
    a = oracle.gen_gaussian(m, n, 21)
    A = cuda.to_device_colmajor(a)
    dev = cuda.dgeqpt(A, d_factor=1.25, nnz=8, seed=2)
    if pinned:
        ah = torch.from_numpy(np.ascontiguousarray(a.T)).pin_memory().t()
        host = cuda.dgeqpt_host(ah, d_factor=1.25, nnz=8, seed=2, wavefront=False)
        q, r, j = host.q.numpy(), host.r.numpy(), host.pivots.numpy()
    else:
        host = cuda.dgeqpt_host(a, d_factor=1.25, nnz=8, seed=2, wavefront=False)
        q, r, j = host.q, host.r, host.pivots
    assert (host.k, host.k0) == (dev.k, dev.k0)
    assert np.array_equal(j, dev.pivots.cpu().numpy())
    assert np.array_equal(q, A[:, :dev.k].cpu().numpy())
    assert np.array_equal(r, dev.r.cpu().numpy())


@pytest.mark.parametrize("case", ["ragged", "truncated", "dups", "wide_blocks"])
def test_dgeqpt_host_wavefront(cuda, oracle, case):
    """The 128-column wavefront (precondition, Gram columns, potrf_cols,
    diagonal-block inverses, Q blocks; on the host entry point also the
    download): the device and host entry points agree bit for bit, the same
    J, k0 and k as the whole passes, Q and R to rounding (its Gram sums m in
    more, fixed slices), bitwise repeatable; including inputs where the
    speculated k = k0 is wrong (stage 2 truncates: the final solve is redone)
    and inputs with duplicated columns (the reference's stage-2 failure
    inputs)."""
    eps = 1e-4
    if case == "ragged":      # k0 = 200: one full wavefront block and one of 72 columns
        a = oracle.gen_gaussian(9000, 200, 31)
    elif case == "truncated":  # tight eps_tol: stage 2 keeps fewer than k0 columns
        u, _ = np.linalg.qr(oracle.gen_gaussian(6000, 160, 32))
        v, _ = np.linalg.qr(oracle.gen_gaussian(160, 160, 33))
        a = np.asfortranarray((u * 10.0 ** (-12.0 * np.arange(160) / 159)) @ v.T)
        eps = 2e-16
    elif case == "dups":
        base = oracle.gen_gaussian(3000, 70, 34)
        a = np.asfortranarray(np.concatenate([base, base[:, :30]], axis=1))
    else:                      # k0 = 384: three blocks, several Cholesky steps per block
        a = oracle.gen_gaussian(70000, 384, 35)
    A = cuda.to_device_colmajor(a)
    dev = cuda.dgeqpt(A, d_factor=1.25, nnz=8, seed=3, eps_tol=eps, wavefront=True)
    W = cuda.to_device_colmajor(a)
    dwhole = cuda.dgeqpt(W, d_factor=1.25, nnz=8, seed=3, eps_tol=eps)
    whole = cuda.dgeqpt_host(a, d_factor=1.25, nnz=8, seed=3, eps_tol=eps, wavefront=False)
    k = dev.k
    assert (whole.k, whole.k0) == (dwhole.k, dwhole.k0) == (dev.k, dev.k0)
    assert np.array_equal(whole.pivots, dwhole.pivots.cpu().numpy())
    assert np.array_equal(whole.q, W[:, :k].cpu().numpy())
    assert np.array_equal(whole.r, dwhole.r.cpu().numpy())
    wav = cuda.dgeqpt_host(a, d_factor=1.25, nnz=8, seed=3, eps_tol=eps)
    again = cuda.dgeqpt_host(a, d_factor=1.25, nnz=8, seed=3, eps_tol=eps)
    assert (wav.k, wav.k0) == (dev.k, dev.k0)
    assert np.array_equal(wav.pivots, whole.pivots)
    assert np.array_equal(wav.pivots, dev.pivots.cpu().numpy())
    assert np.array_equal(wav.q, A[:, :k].cpu().numpy())
    assert np.array_equal(wav.r, dev.r.cpu().numpy())
    assert np.array_equal(again.q, wav.q) and np.array_equal(again.r, wav.r)
    # the in-place variant (Q into A after the whole precondition, blocks still
    # streamed: what the host entry point does when Q's own buffer does not fit)
    import os
    os.environ["CQRRPT_WF_INPLACE"] = "1"
    try:
        inpl = cuda.dgeqpt_host(a, d_factor=1.25, nnz=8, seed=3, eps_tol=eps)
    finally:
        del os.environ["CQRRPT_WF_INPLACE"]
    assert (inpl.k, inpl.k0) == (wav.k, wav.k0) and np.array_equal(inpl.pivots, wav.pivots)
    assert np.array_equal(inpl.q, wav.q) and np.array_equal(inpl.r, wav.r)
    if k:
        assert np.max(np.abs(wav.q - whole.q)) <= 1e-11 * np.max(np.abs(whole.q))
        rn = np.linalg.norm(whole.r, axis=0)
        assert np.all(np.linalg.norm(wav.r - whole.r, axis=0) <= 1e-11 * np.maximum(rn, 1e-300))
    if case == "truncated":
        assert 0 < dev.k < dev.k0, (dev.k, dev.k0)
