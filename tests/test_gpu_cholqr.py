"""Device CholeskyQR / CholeskyQR2 (cqrrpt.cc:75-90, §8(f) row 2) against the
oracle's composition of the reference's own gram/cholesky/trsm, and the
reference test-suite's assertions (test_cqrrpt.cc:36-82)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
U = 1.1102230246251565e-16


def dev(pkg, a):
    return pkg.to_device_colmajor(np.asfortranarray(a))


def with_condition(oracle, m, n, cond, seed):
    # test_cqrrpt.cc:25-32: geometric spectrum from 1 down to 1/cond
    sigma = cond ** (-np.arange(n) / (n - 1))
    return oracle.gen_spectral(m, n, sigma, seed)


def orth_loss(q):
    g = q.T @ q - np.eye(q.shape[1])
    return np.linalg.norm(g, 2)


def run(pkg, a, twice):
    from paper_2311_08316_b200 import kernels
    A = dev(pkg, a)
    r, fi = kernels.cholesky_qr(A, twice=twice)
    return A.cpu().numpy(), (None if r is None else r.cpu().numpy()), fi


@pytest.mark.parametrize("twice", [False, True])
@pytest.mark.parametrize("m,n,seed", [(300, 24, 2), (1000, 100, 3), (5000, 300, 4)])
def test_cholesky_qr_matches_oracle(cuda, oracle, m, n, seed, twice):
    a = oracle.gen_gaussian(m, n, seed)
    q, r, fi = run(cuda, a, twice)
    q_ref, r_ref, fi_ref = oracle.cholesky_qr(a, twice)
    assert fi == fi_ref == 0
    assert np.all(np.tril(r, -1) == 0)
    err = np.linalg.norm(r - r_ref, axis=0) / np.linalg.norm(r_ref, axis=0)
    assert np.max(err) <= 1e3 * n * U
    assert orth_loss(q) <= 10 * max(orth_loss(q_ref), n * U)
    assert np.linalg.norm(q @ r - a) <= 1e2 * n * U * np.linalg.norm(a)


def test_cholesky_qr_orthonormal_input_is_near_noop(cuda, oracle):
    q0 = np.linalg.qr(oracle.gen_gaussian(60, 8, 1))[0]  # test_cqrrpt.cc:36-47
    q, r, fi = run(cuda, q0, False)
    assert fi == 0
    assert np.max(np.abs(r - np.eye(8))) < 1e-13
    assert np.max(np.abs(q - q0)) < 1e-13


def test_cholesky_qr_degrades_as_u_cond_squared(cuda, oracle):
    q, r, fi = run(cuda, with_condition(oracle, 300, 24, 1e3, 2), False)  # test_cqrrpt.cc:49-58
    assert fi == 0 and orth_loss(q) <= 1e-9
    q, r, fi = run(cuda, with_condition(oracle, 300, 24, 1e9, 3), False)
    if fi == 0:
        assert orth_loss(q) >= 1e-3


def test_cholesky_qr2_restores_orthogonality(cuda, oracle):
    q0 = np.linalg.qr(oracle.gen_gaussian(50, 6, 4))[0]  # test_cqrrpt.cc:60-82
    q, r, fi = run(cuda, q0, True)
    assert fi == 0 and orth_loss(q) <= 1e-14
    mid = with_condition(oracle, 300, 24, 1e6, 5)
    q, r, fi = run(cuda, mid, True)
    assert fi == 0 and orth_loss(q) <= 1e-12
    assert np.linalg.norm(q @ r - mid) <= 1e-12 * np.linalg.norm(mid)
    q, r, fi = run(cuda, with_condition(oracle, 300, 24, 1e10, 6), True)
    if fi == 0:
        assert orth_loss(q) >= 1e-6


def test_cholesky_qr_failure_index_matches_reference(cuda, oracle):
    a = oracle.gen_gaussian(30, 7, 13)
    a[:, 5:7] = a[:, :2]  # duplicate columns: exactly singular Gram
    _, r, fi = run(cuda, a, False)
    assert r is None and fi == oracle.cholesky_qr(a)[2] == 6


def test_cholesky_qr_rejects_wide(cuda, oracle):
    from paper_2311_08316_b200 import _lib
    with pytest.raises(_lib.InvalidArgument):
        run(cuda, oracle.gen_gaussian(5, 8, 1), False)
