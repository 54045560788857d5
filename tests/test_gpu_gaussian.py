"""Gaussian sketch family on device (sketch.cc:62-72 + apply = matmul,
SURVEY §8(f) row 3) against the oracle's operator (bit-identical to the
reference's, tests/test_oracle.py) and end to end through dgeqpt."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
U = 1.1102230246251565e-16


def dev(pkg, a):
    return pkg.to_device_colmajor(np.asfortranarray(a))


@pytest.mark.parametrize("m,n,d,seed,c0", [(2000, 40, 50, 7, 0), (777, 33, 41, 3, 1234),
                                           (70000, 64, 80, 11, 0), (5000, 300, 375, 0, 0)])
def test_gaussian_sketch_matches_operator(cuda, oracle, m, n, d, seed, c0):
    from paper_2311_08316_b200 import kernels
    a = oracle.gen_gaussian(m, n, seed + 5)
    got = kernels.gaussian_sketch(dev(cuda, a), d, seed, c0).cpu().numpy()
    ref = oracle.gaussian_apply(d, a, seed, c0)
    # each entry is a length-m dot of N(0, 1/d) with N(0, 1): rounding ~ u sqrt(m)
    assert np.max(np.abs(got - ref)) <= 1e3 * U * np.sqrt(m) * np.max(np.abs(ref)) + 1e-300


def test_gaussian_sketch_deterministic_and_row_offsets_sum(cuda, oracle):
    from paper_2311_08316_b200 import kernels
    a = oracle.gen_gaussian(3000, 24, 2)
    A = dev(cuda, a)
    x = kernels.gaussian_sketch(A, 30, 5).cpu().numpy()
    assert np.array_equal(x, kernels.gaussian_sketch(A, 30, 5).cpu().numpy())
    parts = [kernels.gaussian_sketch(dev(cuda, a[lo:hi]), 30, 5, c0=lo).cpu().numpy()
             for lo, hi in [(0, 1100), (1100, 3000)]]
    assert np.max(np.abs(sum(parts) - x)) <= 1e-12 * np.linalg.norm(x)


def test_dgeqpt_gaussian_family(cuda, oracle):
    """End to end with the Gaussian operator: J and k as the reference's
    algorithm on the oracle's sketch (no near-ties here), Q/R at the
    unit-roundoff level."""
    m, n, gamma, seed = 4096, 96, 1.25, 3
    a = oracle.gen_gaussian(m, n, 1)
    A = dev(cuda, a)
    res = cuda.dgeqpt(A, d_factor=gamma, nnz=4, seed=seed, sketch_family="gaussian")
    d = oracle.sketch_rows_for(gamma, n)
    _, j_ref, k_ref = oracle.qrcp(oracle.gaussian_apply(d, a, seed))
    assert res.k0 == res.k == n == k_ref
    assert np.array_equal(res.pivots.cpu().numpy(), j_ref)
    q = A[:, :res.k].cpu().numpy()
    v = oracle.validate(a, q, res.r.cpu().numpy(), res.pivots.cpu().numpy())
    assert v["orth_fro"] <= 1e2 * n * U and v["recon_rel"] <= 1e2 * n * U


def test_dgeqpt_unknown_family_rejected(cuda, oracle):
    from paper_2311_08316_b200 import _lib
    A = dev(cuda, oracle.gen_gaussian(100, 10, 1))
    with pytest.raises(_lib.InvalidArgument):
        cuda.dgeqpt(A, sketch_family="bogus")


# ---- SRFT family (sketch.cc:100-119, 147-166) --------------------------------
@pytest.mark.parametrize("m,n,d,seed", [(100, 7, 20, 3), (1000, 30, 40, 7), (4096, 16, 100, 1),
                                        (5000, 3, 5000, 2), (70000, 24, 300, 9), (131072, 5, 1280, 0)])
def test_srft_sketch_bit_identical(cuda, oracle, m, n, d, seed):
    """Stage-ordered butterflies (4096-blocks in shared memory, then the
    strided residues) reproduce the reference's fwht bit for bit."""
    from paper_2311_08316_b200 import kernels
    a = oracle.gen_gaussian(m, n, seed + 1)
    got = kernels.srft_sketch(dev(cuda, a), d, seed).cpu().numpy()
    assert np.array_equal(got, oracle.srft_apply(d, a, seed))


def test_dgeqpt_srft_family(cuda, oracle):
    m, n, gamma, seed = 6000, 80, 1.25, 4
    a = oracle.gen_gaussian(m, n, 2)
    A = dev(cuda, a)
    res = cuda.dgeqpt(A, d_factor=gamma, seed=seed, sketch_family="srft")
    d = oracle.sketch_rows_for(gamma, n)
    _, j_ref, k_ref = oracle.qrcp(oracle.srft_apply(d, a, seed))  # bit-identical sketch -> J exact
    assert res.k0 == res.k == k_ref == n
    assert np.array_equal(res.pivots.cpu().numpy(), j_ref)
    q = A[:, :res.k].cpu().numpy()
    v = oracle.validate(a, q, res.r.cpu().numpy(), res.pivots.cpu().numpy())
    assert v["orth_fro"] <= 1e2 * n * U and v["recon_rel"] <= 1e2 * n * U
