"""The exact INT8 tensor-core TRSM engine (csrc/oztrsm.cu, tcgen05 kind::i8)
against the DMMA engine and the CPU oracle (trsm_right, linalg.cc:244-277).

Bars: the emulation is exact integer arithmetic up to the 2^-54 scaling of
each 128-wide step's operands and the dropped digit pairs (<= 2^-61 of the
FP64 GEMM's normwise bound), so the two engines agree column-wise to a few
ulps of the solution and both satisfy the reference TRSM's residual bar.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

U = 1.1102230246251565e-16


def dev(pkg, a):
    return pkg.to_device_colmajor(np.asfortranarray(a))


def host(t):
    return np.asfortranarray(t.cpu().numpy())


@pytest.fixture
def engine(monkeypatch):
    def use(name):
        monkeypatch.setenv("CQRRPT_GPU_TRSM", name)
    return use


def _upper(oracle, k, seed, graded=False):
    g = oracle.gen_gaussian(int(1.25 * k) + 1, k, seed)
    if graded:  # C5-like: columns scaled 1 .. 1e-8 in a seeded order
        perm = np.random.default_rng(seed).permutation(k)
        g = g * (10.0 ** (-8.0 * perm / max(k - 1, 1)))[None, :]
    r, _, _ = oracle.qrcp(g)
    return np.ascontiguousarray(r[:k, :k])


@pytest.mark.parametrize("m,k,graded", [(16384, 256, False), (4098, 300, True), (70002, 513, False),
                                        (2000, 129, True), (262144, 384, False)])
def test_int8_engine_matches_dmma_and_oracle(cuda, oracle, engine, m, k, graded):
    import torch
    from paper_2311_08316_b200 import kernels
    b = oracle.gen_gaussian(m, k + 3, 11)
    u = _upper(oracle, k, 12, graded)
    cols = np.random.default_rng(1).permutation(k + 3)[:k].astype(np.int64)
    B, Ud = dev(cuda, b), dev(cuda, u)
    tc = torch.as_tensor(cols, device="cuda")
    engine("oz")
    assert kernels.trsm_engine(m, k) == "int8"
    x_oz = host(kernels.trsm_right(B, Ud, cols=tc))
    engine("dmma")
    x_dm = host(kernels.trsm_right(B, Ud, cols=tc))
    bc = b[:, cols]
    # both engines: the reference TRSM's residual bar
    for x in (x_oz, x_dm):
        assert np.linalg.norm(x @ u - bc) <= 1e-12 * np.linalg.norm(np.abs(x) @ np.abs(u))
    # column-wise agreement of the two engines
    diff = np.linalg.norm(x_oz - x_dm, axis=0) / np.linalg.norm(x_dm, axis=0)
    assert np.max(diff) <= 1e3 * k * U
    if m * k <= 16384 * 256:  # the oracle's own solve
        ref = oracle.trsm_right(np.asfortranarray(bc), u)
        err = np.linalg.norm(x_oz - ref, axis=0) / np.linalg.norm(ref, axis=0)
        assert np.max(err) <= 1e3 * k * U


def test_int8_engine_deterministic_and_exact_on_identity(cuda, oracle, engine):
    from paper_2311_08316_b200 import kernels
    engine("oz")
    b = oracle.gen_gaussian(8192, 300, 3)
    B = dev(cuda, b)
    # U = I: every update subtracts exact zeros, the diagonal solves are exact
    x = host(kernels.trsm_right(B, dev(cuda, np.eye(300))))
    assert np.array_equal(x, b)
    u = _upper(oracle, 300, 4)
    Ud = dev(cuda, u)
    x1 = host(kernels.trsm_right(B, Ud))
    x2 = host(kernels.trsm_right(B, Ud))
    assert np.array_equal(x1, x2)


def test_int8_engine_propagates_non_finite(cuda, oracle, engine):
    from paper_2311_08316_b200 import kernels
    engine("oz")
    b = oracle.gen_gaussian(4096, 260, 5)
    b[17, 3] = np.nan  # row 17 of the first block: its updates must be NaN, not garbage
    u = _upper(oracle, 260, 6)
    x = host(kernels.trsm_right(dev(cuda, b), dev(cuda, u)))
    assert np.all(np.isnan(x[17, 128:]))
    assert np.all(np.isfinite(np.delete(x, 17, axis=0)))


def test_dgeqpt_with_int8_engine_matches_dmma(cuda, oracle, engine):
    """The whole driver (both solves on the INT8 engine) against the DMMA run:
    same J and k (decided before the solves), Q and R to rounding."""
    from paper_2311_08316_b200 import dgeqpt
    a = oracle.gen_gaussian(65536, 512, 21)
    res = {}
    for name in ("oz", "dmma"):
        engine(name)
        A = dev(cuda, a)
        r = dgeqpt(A, d_factor=1.25, nnz=8, seed=0)
        res[name] = (host(A[:, : r.k]), host(r.r), r.pivots.cpu().numpy(), r.k)
    qo, ro, jo, ko = res["oz"]
    qd, rd, jd, kd = res["dmma"]
    assert ko == kd and np.array_equal(jo, jd)
    assert np.linalg.norm(qo.T @ qo - np.eye(ko)) <= 1e-13
    assert np.linalg.norm(a[:, jo] - qo @ ro) <= 1e-14 * np.linalg.norm(a)
    assert np.max(np.abs(ro - rd)) <= 1e3 * 512 * U * np.max(np.abs(rd))


def test_int8_engine_odd_rows_even_leading_dimension(cuda, oracle, engine):
    """m odd with even leading dimensions: TMA applies the row bound of a box
    at 16-byte granularity, so the engine stands down for odd m (DMMA takes
    the solve); the padding row below the matrix stays untouched."""
    import torch
    from paper_2311_08316_b200 import _lib, kernels
    from paper_2311_08316_b200.kernels import _p
    m, k, ld = 70001, 300, 70002
    b = oracle.gen_gaussian(m, k + 3, 31)
    u = _upper(oracle, k, 32)
    cols = np.random.default_rng(2).permutation(k + 3)[:k].astype(np.int64)
    bbuf = torch.zeros((k + 3, ld), dtype=torch.float64, device="cuda")
    bbuf[:, :m] = torch.from_numpy(np.ascontiguousarray(b.T)).cuda()
    xbuf = torch.full((k, ld), 7.0, dtype=torch.float64, device="cuda")
    ud = dev(cuda, u)
    tc = torch.as_tensor(cols, device="cuda")
    engine("oz")
    _lib.check(_lib.load().cqrrpt_gpu_trsm_right(m, k, _p(bbuf), ld, _p(tc), _p(ud), k, _p(xbuf), ld, None),
               "trsm_right")
    x = np.asfortranarray(xbuf.t()[:m].cpu().numpy())
    assert np.all(xbuf[:, m].cpu().numpy() == 7.0)  # the padding row is not written
    engine("dmma")
    ref = host(kernels.trsm_right(dev(cuda, b), ud, cols=tc))
    diff = np.linalg.norm(x - ref, axis=0) / np.linalg.norm(ref, axis=0)
    assert np.max(diff) <= 1e3 * k * U
