"""Pin the device restatement of the reference generators (tests/gen, test
infrastructure for the full-size parity tests) to the oracle's CPU
generators, which tests/test_oracle.py pins to the built reference: bitwise
equal outputs on odd sizes (ragged 128-element chunks, 1-3 element dot
epilogues)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,seed", [(1000, 48, 3), (2051, 64, 0), (517, 130, 7)])
def test_gen_spectral_bitwise(cuda, oracle, m, n, seed):
    from gen import gen
    sig = 10.0 ** (-10.0 * np.arange(n) / (n - 1))
    want = oracle.gen_spectral(m, n, sig, seed)
    got = gen.gen_spectral(oracle, m, n, sig, seed).cpu().numpy()
    assert np.array_equal(got, want)


@pytest.mark.parametrize("m,n,r,seed", [(3001, 80, 20, 0), (1024, 33, 33, 5)])
def test_gen_exact_rank_bitwise(cuda, oracle, m, n, r, seed):
    from gen import gen
    want = oracle.gen_exact_rank(m, n, r, seed)
    got = gen.gen_exact_rank(oracle, m, n, r, seed).cpu().numpy()
    assert np.array_equal(got, want)


def test_cqrrpt_does_not_modify_cuda_input(cuda, oracle):
    """cqrrpt() takes M by const reference (cqrrpt.hh:140): a column-major
    float64 CUDA input must come back unchanged (the working copy
    used to alias it)."""
    import torch
    a = cuda.to_device_colmajor(oracle.gen_gaussian(2000, 40, 9))
    before = a.clone()
    out = cuda.cqrrpt(a, cuda.CqrrptConfig(nnz_per_col=8, validate_output=False))
    torch.cuda.synchronize()
    assert out.k == 40
    assert torch.equal(a, before)
