"""The two Gram engines (reference gram, linalg.cc:298-307): the INT8
tensor-core emulation (csrc/ozaki.cu, Ozaki scheme II) and the DMMA SYRK.

For the emulation: error against an extended-precision Gram within a small
multiple of u ||x_i|| ||x_j|| (the DMMA engine's own level), bitwise symmetry,
the leading-block property the stage-2 Cholesky retry relies on
(gram(X[:, :j]) == gram(X)[:j, :j] bitwise; cqrrpt.cc:162-164), ragged row
chunks, the split (symmetric half-block) and full product layouts, zero
columns, and determinism."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

U = 1.1102230246251565e-16


def _gram(kernels, x, engine, monkeypatch):
    import torch
    monkeypatch.setenv("CQRRPT_GPU_GRAM", engine)
    g = kernels.gram(x)
    torch.cuda.synchronize()
    return g.cpu().numpy()


def _exact(xh, pairs):
    return np.array([float(np.sum(xh[:, i].astype(np.longdouble) * xh[:, j].astype(np.longdouble)))
                     for i, j in pairs])


@pytest.mark.parametrize("m,k,kind", [(200000, 384, "gauss"), (200000, 1032, "gauss"), (140000, 1024, "spiky"),
                                      (70000, 40, "graded"), (131072, 264, "zerocol")])
def test_int8_gram_accuracy_symmetry(cuda, monkeypatch, m, k, kind):
    import torch
    from paper_2311_08316_b200 import kernels
    g = torch.Generator(device="cuda").manual_seed(k)
    x = torch.randn((k, m), dtype=torch.float64, device="cuda", generator=g).t()
    if kind == "spiky":
        x[:7] *= 1e5
    if kind == "graded":
        x *= (10.0 ** (-8.0 * torch.rand(k, dtype=torch.float64, device="cuda", generator=g)))[None, :]
    if kind == "zerocol":
        x[:, 5] = 0.0
    xh = x.cpu().numpy()
    go = _gram(kernels, x, "ozaki", monkeypatch)
    gd = _gram(kernels, x, "dmma", monkeypatch)
    assert np.array_equal(go, go.T)
    rng = np.random.default_rng(1)
    pairs = [(int(a), int(b)) for a, b in zip(rng.integers(0, k, 300), rng.integers(0, k, 300))]
    pairs += [(i, i) for i in range(min(k, 40))]
    ex = _exact(xh, pairs)
    nrm = np.linalg.norm(xh, axis=0)
    scale = np.array([nrm[i] * nrm[j] for i, j in pairs])
    scale[scale == 0] = 1.0
    err_o = np.max(np.abs(np.array([go[i, j] for i, j in pairs]) - ex) / scale) / U
    err_d = np.max(np.abs(np.array([gd[i, j] for i, j in pairs]) - ex) / scale) / U
    assert err_o <= max(4 * err_d, 64.0), (err_o, err_d)
    if kind == "zerocol":
        assert np.all(go[5] == 0.0) and np.all(go[:, 5] == 0.0)


def test_int8_gram_leading_block_and_determinism(cuda, monkeypatch):
    import torch
    from paper_2311_08316_b200 import kernels
    m, k = 150000, 1024
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn((k, m), dtype=torch.float64, device="cuda", generator=g).t()
    full = _gram(kernels, x, "ozaki", monkeypatch)
    again = _gram(kernels, x, "ozaki", monkeypatch)
    assert np.array_equal(full, again)
    for j in (1, 37, 512, 999):  # full-layout and split-layout leading blocks
        lead = _gram(kernels, x[:, :j], "ozaki", monkeypatch)
        assert np.array_equal(lead, full[:j, :j]), j
