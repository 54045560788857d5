"""BASELINE workloads for bench.py and the tools (harness only, not product).

Synthetic inputs with the shapes, sizes and value distributions of
BASELINE.json's configs; seeded, generated on the device with
torch in fixed 65536-row tiles so that any row block of the one global matrix
can be produced independently: rank r of an N-GPU run generates exactly rows
[r m/N, (r+1) m/N) of the same matrix the 1-GPU run factors, and the CPU
reference arm takes the matrix's first S rows. (The bit-exact reference
generators are used by the parity tests, tests/gen; timing does not depend
on the bits.)

  C1  16384 x 256     i.i.d. N(0,1)
  C2  131072 x 1024   U diag(sigma) V^T, sigma_i = 10^(-10 i/(n-1)), U, V from QR of Gaussians (one rank)
  C3  262144 x 2048   A B + 1e-12 ||A B||_F / sqrt(mn) G, A m x 1024, B 1024 x n (numerical rank 1024)
  C3b as C3 with noise 1e-14
  C4  1048576 x 4096  i.i.d. N(0,1)
  C5  4194304 x n     N(0,1) columns scaled by 10^(-8 pi(j)/(n-1)), pi a seeded permutation (n = 256..2048)
"""
from __future__ import annotations

import numpy as np

TILE = 65536
SEED = 0

CONFIGS = {
    "C1": dict(m=16384, n=256, gamma=1.25, kind="gauss"),
    "C2": dict(m=131072, n=1024, gamma=1.25, kind="spectral"),
    "C3": dict(m=262144, n=2048, gamma=1.25, kind="lowrank", rank=1024, noise=1e-12),
    "C3b": dict(m=262144, n=2048, gamma=1.25, kind="lowrank", rank=1024, noise=1e-14),
    "C4": dict(m=1048576, n=4096, gamma=1.25, kind="gauss"),
    "C5_256": dict(m=4194304, n=256, gamma=1.25, kind="graded"),
    "C5_512": dict(m=4194304, n=512, gamma=1.25, kind="graded"),
    "C5_1024": dict(m=4194304, n=1024, gamma=1.25, kind="graded"),
    "C5_2048": dict(m=4194304, n=2048, gamma=1.25, kind="graded"),
}

DESCRIPTION = {
    "C1": "BASELINE configs[0]: M 16384x256 FP64 i.i.d. N(0,1)",
    "C2": "BASELINE configs[1]: M 131072x1024 FP64 = U diag(sigma) V^T, sigma_i = 10^(-10 i/(n-1)) (cond 1e10)",
    "C3": "BASELINE configs[2]: M 262144x2048 FP64 = A B + 1e-12 ||AB||_F/sqrt(mn) G (numerical rank 1024)",
    "C3b": "C3 with noise 1e-14 (SURVEY C3b: the reference truncates to k = 1024)",
    "C4": "BASELINE configs[3]: M 1048576x4096 FP64 i.i.d. N(0,1) (32 GiB)",
    "C5_256": "BASELINE configs[4]: M 4194304x256 FP64, Gaussian columns scaled 1..1e-8 in a seeded random order",
    "C5_512": "BASELINE configs[4]: M 4194304x512 FP64, Gaussian columns scaled 1..1e-8 in a seeded random order",
    "C5_1024": "BASELINE configs[4]: M 4194304x1024 FP64, Gaussian columns scaled 1..1e-8 in a seeded random order",
    "C5_2048": "BASELINE configs[4]: M 4194304x2048 FP64 (64 GiB), Gaussian columns scaled 1..1e-8 in a "
               "seeded random order",
}


def canonical_flops(m, n):
    """CQRRPT canonical flops 2 m n^2 - 2 n^3 / 3."""
    return 2.0 * m * n * n - 2.0 * n ** 3 / 3.0


def _gen(torch, device, seed):
    return torch.Generator(device=device).manual_seed(int(seed))


def column_factors(n, seed=SEED):
    """C5: 10^(-8 pi(j)/(n-1)) with pi a seeded permutation of 0..n-1."""
    perm = np.random.default_rng(seed + 0x7065726D).permutation(n)
    return 10.0 ** (-8.0 * perm / (n - 1))


def fill_rows(cfg, r0, r1, out, device="cuda", seed=SEED, fro_sq_total=None):
    """Write rows [r0, r1) of the config's global matrix into ``out``, a
    column-major (r1-r0) x n tensor on ``device``. ``fro_sq_total`` (C3 only)
    is ||A B||_F^2 of the WHOLE matrix (see lowrank_fro_sq) for the noise
    scale."""
    import torch
    m, n, kind = cfg["m"], cfg["n"], cfg["kind"]
    store = out.t()  # (n, rows) row-major view of the column-major block
    if kind == "spectral":
        if (r0, r1) != (0, m):
            raise ValueError("the C2 spectral workload is generated whole (one rank)")
        g = _gen(torch, device, seed)
        u = torch.linalg.qr(torch.randn((m, n), dtype=torch.float64, device=device, generator=g))[0]
        v = torch.linalg.qr(torch.randn((n, n), dtype=torch.float64, device=device, generator=g))[0]
        sig = 10.0 ** (-10.0 * torch.arange(n, dtype=torch.float64, device=device) / (n - 1))
        store.copy_(((u * sig) @ v.T).T)
        return out
    if kind == "lowrank":
        r = cfg["rank"]
        bt = torch.randn((n, r), dtype=torch.float64, device=device, generator=_gen(torch, device, seed + 77))
        scale = None
        if fro_sq_total is not None:
            scale = cfg["noise"] * float(fro_sq_total) ** 0.5 / (float(m) * float(n)) ** 0.5
    f = None
    if kind == "graded":
        f = torch.as_tensor(column_factors(n, seed), device=device)[:, None]
    for t in range(r0 // TILE, (r1 + TILE - 1) // TILE):
        a, b = t * TILE, min(m, (t + 1) * TILE)
        lo, hi = max(a, r0), min(b, r1)
        if lo >= hi:
            continue
        g = _gen(torch, device, seed * 7919 + t + 1)
        if kind == "lowrank":
            at = torch.randn((r, b - a), dtype=torch.float64, device=device, generator=g)
            tile = bt @ at
            if scale is not None:
                noise = torch.randn((n, b - a), dtype=torch.float64, device=device,
                                    generator=_gen(torch, device, seed * 7919 + t + 1_000_003))
                tile += noise * scale
        else:
            tile = torch.randn((n, b - a), dtype=torch.float64, device=device, generator=g)
            if f is not None:
                tile *= f
        store[:, lo - r0:hi - r0].copy_(tile[:, lo - a:hi - a])
        del tile
    return out


def lowrank_tile_sq(cfg, r0, r1, device="cuda", seed=SEED):
    """{tile index: ||tile of A B||_F^2} for the 65536-row tiles that rows
    [r0, r1) cover (r0, r1 tile-aligned or the matrix end). Summed in tile
    order, these give a noise scale that does not depend on the rank count."""
    import torch
    out = {}
    for t in range(r0 // TILE, (r1 + TILE - 1) // TILE):
        a, b = t * TILE, min(cfg["m"], (t + 1) * TILE)
        tmp = torch.empty((cfg["n"], b - a), dtype=torch.float64, device=device).t()
        fill_rows(cfg, a, b, tmp, device, seed, fro_sq_total=None)
        out[t] = float((tmp * tmp).sum().item())
        del tmp
    return out


def lowrank_fro_sq(cfg, device="cuda", seed=SEED, dist=None, r0=0, r1=None):
    """||A B||_F^2 of the whole C3 matrix: per-tile sums (this rank's rows,
    all-gathered across ranks when ``dist`` is given) added in tile order."""
    r1 = cfg["m"] if r1 is None else r1
    parts = lowrank_tile_sq(cfg, r0, r1, device, seed)
    if dist is not None:
        gathered = [None] * dist.get_world_size()
        dist.all_gather_object(gathered, parts)
        parts = {}
        for g in gathered:
            parts.update(g)
    return float(sum(parts[t] for t in sorted(parts)))


def make_rows(cfg, r0, r1, device="cuda", seed=SEED, dist=None):
    """Allocate and fill rows [r0, r1) (column-major). For C3 the global
    noise scale needs ||AB||_F^2 over all ranks (``dist`` all-reduces it)."""
    import torch
    out = torch.empty((cfg["n"], r1 - r0), dtype=torch.float64, device=device).t()
    fro = None
    if cfg["kind"] == "lowrank":
        if dist is None and (r0, r1) != (0, cfg["m"]):
            raise ValueError("C3 rows of part of the matrix need the whole ||AB||_F: pass dist, or r0=0, r1=m")
        fro = lowrank_fro_sq(cfg, device, seed, dist, r0, r1)
    return fill_rows(cfg, r0, r1, out, device, seed, fro_sq_total=fro)
