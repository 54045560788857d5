"""Phase-level launch helpers over the C ABI (include/cqrrpt_gpu.h).

Each wraps one exported entry point and takes column-major float64 CUDA
tensors (stride (1, ld)). These are the building blocks the driver composes
and what the per-kernel parity tests call; each cites the reference
function it replaces.
"""
from __future__ import annotations

import ctypes

from . import _lib
from .cqrrpt import _ld, _stream_ptr, _torch, colmajor_empty


def _p(t):
    return t.data_ptr() if t is not None and t.numel() else None


def saso_plan(d: int, m: int, nnz: int, seed: int, c0: int = 0, stream=None):
    """sample_sketch SASO (sketch.cc:73-99) -> uint32 plan (m x nnz): row | sign<<31."""
    torch = _torch()
    plan = torch.empty((max(m, 1), nnz), dtype=torch.int32, device="cuda")
    _lib.check(_lib.load().cqrrpt_gpu_saso_plan(d, c0, m, nnz, seed, plan.data_ptr(), _stream_ptr(stream)),
               "saso_plan")
    return plan[:m]


def saso_sketch(a, d: int, nnz: int, seed: int, c0: int = 0, stream=None, fast: bool = False):
    """apply(S, M) for SASO (sketch.cc:131-146) -> d x n column-major.
    ``fast``: allow the c-split decomposition (not bit-identical)."""
    m, n = a.shape
    out = colmajor_empty(d, n)
    _lib.check(_lib.load().cqrrpt_gpu_saso_sketch_ex(m, n, _p(a), _ld(a) if m else 1, d, nnz, seed, c0,
                                                     out.data_ptr(), _ld(out), _lib.F_FAST_SKETCH if fast else 0,
                                                     _stream_ptr(stream)), "saso_sketch")
    return out


def gaussian_sketch(a, d: int, seed: int, c0: int = 0, stream=None):
    """apply(S, M) for the Gaussian family (sketch.cc:62-72, 124-127) -> d x n."""
    m, n = a.shape
    out = colmajor_empty(d, n)
    _lib.check(_lib.load().cqrrpt_gpu_gaussian_sketch(m, n, _p(a), _ld(a) if m else 1, d, seed, c0, out.data_ptr(),
                                                      _ld(out), _stream_ptr(stream)), "gaussian_sketch")
    return out


def srft_sketch(a, d: int, seed: int, stream=None):
    """apply(S, M) for the SRFT family (sketch.cc:100-119, 147-166) -> d x n, bit-identical."""
    m, n = a.shape
    out = colmajor_empty(d, n)
    _lib.check(_lib.load().cqrrpt_gpu_srft_sketch(m, n, _p(a), _ld(a) if m else 1, d, seed, out.data_ptr(),
                                                  _ld(out), _stream_ptr(stream)), "srft_sketch")
    return out


def qrcp(msk, rank_tol: float = -1.0, stream=None):
    """qrcp_maxnorm(M_sk, rank_tol, want_q=false) (qrcp.cc:35-97) -> (R k x n, pivots, k).
    ``msk`` is overwritten."""
    torch = _torch()
    d, n = msk.shape
    r = colmajor_empty(n, n)
    j = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    k = _lib._i64()
    _lib.check(_lib.load().cqrrpt_gpu_qrcp(d, n, _p(msk), _ld(msk) if d else 1, float(rank_tol), _p(r),
                                           _ld(r) if n else 1, j.data_ptr(), ctypes.byref(k), _stream_ptr(stream)),
               "qrcp")
    return r[: k.value, :], j[:n], k.value


def rank_stage1(r, stream=None) -> int:
    """rank_stage1 (cqrrpt.cc:92-112)."""
    k, n = r.shape
    k0 = _lib._i64()
    _lib.check(_lib.load().cqrrpt_gpu_rank_stage1(k, n, _p(r), _ld(r) if k else 1, ctypes.byref(k0),
                                                  _stream_ptr(stream)), "rank_stage1")
    return k0.value


def rank_stage2(m_k0, a_sk, eps_tol: float = 1e-4, method: int = _lib.COND_IDENTITY_DEVIATION,
                exact: bool = False, stream=None) -> dict:
    """rank_stage2(M_k0, A_sk, eps_tol) (cqrrpt.cc:149-209): the routine the
    driver runs after stage 1. Returns rank, k0_final, retries, cond_at_rank
    and the device factors r_pre (rank x rank) and m_pre (m x k0_final)."""
    m, k0 = m_k0.shape
    mpre = colmajor_empty(m, k0)
    rpre = colmajor_empty(k0, k0)
    rank, k0f = _lib._i64(), _lib._i64()
    retries, cond = _lib._i32(), _lib._f64()
    _lib.check(_lib.load().cqrrpt_gpu_rank_stage2(m, k0, _p(m_k0), _ld(m_k0) if m else 1, _p(a_sk), _ld(a_sk),
                                                  float(eps_tol), int(method), _lib.F_EXACT_STAGE2 if exact else 0,
                                                  _p(mpre), _ld(mpre) if m else 1, _p(rpre), _ld(rpre),
                                                  ctypes.byref(rank), ctypes.byref(k0f), ctypes.byref(retries),
                                                  ctypes.byref(cond), _stream_ptr(stream)), "rank_stage2")
    k = rank.value
    return dict(rank=k, k0_final=k0f.value, retries=retries.value, cond_at_rank=cond.value,
                r_pre=rpre[:k, :k], m_pre=mpre[:, : k0f.value])


def trsm_right(b, u, cols=None, stream=None):
    """trsm_right(B[:, cols], U) (linalg.cc:244-277) -> X = B[:, cols] U^{-1}."""
    m = b.shape[0]
    k = u.shape[0]
    x = colmajor_empty(m, k)
    _lib.check(_lib.load().cqrrpt_gpu_trsm_right(m, k, _p(b), _ld(b) if m else 1, _p(cols), _p(u),
                                                 _ld(u) if k else 1, _p(x), _ld(x) if m else 1,
                                                 _stream_ptr(stream)), "trsm_right")
    return x


def trsm_engine(m, k):
    """Engine of an m x k trsm_right: "dmma" (FP64 tensor cores) or "int8" (the
    exact tcgen05 kind::i8 emulation, csrc/oztrsm.cu)."""
    return "int8" if _lib.load().cqrrpt_gpu_trsm_engine(m, k) else "dmma"


def gram(x, stream=None):
    """gram(M) (linalg.cc:298-307) -> k x k, bitwise symmetric."""
    m, k = x.shape
    g = colmajor_empty(k, k)
    _lib.check(_lib.load().cqrrpt_gpu_gram(m, k, _p(x), _ld(x) if m else 1, _p(g), _ld(g) if k else 1,
                                           _stream_ptr(stream)), "gram")
    return g


def potrf(g, stream=None):
    """cholesky(G) (linalg.cc:223-242) -> (R leading block, failure_index). G is overwritten."""
    n = g.shape[0]
    fi = _lib._i64()
    _lib.check(_lib.load().cqrrpt_gpu_potrf(n, _p(g), _ld(g) if n else 1, ctypes.byref(fi), _stream_ptr(stream)),
               "potrf")
    j = n if fi.value == 0 else fi.value - 1
    return g[:j, :j], fi.value


def cond_estimate(r, method: int, stream=None) -> float:
    """cond_estimate(R, method) (cqrrpt.cc:114-147), reference semantics."""
    n = r.shape[0]
    v = _lib._f64()
    _lib.check(_lib.load().cqrrpt_gpu_cond_estimate(n, _p(r), _ld(r) if n else 1, int(method), ctypes.byref(v),
                                                    _stream_ptr(stream)), "cond_estimate")
    return v.value


def trmm_upper(a, b, stream=None):
    """multiply_upper_triangular(A, B) (cqrrpt.cc:23-36) -> k x n."""
    k, n = b.shape
    c = colmajor_empty(k, n)
    _lib.check(_lib.load().cqrrpt_gpu_trmm_upper(k, n, _p(a), _ld(a) if k else 1, _p(b), _ld(b) if k else 1, _p(c),
                                                 _ld(c) if k else 1, _stream_ptr(stream)), "trmm_upper")
    return c


def cholesky_qr(a, twice: bool = False, stream=None):
    """cholesky_qr / cholesky_qr2 (cqrrpt.cc:75-90) on a column-major CUDA
    tensor: Q overwrites ``a``; returns (R, failure_index) with R None on
    failure."""
    m, n = a.shape
    r = colmajor_empty(n, n)
    fi = _lib._i64(0)
    _lib.check(_lib.load().cqrrpt_gpu_cholesky_qr(m, n, _p(a), _ld(a) if n else 1, _p(r), _ld(r) if n else 1,
                                                  1 if twice else 0, ctypes.byref(fi), _stream_ptr(stream)),
               "cholesky_qr")
    return (r, 0) if fi.value == 0 else (None, fi.value)


def trtri_upper(r, stream=None):
    """X = triu(R)^{-1} (k x k), the inverse stage 2 applies in place of the
    reference's triangular solves (linalg.cc:486-500)."""
    k = r.shape[0]
    x = colmajor_empty(k, k)
    _lib.check(_lib.load().cqrrpt_gpu_trtri_upper(k, _p(r), _ld(r) if k else 1, _p(x), _ld(x) if k else 1,
                                                  _stream_ptr(stream)), "trtri_upper")
    return x


def launch_count(reset: bool = False) -> int:
    return int(_lib.load().cqrrpt_gpu_launch_count(1 if reset else 0))
