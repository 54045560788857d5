"""TEST INFRASTRUCTURE ONLY — numpy/ctypes front-end to the CPU oracle.

Two back-ends with the same Python surface:

* ``Oracle``    — oracle/_build/liboracle.so, the plain-C restatement of the
                  reference algorithm (oracle/cqrrpt_oracle.c).
* ``Reference`` — oracle/_ref/libcqrrpt_ref.so, the UNMODIFIED reference
                  library compiled from /root/reference/proj/src by
                  oracle/Makefile plus a C-ABI shim (oracle/ref_shim.cc).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline /
``--impl reference`` arm import this module, and only as the checker or the
timed CPU baseline. The product package never imports it.

All matrices cross this boundary as Fortran-ordered float64 numpy arrays
(column-major, like the reference's ``DenseMatrix``).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcqrrpt_ref.so")
UNIT_ROUNDOFF = 1.1102230246251565e-16

_c = ctypes
_i64, _u64, _f64, _i32 = _c.c_int64, _c.c_uint64, _c.c_double, _c.c_int32
_vp = _c.c_void_p


def build(ref: bool = True) -> None:
    """Compile the oracle (and the reference when /root/reference exists)."""
    target = ["all"] if ref else ["oracle"]
    subprocess.run(["make", "-s", "-C", HERE] + target, check=True)


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(_vp)


def _f(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def fnv_pivots(piv) -> str:
    """SURVEY §9 P11 pivot hash (FNV-style over int64 pivots)."""
    x = 1469598103934665603
    for v in np.asarray(piv, dtype=np.int64):
        x = ((x ^ (int(v) & 0xFFFFFFFFFFFFFFFF)) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{x:016x}"


@dataclass
class CqrrptResult:
    q: np.ndarray
    r: np.ndarray
    pivots: np.ndarray
    k0: int
    k: int
    cond_m_pre: float = 1.0
    truncation_ratio: float = 0.0
    flop_estimate: float = 0.0
    extra: dict = field(default_factory=dict)


class Oracle:
    """The C restatement (oracle/cqrrpt_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        self.lib = _c.CDLL(path)
        L = self.lib
        L.orc_rng_bits.restype = _u64
        L.orc_rng_bits.argtypes = [_u64, _u64]
        L.orc_mix_seed.restype = _u64
        L.orc_mix_seed.argtypes = [_u64, _u64]
        L.orc_rng_normal.restype = _f64
        L.orc_rng_normal.argtypes = [_u64, _u64]
        L.orc_dot.restype = _f64
        L.orc_flop_model.restype = _f64
        L.orc_flop_model.argtypes = [_i64, _i64, _i64, _i64, _f64]
        L.orc_sketch_rows_for.restype = _i64
        L.orc_sketch_rows_for.argtypes = [_f64, _i64]
        L.orc_rank_stage1.restype = _i64
        L.orc_rank_stage1.argtypes = [_i64, _i64, _vp, _i64, _f64]
        L.orc_spectral_norm_estimate.restype = _f64
        L.orc_spectral_norm_estimate.argtypes = [_i64, _i64, _vp, _i64, _vp]
        L.orc_inverse_norm_estimate.restype = _f64
        L.orc_inverse_norm_estimate.argtypes = [_i64, _vp, _i64, _vp]
        L.orc_cond_estimate.restype = _f64
        L.orc_cond_estimate.argtypes = [_i64, _vp, _i64, _c.c_int, _vp, _vp]

    # ---- generators -----------------------------------------------------
    def gen_gaussian(self, m, n, seed):
        out = np.empty((m, n), order="F")
        assert self.lib.orc_gen_gaussian(_i64(m), _i64(n), _u64(seed), _p(out)) == 0
        return out

    def gen_exact_rank(self, m, n, r, seed):
        out = np.empty((m, n), order="F")
        rc = self.lib.orc_gen_exact_rank(_i64(m), _i64(n), _i64(r), _u64(seed), _p(out))
        if rc:
            raise ValueError("gen_exact_rank: need 1 <= r <= min(m, n)")
        return out

    def gen_spectral(self, m, n, sigma, seed):
        sig = np.ascontiguousarray(sigma, dtype=np.float64)
        out = np.empty((m, n), order="F")
        rc = self.lib.orc_gen_spectral_list(_i64(m), _i64(n), _p(sig), _u64(seed), _p(out))
        if rc:
            raise ValueError("gen_spectral: bad spectrum")
        return out

    def gen_kahan(self, n, theta):
        out = np.empty((n, n), order="F")
        assert self.lib.orc_gen_kahan(_i64(n), _f64(theta), _p(out)) == 0
        return out

    def gaussian_block(self, m, n, stream_seed):
        """gaussian_block (testmat.cc:17-25) on a mixed stream seed."""
        out = np.empty((m, n), order="F")
        assert self.lib.orc_gaussian_block(_i64(m), _i64(n), _u64(stream_seed), _p(out)) == 0
        return out

    def gen_gaussian_rows(self, m, n, seed, r0, r1):
        """Rows [r0, r1) of gen_gaussian(m, n, seed) (testmat.cc:141-143),
        bitwise, without materialising the whole matrix."""
        out = np.empty((r1 - r0, n), order="F")
        rc = self.lib.orc_gen_gaussian_rows(_i64(m), _i64(n), _u64(seed), _i64(r0), _i64(r1), _p(out),
                                            _i64(max(r1 - r0, 1)))
        if rc:
            raise ValueError("gen_gaussian_rows: bad row range")
        return out

    def c5_column_factors(self, n, span=8.0, seed=0):
        """C5 column factors 10^(-span*pi[j]/(n-1)); a block
        scaled by them equals the same block of c5_scale_columns bitwise."""
        f = np.empty(n)
        self.lib.orc_c5_column_factors(_i64(n), _f64(span), _u64(seed), _p(f))
        return f

    def c5_scale_columns(self, a, span=8.0, seed=0):
        a = _f(a).copy(order="F")
        perm = np.empty(a.shape[1], dtype=np.int64)
        self.lib.orc_c5_scale_columns(_i64(a.shape[0]), _i64(a.shape[1]), _i64(a.shape[0]),
                                      _f64(span), _u64(seed), _p(a), _p(perm))
        return a, perm

    # ---- rng -------------------------------------------------------------
    def rng_bits(self, seed, ctr):
        return int(self.lib.orc_rng_bits(seed, ctr))

    def mix_seed(self, seed, salt):
        return int(self.lib.orc_mix_seed(seed, salt))

    # ---- sketch ----------------------------------------------------------
    def saso_sample(self, d, m, nnz, seed, c0=0):
        rows = np.empty(m * nnz, dtype=np.int64)
        vals = np.empty(m * nnz, dtype=np.float64)
        rc = self.lib.orc_saso_sample(_i64(d), _i64(c0), _i64(m), _i64(nnz), _u64(seed), _p(rows), _p(vals))
        if rc:
            raise ValueError("sample_sketch: SASO needs d >= 1 and 1 <= nnz <= d")
        return rows.reshape(m, nnz), vals.reshape(m, nnz)

    def gaussian_sample(self, d, m, seed, c0=0):
        """sketch.cc:62-72: the Gaussian operator's columns c0..c0+m-1 (d x m)."""
        s = np.empty((d, m), order="F")
        assert self.lib.orc_gaussian_sample(_i64(d), _i64(m), _u64(seed), _i64(c0), _p(s)) == 0
        return s

    def gaussian_apply(self, d, a, seed, c0=0):
        """apply for the Gaussian family (sketch.cc:124-127: matmul(S, M)); the
        product is formed by numpy (the reference's matmul order is not
        restated: the device GEMM is compared with a rounding tolerance)."""
        a = _f(a)
        return np.asfortranarray(self.gaussian_sample(d, a.shape[0], seed, c0) @ a)

    def srft_apply(self, d, a, seed):
        """SRFT family apply (sketch.cc:100-119, 147-166), bit-exact."""
        a = _f(a)
        m, n = a.shape
        out = np.zeros((d, n), order="F")
        rc = self.lib.orc_srft_apply(_i64(d), _i64(m), _i64(n), _u64(seed), _p(a), _i64(m), _p(out), _i64(d))
        if rc:
            raise ValueError("srft: needs 1 <= d <= m")
        return out

    def saso_apply(self, d, a, nnz, seed, c0=0, out=None):
        a = _f(a)
        m, n = a.shape
        if out is None:
            out = np.zeros((d, n), order="F")
        rc = self.lib.orc_saso_apply(_i64(d), _i64(m), _i64(n), _i64(nnz), _u64(seed), _i64(c0),
                                     _p(a), _i64(m), _p(out), _i64(d))
        if rc:
            raise ValueError("apply: invalid SASO parameters")
        return out

    # ---- factorizations --------------------------------------------------
    def qrcp(self, a, rank_tol=-1.0, gaps=False):
        a = _f(a)
        rows, n = a.shape
        kmax = min(rows, n)
        r = np.zeros(kmax * n)
        piv = np.empty(n, dtype=np.int64)
        rank = _i64()
        g = np.full(kmax, np.inf) if gaps else None
        rc = self.lib.orc_qrcp_maxnorm(_i64(rows), _i64(n), _p(a), _i64(rows), _f64(rank_tol),
                                       _p(r), _p(piv), _c.byref(rank), _p(g))
        if rc:
            raise ValueError("qrcp_maxnorm: need at least one row")
        k = rank.value
        R = r[: k * n].reshape((k, n), order="F")
        return (R, piv, k, g) if gaps else (R, piv, k)

    def rank_stage1(self, r, u=UNIT_ROUNDOFF):
        r = _f(r)
        return int(self.lib.orc_rank_stage1(r.shape[0], r.shape[1], _p(r), max(r.shape[0], 1), u))

    def cholesky(self, g):
        g = _f(g)
        n = g.shape[0]
        out = np.zeros(max(n * n, 1))
        fi = _i64()
        self.lib.orc_cholesky(_i64(n), _p(g), _i64(n), _p(out), _c.byref(fi))
        j = n if fi.value == 0 else fi.value - 1
        return out[: j * j].reshape((j, j), order="F"), fi.value

    def trsm_right(self, b, r):
        b, r = _f(b), _f(r)
        x = np.empty_like(b, order="F")
        rc = self.lib.orc_trsm_right(_i64(b.shape[0]), _i64(b.shape[1]), _p(b), _i64(b.shape[0]),
                                     _p(r), _i64(r.shape[0]), _p(x), _i64(b.shape[0]))
        if rc == -2:
            raise ZeroDivisionError("trsm_right: singular preconditioner (zero diagonal)")
        return x

    def gram(self, a):
        a = _f(a)
        g = np.empty((a.shape[1], a.shape[1]), order="F")
        self.lib.orc_gram(_i64(a.shape[0]), _i64(a.shape[1]), _p(a), _i64(a.shape[0]), _p(g))
        return g

    def spectral_norm_estimate(self, a):
        a = _f(a)
        conv = _c.c_int()
        v = self.lib.orc_spectral_norm_estimate(a.shape[0], a.shape[1], _p(a), max(a.shape[0], 1), _c.byref(conv))
        return v, bool(conv.value)

    def inverse_norm_estimate(self, r):
        r = _f(r)
        conv = _c.c_int()
        v = self.lib.orc_inverse_norm_estimate(r.shape[0], _p(r), max(r.shape[0], 1), _c.byref(conv))
        return v, bool(conv.value)

    def cond_estimate(self, x, method):
        x = _f(x)
        up, conv = _c.c_int(), _c.c_int()
        v = self.lib.orc_cond_estimate(x.shape[0], _p(x), max(x.shape[0], 1), method, _c.byref(up), _c.byref(conv))
        return v, bool(up.value), bool(conv.value)

    def rank_stage2(self, m_k0, a_sk, eps_tol=1e-4, method=2, u=UNIT_ROUNDOFF):
        class Info(_c.Structure):
            _fields_ = [("rank", _i64), ("k0_final", _i64), ("retries", _i32), ("cond_at_rank", _f64),
                        ("n_probes", _i32), ("probes", _i64 * 64), ("probe_raw", _f64 * 64)]
        m_k0, a_sk = _f(m_k0), _f(a_sk)
        m, k0 = m_k0.shape
        info = Info()
        m_pre = np.zeros((m, k0), order="F")
        r_pre = np.zeros(k0 * k0)
        rc = self.lib.orc_rank_stage2(_i64(m), _i64(k0), _p(m_k0), _i64(m), _p(a_sk), _i64(k0),
                                      _f64(eps_tol), _f64(u), _c.c_int(method), _p(m_pre), _p(r_pre),
                                      _c.byref(info))
        if rc == -2:
            raise ZeroDivisionError("trsm_right: singular preconditioner")
        if rc:
            raise ValueError("rank_stage2: requires k0 >= 1")
        k = info.rank
        return dict(rank=k, k0_final=info.k0_final, retries=info.retries, cond_at_rank=info.cond_at_rank,
                    probes=[info.probes[i] for i in range(info.n_probes)],
                    probe_raw=[info.probe_raw[i] for i in range(info.n_probes)],
                    r_pre=r_pre[: k * k].reshape((k, k), order="F"),
                    m_pre=m_pre[:, : info.k0_final])

    def multiply_upper_triangular(self, a, b):
        a, b = _f(a), _f(b)
        k, n = b.shape
        c = np.zeros((k, n), order="F")
        self.lib.orc_multiply_upper_triangular(_i64(k), _i64(n), _p(a), _i64(k), _p(b), _i64(k), _p(c))
        return c

    def cholesky_qr(self, a, twice=False):
        """cholesky_qr / cholesky_qr2 (cqrrpt.cc:75-90) composed from the
        restated gram, cholesky, trsm_right and multiply_upper_triangular.
        Returns (q, r, failure_index); q, r are None on failure."""
        a = _f(a)
        if a.shape[0] < a.shape[1]:
            raise ValueError("cholesky_qr: requires rows >= cols")
        r1, fi = self.cholesky(self.gram(a))
        if fi:
            return None, None, fi
        q1 = self.trsm_right(a, r1)
        if not twice:
            return q1, r1, 0
        r2, fi = self.cholesky(self.gram(q1))
        if fi:
            return None, None, fi
        return self.trsm_right(q1, r2), self.multiply_upper_triangular(r2, r1), 0

    def flop_model(self, m, n, k, d, c_sk=0.0):
        v = self.lib.orc_flop_model(m, n, k, d, c_sk)
        if v < 0:
            raise ValueError("flop_model: requires 0 <= k <= min(d, n)")
        return v

    def sketch_rows_for(self, gamma, n):
        return int(self.lib.orc_sketch_rows_for(gamma, n))

    def cqrrpt(self, a, gamma=1.25, nnz=4, eps_tol=1e-4, seed=0, method=2, stage1=True,
               want_sketch=False) -> CqrrptResult:
        a = _f(a)
        m, n = a.shape
        q = np.zeros(max(m * n, 1))
        r = np.zeros(max(n * n, 1))
        piv = np.zeros(n, dtype=np.int64)
        k0, k = _i64(), _i64()
        diag = np.zeros(8)
        d = self.sketch_rows_for(gamma, n) if n else 0
        msk = np.zeros((d, n), order="F") if want_sketch else None
        rsk = np.zeros(max(min(d, n) * n, 1)) if want_sketch else None
        rc = self.lib.orc_cqrrpt(_i64(m), _i64(n), _p(a), _i64(m), _f64(gamma), _i64(nnz), _f64(eps_tol),
                                 _u64(seed), _c.c_int(method), _c.c_int(int(stage1)), _p(q), _p(r), _p(piv),
                                 _c.byref(k0), _c.byref(k), _p(diag), _p(msk), _p(rsk))
        if rc == -1:
            raise ValueError("cqrrpt: invalid argument")
        if rc == -2:
            raise ZeroDivisionError("cqrrpt: singular preconditioner")
        kk = k.value
        res = CqrrptResult(q=q[: m * kk].reshape((m, kk), order="F"),
                           r=r[: kk * n].reshape((kk, n), order="F"), pivots=piv, k0=k0.value, k=kk,
                           cond_m_pre=diag[0], truncation_ratio=diag[1], flop_estimate=diag[2],
                           extra=dict(k_sk=int(diag[3]), d=int(diag[4]), retries=int(diag[5]),
                                      k0_final=int(diag[6])))
        if want_sketch:
            ksk = int(diag[3])
            res.extra["m_sk"] = msk
            res.extra["r_sk"] = rsk[: ksk * n].reshape((ksk, n), order="F")
        return res

    def validate(self, a, q, r, pivots):
        a, q, r = _f(a), _f(q), _f(r)
        m, n = a.shape
        k = q.shape[1]
        piv = np.ascontiguousarray(pivots, dtype=np.int64)
        orth, orth_f, recon, below = _f64(), _f64(), _f64(), _f64()
        rc = self.lib.orc_validate(_i64(m), _i64(n), _i64(k), _p(a), _i64(m), _p(q), _i64(max(m, 1)),
                                   _p(r), _i64(max(k, 1)), _p(piv), _c.byref(orth), _c.byref(orth_f),
                                   _c.byref(recon), _c.byref(below))
        return dict(pivots_valid=(rc == 0), orth_loss=orth.value, orth_fro=orth_f.value,
                    recon_rel=recon.value, max_below_diag=below.value)


class Reference:
    """The unmodified reference library through oracle/ref_shim.cc."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"reference oracle not built: {path} (run make -C oracle ref)")
        self.lib = _c.CDLL(path)
        L = self.lib
        L.ref_rng_bits.restype = _u64
        L.ref_rng_bits.argtypes = [_u64, _u64]
        L.ref_mix_seed.restype = _u64
        L.ref_mix_seed.argtypes = [_u64, _u64]
        L.ref_rng_normal.restype = _f64
        L.ref_rng_normal.argtypes = [_u64, _u64]
        L.ref_flop_model.restype = _f64
        L.ref_flop_model.argtypes = [_i64, _i64, _i64, _i64, _f64]
        L.ref_sketch_rows_for.restype = _i64
        L.ref_sketch_rows_for.argtypes = [_f64, _i64]
        L.ref_sketch_flops_saso.restype = _f64
        L.ref_sketch_flops_saso.argtypes = [_i64, _i64, _i64, _i64]

    def num_threads(self):
        return int(self.lib.ref_num_threads())

    def set_threads(self, n):
        self.lib.ref_set_threads(_c.c_int(n))

    def gen_gaussian(self, m, n, seed):
        out = np.empty((m, n), order="F")
        assert self.lib.ref_gen_gaussian(_i64(m), _i64(n), _u64(seed), _p(out)) == 0
        return out

    def gen_exact_rank(self, m, n, r, seed):
        out = np.empty((m, n), order="F")
        if self.lib.ref_gen_exact_rank(_i64(m), _i64(n), _i64(r), _u64(seed), _p(out)):
            raise ValueError("gen_exact_rank")
        return out

    def gen_spectral(self, m, n, sigma, seed):
        sig = np.ascontiguousarray(sigma, dtype=np.float64)
        out = np.empty((m, n), order="F")
        if self.lib.ref_gen_spectral_list(_i64(m), _i64(n), _p(sig), _u64(seed), _p(out)):
            raise ValueError("gen_spectral")
        return out

    def gen_spectral_poly(self, m, n, cond, seed):
        out = np.empty((m, n), order="F")
        if self.lib.ref_gen_spectral_poly(_i64(m), _i64(n), _f64(cond), _u64(seed), _p(out)):
            raise ValueError("gen_spectral")
        return out

    def gen_kahan(self, n, theta):
        out = np.empty((n, n), order="F")
        assert self.lib.ref_gen_kahan(_i64(n), _f64(theta), _p(out)) == 0
        return out

    def rng_bits(self, seed, ctr):
        return int(self.lib.ref_rng_bits(seed, ctr))

    def mix_seed(self, seed, salt):
        return int(self.lib.ref_mix_seed(seed, salt))

    def saso_sample(self, d, m, nnz, seed):
        rows = np.empty(m * nnz, dtype=np.int64)
        vals = np.empty(m * nnz, dtype=np.float64)
        if self.lib.ref_saso_sample(_i64(d), _i64(m), _i64(nnz), _u64(seed), _p(rows), _p(vals)):
            raise ValueError("sample_sketch")
        return rows.reshape(m, nnz), vals.reshape(m, nnz)

    def saso_apply(self, d, a, nnz, seed):
        a = _f(a)
        out = np.empty((d, a.shape[1]), order="F")
        if self.lib.ref_saso_apply(_i64(d), _i64(a.shape[0]), _i64(a.shape[1]), _i64(nnz), _u64(seed), _p(a), _p(out)):
            raise ValueError("apply")
        return out

    def gaussian_sketch_apply(self, d, a, seed):
        a = _f(a)
        out = np.empty((d, a.shape[1]), order="F")
        if self.lib.ref_gaussian_sketch_apply(_i64(d), _i64(a.shape[0]), _i64(a.shape[1]), _u64(seed), _p(a), _p(out)):
            raise ValueError("apply")
        return out

    def qrcp(self, a, rank_tol=-1.0):
        a = _f(a)
        rows, n = a.shape
        r = np.zeros(max(min(rows, n) * n, 1))
        piv = np.empty(n, dtype=np.int64)
        rank = _i64()
        if self.lib.ref_qrcp_maxnorm(_i64(rows), _i64(n), _p(a), _f64(rank_tol), _p(r), _p(piv), _c.byref(rank)):
            raise ValueError("qrcp_maxnorm")
        k = rank.value
        return r[: k * n].reshape((k, n), order="F"), piv, k

    def rank_stage1(self, r):
        r = _f(r)
        k0 = _i64()
        self.lib.ref_rank_stage1(_i64(r.shape[0]), _i64(r.shape[1]), _p(r), _c.byref(k0))
        return k0.value

    def cholesky(self, g):
        g = _f(g)
        n = g.shape[0]
        out = np.zeros(max(n * n, 1))
        fi = _i64()
        self.lib.ref_cholesky(_i64(n), _p(g), _p(out), _c.byref(fi))
        j = n if fi.value == 0 else fi.value - 1
        return out[: j * j].reshape((j, j), order="F"), fi.value

    def trsm_right(self, b, r):
        b, r = _f(b), _f(r)
        x = np.empty_like(b, order="F")
        rc = self.lib.ref_trsm_right(_i64(b.shape[0]), _i64(b.shape[1]), _p(b), _p(r), _p(x))
        if rc == -2:
            raise ZeroDivisionError("trsm_right: singular preconditioner (zero diagonal)")
        return x

    def gram(self, a):
        a = _f(a)
        g = np.empty((a.shape[1], a.shape[1]), order="F")
        self.lib.ref_gram(_i64(a.shape[0]), _i64(a.shape[1]), _p(a), _p(g))
        return g

    def mm_write(self, path, a, coordinate=False):
        a = _f(a)
        rc = self.lib.ref_mm_write(path.encode(), _i64(a.shape[0]), _i64(a.shape[1]), _p(a),
                                   _i32(1 if coordinate else 0))
        if rc:
            raise RuntimeError(f"ref_mm_write failed ({rc})")

    def mm_read(self, path):
        m, n = _i64(), _i64()
        rc = self.lib.ref_mm_read(path.encode(), _c.byref(m), _c.byref(n), None)
        if rc:
            raise RuntimeError(f"ref_mm_read failed ({rc})")
        out = np.zeros((m.value, n.value), order="F")
        self.lib.ref_mm_read(path.encode(), _c.byref(m), _c.byref(n), _p(out))
        return out

    def srft_sketch_apply(self, d, a, seed):
        a = _f(a)
        m, n = a.shape
        out = np.zeros((d, n), order="F")
        rc = self.lib.ref_srft_sketch_apply(_i64(d), _i64(m), _i64(n), _u64(seed), _p(a), _p(out))
        if rc:
            raise ValueError(f"ref_srft_sketch_apply failed ({rc})")
        return out

    def cholesky_qr(self, a, twice=False):
        a = _f(a)
        m, n = a.shape
        q = np.zeros((m, n), order="F")
        r = np.zeros((n, n), order="F")
        fi = _i64()
        rc = self.lib.ref_cholesky_qr(_i64(m), _i64(n), _p(a), _i32(1 if twice else 0), _p(q), _p(r),
                                      _c.byref(fi))
        if rc == -1:
            raise ValueError("cholesky_qr: requires rows >= cols")
        if rc:
            raise RuntimeError(f"ref_cholesky_qr failed ({rc})")
        return (q, r, 0) if fi.value == 0 else (None, None, fi.value)

    def spectral_norm_estimate(self, a):
        a = _f(a)
        v, c = _f64(), _i32()
        self.lib.ref_spectral_norm_estimate(_i64(a.shape[0]), _i64(a.shape[1]), _p(a), _c.byref(v), _c.byref(c))
        return v.value, bool(c.value)

    def inverse_norm_estimate(self, r):
        r = _f(r)
        v, c = _f64(), _i32()
        self.lib.ref_inverse_norm_estimate(_i64(r.shape[0]), _p(r), _c.byref(v), _c.byref(c))
        return v.value, bool(c.value)

    def cond_estimate(self, x, method):
        x = _f(x)
        v, up, c = _f64(), _i32(), _i32()
        self.lib.ref_cond_estimate(_i64(x.shape[0]), _p(x), _i32(method), _c.byref(v), _c.byref(up), _c.byref(c))
        return v.value, bool(up.value), bool(c.value)

    def rank_stage2(self, m_k0, a_sk, eps_tol=1e-4, method=2):
        m_k0, a_sk = _f(m_k0), _f(a_sk)
        m, k0 = m_k0.shape
        rank, k0f = _i64(), _i64()
        retries = _i32()
        cond = _f64()
        r_pre = np.zeros(max(k0 * k0, 1))
        m_pre = np.zeros(max(m * k0, 1))
        rc = self.lib.ref_rank_stage2(_i64(m), _i64(k0), _p(m_k0), _p(a_sk), _f64(eps_tol), _i32(method),
                                      _c.byref(rank), _c.byref(k0f), _c.byref(retries), _c.byref(cond),
                                      _p(r_pre), _p(m_pre))
        if rc:
            raise ValueError(f"rank_stage2 rc={rc}")
        k, kf = rank.value, k0f.value
        return dict(rank=k, k0_final=kf, retries=retries.value, cond_at_rank=cond.value,
                    r_pre=r_pre[: k * k].reshape((k, k), order="F"),
                    m_pre=m_pre[: m * kf].reshape((m, kf), order="F"))

    def flop_model(self, m, n, k, d, c_sk=0.0):
        v = self.lib.ref_flop_model(m, n, k, d, c_sk)
        if v < 0:
            raise ValueError("flop_model")
        return v

    def sketch_rows_for(self, gamma, n):
        return int(self.lib.ref_sketch_rows_for(gamma, n))

    def cqrrpt(self, a, gamma=1.25, nnz=4, eps_tol=1e-4, seed=0, method=2, stage1=True,
               validate=False) -> CqrrptResult:
        a = _f(a)
        m, n = a.shape
        q = np.zeros(max(m * n, 1))
        r = np.zeros(max(n * n, 1))
        piv = np.zeros(n, dtype=np.int64)
        k0, k = _i64(), _i64()
        diag, tim, val = np.zeros(4), np.zeros(7), np.zeros(3)
        rc = self.lib.ref_cqrrpt(_i64(m), _i64(n), _p(a), _f64(gamma), _i64(nnz), _f64(eps_tol), _u64(seed),
                                 _i32(method), _i32(int(stage1)), _i32(int(validate)), _p(q), _p(r), _p(piv),
                                 _c.byref(k0), _c.byref(k), _p(diag), _p(tim), _p(val))
        if rc == -1:
            raise ValueError("cqrrpt: invalid argument")
        if rc:
            raise RuntimeError(f"cqrrpt rc={rc}")
        kk = k.value
        names = ["sketch", "qrcp", "rank_select", "precondition", "cholesky_qr", "undo", "total"]
        return CqrrptResult(q=q[: m * kk].reshape((m, kk), order="F"),
                            r=r[: kk * n].reshape((kk, n), order="F"), pivots=piv, k0=k0.value, k=kk,
                            cond_m_pre=diag[0], truncation_ratio=diag[1], flop_estimate=diag[2],
                            extra=dict(timings=dict(zip(names, tim.tolist())),
                                       validation=(dict(pass_=diag[3] == 1.0, orth_loss=val[0], recon_rel=val[1],
                                                        max_below_diag=val[2]) if validate else None)))

    def validate(self, a, q, r, pivots, tol=1.0):
        a, q, r = _f(a), _f(q), _f(r)
        m, n = a.shape
        k = q.shape[1]
        piv = np.ascontiguousarray(pivots, dtype=np.int64)
        orth, recon, below = _f64(), _f64(), _f64()
        ok = _i32()
        self.lib.ref_validate(_i64(m), _i64(n), _i64(k), _p(a), _p(q), _p(r), _p(piv), _f64(tol),
                              _c.byref(orth), _c.byref(recon), _c.byref(below), _c.byref(ok))
        return dict(orth_loss=orth.value, recon_rel=recon.value, max_below_diag=below.value, pass_=bool(ok.value))
