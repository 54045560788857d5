"""Python mirror of the reference's CQRRPT interface, on the sm_100a library.

Reference interface (/root/reference/proj/include/cqrrpt/cqrrpt.hh):

    struct CqrrptConfig   { gamma, family, nnz_per_col, eps_tol, cond_method,
                            stage1_enabled, seed, measure_distortion,
                            validate_output }                       (:92-102)
    struct PhaseTimings   { sketch, qrcp, rank_select, precondition,
                            cholesky_qr, undo, total }              (:104-112)
    struct CqrrptDiagnostics { cond_m_pre, truncation_ratio,
                            flop_estimate, timings, validation }    (:114-122)
    struct CqrrptOutput   { factorization (PivotedQR), k0, k, diagnostics } (:124-129)
    CqrrptOutput cqrrpt(const DenseMatrix &m, const CqrrptConfig &cfg = {}); (:140)
    int64_t sketch_rows_for(double gamma, int64_t n);                (:143)
    double flop_model(m, n, k, d, c_sk);                             (:150)

Same names, argument meaning and error behaviour: invalid configurations
raise ``InvalidArgument`` (a ``ValueError``, the reference's
std::invalid_argument), a zero diagonal raises ``DomainError``. Every call
runs on the GPU through the C ABI (include/cqrrpt_gpu.h); there is no CPU
path. Matrices are column-major like ``DenseMatrix``: a host ``numpy`` array
(any order; copied to the device) or a CUDA ``torch`` tensor whose storage is
column-major (stride ``(1, lda)``).
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import DomainError, InvalidArgument  # noqa: F401  (re-exported)

UNIT_ROUNDOFF = 1.1102230246251565e-16  # cqrrpt.hh:14


class SketchFamily(enum.Enum):  # sketch.hh:24
    gaussian = 0
    saso = 1
    srft = 2


class CondMethod(enum.IntEnum):  # cqrrpt.hh:61
    diag_ratio = 0
    krylov_bounds = 1
    identity_deviation = 2


@dataclass
class CqrrptConfig:  # cqrrpt.hh:92-102
    gamma: float = 1.25
    family: SketchFamily = SketchFamily.saso
    nnz_per_col: int = 4
    eps_tol: float = 1e-4
    cond_method: CondMethod = CondMethod.identity_deviation
    stage1_enabled: bool = True
    seed: int = 0
    measure_distortion: bool = False
    validate_output: bool = True


@dataclass
class PhaseTimings:  # cqrrpt.hh:104-112 (seconds, CUDA events)
    sketch: float = 0.0
    qrcp: float = 0.0
    rank_select: float = 0.0
    precondition: float = 0.0
    cholesky_qr: float = 0.0
    undo: float = 0.0
    total: float = 0.0
    communication: float = 0.0


@dataclass
class ValidationReport:  # qrcp.hh:53-60 (+ the BASELINE Frobenius metric)
    orth_loss: float = 0.0
    orth_loss_fro: float = 0.0
    recon_rel: float = 0.0
    max_below_diag: float = 0.0
    pivots_valid: bool = False
    diag_nonincreasing: bool = False
    passed: bool = False


@dataclass
class CqrrptDiagnostics:  # cqrrpt.hh:114-122
    distortion: Optional[float] = None
    effective_distortion: Optional[float] = None
    cond_m_pre: float = 1.0
    truncation_ratio: float = 0.0
    flop_estimate: float = 0.0
    timings: PhaseTimings = field(default_factory=PhaseTimings)
    validation: Optional[ValidationReport] = None
    # device-path extras
    d: int = 0
    k_sk: int = 0
    k0_final: int = 0
    retries: int = 0
    stage2_exact: bool = False
    cond_upper_bound: float = 0.0


@dataclass
class PivotedQR:  # qrcp.hh:19-24
    q: object
    r: object
    pivots: np.ndarray
    rank: int = 0


@dataclass
class CqrrptOutput:  # cqrrpt.hh:124-129
    factorization: PivotedQR
    k0: int = 0
    k: int = 0
    diagnostics: CqrrptDiagnostics = field(default_factory=CqrrptDiagnostics)


def sketch_rows_for(gamma: float, n: int) -> int:  # cqrrpt.cc:211-213
    return int(_lib.load().cqrrpt_gpu_sketch_rows(float(gamma), int(n)))


def flop_model(m: int, n: int, k: int, d: int, c_sk: float) -> float:  # cqrrpt.cc:330-338
    v = _lib.load().cqrrpt_gpu_flop_model(int(m), int(n), int(k), int(d), float(c_sk))
    if v < 0:
        raise InvalidArgument("flop_model: requires 0 <= k <= min(d, n)")
    return v


def sketch_flops_saso(nnz: int, m: int, n_cols: int) -> float:  # sketch.cc:216-217
    return 2.0 * nnz * m * n_cols


def check_config(cfg: CqrrptConfig) -> None:  # cqrrpt.cc:38-42
    if cfg.gamma < 1.0:
        raise InvalidArgument("cqrrpt: gamma must be >= 1")
    if not (cfg.eps_tol > UNIT_ROUNDOFF):
        raise InvalidArgument("cqrrpt: eps_tol must exceed the unit roundoff")


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2311_08316_b200 needs a CUDA device (no CPU fallback)")
    return torch


def colmajor_empty(m: int, n: int, device=None, dtype=None, pad_to: int = 1):
    """Uninitialised column-major (m x n) CUDA tensor (stride (1, ld))."""
    torch = _torch()
    ld = max(1, -(-m // pad_to) * pad_to)
    store = torch.empty((n, ld), dtype=dtype or torch.float64, device=device or "cuda")
    return store[:, :m].t() if ld != m else store.t()


def to_device_colmajor(a, device=None):
    """Host/device array -> column-major float64 CUDA tensor. Always a fresh
    copy, also when ``a`` already is a column-major float64 CUDA tensor (the
    callers write Q into it in place)."""
    torch = _torch()
    if isinstance(a, torch.Tensor):
        dev = device or (a.device if a.is_cuda else "cuda")
        m, n = a.shape
        out = colmajor_empty(m, n, device=dev)
        out.copy_(a)
        return out
    arr = np.asarray(a, dtype=np.float64)
    host = torch.from_numpy(np.ascontiguousarray(arr.T)).pin_memory()
    return host.to(device or "cuda", non_blocking=True).t()


def release_workspace() -> None:
    """Free the library's cached device workspaces of the calling thread
    (cqrrpt_gpu_release_workspace)."""
    _lib.load().cqrrpt_gpu_release_workspace()


def _ld(t) -> int:
    if t.dim() != 2:
        raise InvalidArgument("expected a matrix")
    m, n = t.shape
    s0, s1 = t.stride()
    if n <= 1 and s0 == 1:
        return max(m, 1)
    if s0 != 1 or s1 < max(m, 1):
        raise InvalidArgument("matrix must be column-major (stride (1, ld >= rows))")
    return s1


def _stream_ptr(stream, device=None) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return s.cuda_stream


class Comm:
    """NCCL communicator of the library (cqrrpt_gpu_comm_*), one per rank."""

    def __init__(self, handle: int, nranks: int, rank: int):
        self.handle, self.nranks, self.rank = handle, nranks, rank

    @classmethod
    def from_torch_distributed(cls, group=None) -> "Comm":
        import torch.distributed as dist
        L = _lib.load()
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [None]
        if rank == 0:
            buf = ctypes.create_string_buffer(128)
            _lib.check(L.cqrrpt_gpu_comm_unique_id(buf), "comm_unique_id")
            obj[0] = bytes(buf.raw)
        dist.broadcast_object_list(obj, src=0, group=group)
        h = _lib._vp()
        _lib.check(L.cqrrpt_gpu_comm_init(world, rank, obj[0], ctypes.byref(h)), "comm_init")
        return cls(h.value, world, rank)

    def allreduce(self, t, stream=None) -> None:
        _lib.check(_lib.load().cqrrpt_gpu_comm_allreduce(self.handle, t.data_ptr(), t.numel(), _stream_ptr(stream)),
                   "comm_allreduce")

    def close(self) -> None:
        if self.handle:
            _lib.load().cqrrpt_gpu_comm_destroy(self.handle)
            self.handle = 0


@dataclass
class DeviceResult:
    """Raw outputs of one cqrrpt_gpu_dgeqpt call (device tensors)."""
    r: object          # k x n column-major view (torch, cuda)
    pivots: object     # int64 n (torch, cuda)
    k: int
    k0: int
    ctx: _lib.Ctx


def dgeqpt(a, d_factor: float = 1.25, nnz: int = 4, seed: int = 0, eps_tol: float = 1e-4,
           cond_method: int = CondMethod.identity_deviation, stage1: bool = True, exact_stage2: bool = False,
           diagnostics: bool = False, timings: bool = False, stream=None, comm: Optional[Comm] = None,
           global_row_offset: int = 0, r_out=None, j_out=None, allreduce=None, nranks: int = 1,
           rank: int = 0, fast_sketch: bool = False, sketch_family: str = "saso",
           wavefront: bool = False) -> DeviceResult:
    """The north-star entry point on a column-major CUDA tensor ``a``
    (m_local x n). Q overwrites ``a[:, :k]`` in place; R (k x n) and the
    0-based pivots are returned as device tensors.

    Multi-rank: pass ``comm`` (NCCL, cqrrpt_gpu_comm_*) or ``allreduce`` — a
    Python callable ``(ptr, count, stream_ptr) -> None`` that sum-allreduces
    ``count`` doubles in place — together with ``nranks``/``rank`` and this
    rank's ``global_row_offset``.

    ``sketch_family``: "saso" (default, ``nnz`` nonzeros per column),
    "gaussian" (dense N(0, 1/d) operator) or "srft" (subsampled randomized
    Walsh-Hadamard, single rank) -- SketchFamily; ``nnz`` is SASO-only.

    ``fast_sketch``: allow a c-split sketch (CQRRPT_GPU_FAST_SKETCH) that
    fills the GPU when n is small; deterministic, but J then matches the
    reference only away from near-ties (the default sketch is bit-identical).

    ``wavefront`` (one rank, CQRRPT_GPU_WAVEFRONT): precondition, Gram,
    Cholesky and Q run as the 128-column wavefront dgeqpt_host uses (Q
    speculated on k = k0; if stage 2 truncates, ``a[:, k:k0]`` is left with
    speculative columns). Slower on the device alone; gives dgeqpt_host's
    default bits (whole passes: a different Gram slicing, so Q and R agree to
    rounding, J and k are the same)."""
    torch = _torch()
    L = _lib.load()
    m, n = a.shape
    if a.dtype != torch.float64 or not a.is_cuda:
        raise InvalidArgument("a must be a float64 CUDA tensor")
    lda = _ld(a)
    if r_out is None:
        r_out = colmajor_empty(n, n, device=a.device)
    ldr = _ld(r_out) if n > 0 else 1
    if j_out is None:
        j_out = torch.empty(max(n, 1), dtype=torch.int64, device=a.device)
    ctx = _lib.new_ctx()
    ctx.stream = _stream_ptr(stream, a.device)
    ctx.cond_method = int(cond_method)
    flags = 0
    if not stage1:
        flags |= _lib.F_NO_STAGE1
    if exact_stage2:
        flags |= _lib.F_EXACT_STAGE2
    if diagnostics:
        flags |= _lib.F_DIAGNOSTICS
    if timings:
        flags |= _lib.F_TIMINGS
    if fast_sketch:
        flags |= _lib.F_FAST_SKETCH
    if wavefront:
        flags |= _lib.F_WAVEFRONT
    ctx.flags = flags
    families = {"saso": _lib.SKETCH_SASO, "gaussian": _lib.SKETCH_GAUSSIAN, "srft": _lib.SKETCH_SRFT}
    if sketch_family not in families:
        raise InvalidArgument(f"sketch_family must be one of {sorted(families)}")
    ctx.sketch_family = families[sketch_family]
    cb = None
    if comm is not None:
        ctx.comm = comm.handle
        ctx.nranks = comm.nranks
        ctx.rank = comm.rank
        ctx.global_row_offset = int(global_row_offset)
    elif allreduce is not None:
        def _ar(buf, count, st, user):
            try:
                allreduce(ctypes.cast(buf, ctypes.c_void_p).value, int(count), st)
                return 0
            except Exception:  # reported to the library as a failed collective
                return 1
        cb = _lib.ALLREDUCE_FN(_ar)  # kept alive for the duration of the call
        ctx.allreduce = cb
        ctx.nranks = int(nranks)
        ctx.rank = int(rank)
        ctx.global_row_offset = int(global_row_offset)
    k, k0 = _lib._i64(), _lib._i64()
    with torch.cuda.device(a.device):  # the library works on the current device
        rc = L.cqrrpt_gpu_dgeqpt(m, n, a.data_ptr() if a.numel() else None, lda, float(d_factor), int(nnz),
                                 int(seed), float(eps_tol), r_out.data_ptr() if n else None, ldr, j_out.data_ptr(),
                                 ctypes.byref(k), ctypes.byref(k0), ctypes.byref(ctx))
    _lib.check(rc, "cqrrpt_gpu_dgeqpt")
    return DeviceResult(r=r_out[: k.value, :], pivots=j_out[:n], k=k.value, k0=k0.value, ctx=ctx)


def _diagnostics_from(ctx: _lib.Ctx) -> CqrrptDiagnostics:
    t = [v / 1e3 for v in ctx.timings_ms]
    return CqrrptDiagnostics(
        cond_m_pre=ctx.cond_m_pre, truncation_ratio=ctx.truncation_ratio, flop_estimate=ctx.flop_estimate,
        timings=PhaseTimings(sketch=t[0], qrcp=t[1], rank_select=t[2], precondition=t[3], cholesky_qr=t[4],
                             undo=t[5], total=t[6], communication=t[7]),
        d=ctx.d, k_sk=ctx.k_sk, k0_final=ctx.k0_final, retries=ctx.retries, stage2_exact=bool(ctx.stage2_exact),
        cond_upper_bound=ctx.cond_upper_bound)


@dataclass
class HostResult:
    """Outputs of one cqrrpt_gpu_dgeqpt_host call (host arrays)."""
    q: object          # m x k column-major (views of the caller's buffers when given)
    r: object          # k x n
    pivots: object     # int64 n, 0-based
    k: int
    k0: int
    ctx: _lib.Ctx


def dgeqpt_host(a, d_factor: float = 1.25, nnz: int = 4, seed: int = 0, eps_tol: float = 1e-4,
                cond_method: int = CondMethod.identity_deviation, q_out=None, r_out=None, j_out=None,
                sketch_family: str = "saso", stream=None, comm: Optional[Comm] = None,
                global_row_offset: int = 0, wavefront: bool = True) -> HostResult:
    """Host data in, host factors out (cqrrpt_gpu_dgeqpt_host): ``a`` is a
    column-major float64 numpy array or CPU torch tensor (pin it for full
    PCIe bandwidth); Q is downloaded block by block while the device is still
    computing (one rank: as a 128-column wavefront through precondition, Gram,
    Cholesky and the final solve; ``wavefront=False`` runs those as whole
    passes, CQRRPT_GPU_NO_WAVEFRONT). Both give dgeqpt's factors bit for bit
    with the same ``wavefront`` setting.
    ``q_out`` (m x n), ``r_out`` (n x n), ``j_out`` (n) may be preallocated
    (pinned) buffers; the results are their leading k columns / rows."""
    torch = _torch()
    tensor = isinstance(a, torch.Tensor)
    if tensor:
        if a.dtype != torch.float64 or a.is_cuda or a.stride(0) != 1:
            raise InvalidArgument("a must be a column-major float64 CPU tensor")
        m, n = a.shape
        lda, pa = max(a.stride(1), 1), a.data_ptr()
    else:
        a = np.asfortranarray(a, dtype=np.float64)
        m, n = a.shape
        lda, pa = max(m, 1), a.ctypes.data
    alloc = (lambda r, c: torch.empty((c, r), dtype=torch.float64).t()) if tensor else \
        (lambda r, c: np.empty((r, c), order="F"))
    q = q_out if q_out is not None else alloc(m, n)
    r = r_out if r_out is not None else alloc(n, n)
    j = j_out if j_out is not None else (torch.empty(max(n, 1), dtype=torch.int64) if tensor
                                         else np.empty(max(n, 1), dtype=np.int64))
    ptr = (lambda t: t.data_ptr()) if tensor else (lambda t: t.ctypes.data)
    ctx = _lib.new_ctx()
    ctx.stream = _stream_ptr(stream)
    ctx.cond_method = int(cond_method)
    if not wavefront:
        ctx.flags |= _lib.F_NO_WAVEFRONT
    families = {"saso": _lib.SKETCH_SASO, "gaussian": _lib.SKETCH_GAUSSIAN, "srft": _lib.SKETCH_SRFT}
    if sketch_family not in families:
        raise InvalidArgument(f"sketch_family must be one of {sorted(families)}")
    ctx.sketch_family = families[sketch_family]
    if comm is not None:  # row shard of a multi-GPU job (NCCL communicator)
        ctx.comm = comm.handle
        ctx.nranks = comm.nranks
        ctx.rank = comm.rank
        ctx.global_row_offset = int(global_row_offset)
    k, k0 = _lib._i64(), _lib._i64()
    _lib.check(_lib.load().cqrrpt_gpu_dgeqpt_host(m, n, pa, lda, float(d_factor), int(nnz), int(seed), float(eps_tol),
                                                  ptr(q), max(m, 1), ptr(r), max(n, 1), ptr(j), ctypes.byref(k),
                                                  ctypes.byref(k0), ctypes.byref(ctx)), "dgeqpt_host")
    kk = k.value
    return HostResult(q[:, :kk], r[:kk, :], j[:n], kk, k0.value, ctx)


def validate(dec: PivotedQR, m, tol: float) -> ValidationReport:
    """validate() (qrcp.cc:150-196) evaluated on the GPU (DMMA Gram + GEMM)."""
    torch = _torch()
    L = _lib.load()
    A = m if (isinstance(m, torch.Tensor) and m.is_cuda) else to_device_colmajor(m)
    Q = dec.q if isinstance(dec.q, torch.Tensor) else to_device_colmajor(dec.q)
    R = dec.r if isinstance(dec.r, torch.Tensor) else to_device_colmajor(dec.r)
    piv = torch.as_tensor(np.asarray(dec.pivots.cpu() if isinstance(dec.pivots, torch.Tensor) else dec.pivots),
                          dtype=torch.int64)
    mm, n = A.shape
    k = int(dec.rank)
    rep = ValidationReport()
    p = piv.numpy()
    rep.pivots_valid = (p.size == n and np.array_equal(np.sort(p), np.arange(n)))
    rep.diag_nonincreasing = True
    rh = R.cpu().numpy() if k else np.zeros((0, n))
    for i in range(1, min(k, n)):
        if abs(rh[i, i]) > abs(rh[i - 1, i - 1]):
            rep.diag_nonincreasing = False
    rep.max_below_diag = float(np.max(np.abs(np.tril(rh, -1)))) if rh.size else 0.0
    if rep.pivots_valid:
        of, o2, rc = _lib._f64(), _lib._f64(), _lib._f64()
        Qc = Q if k else colmajor_empty(mm, 1)
        Rc = R if k else colmajor_empty(1, n)
        _lib.check(L.cqrrpt_gpu_validate(mm, n, k, A.data_ptr(), _ld(A), Qc.data_ptr(), _ld(Qc), Rc.data_ptr(),
                                         _ld(Rc), piv.to(A.device).data_ptr(), ctypes.byref(of), ctypes.byref(o2),
                                         ctypes.byref(rc), _stream_ptr(None)), "validate")
        rep.orth_loss, rep.orth_loss_fro, rep.recon_rel = o2.value, of.value, rc.value
    else:
        rep.recon_rel = float("inf")
    rep.passed = rep.pivots_valid and rep.max_below_diag == 0.0 and rep.orth_loss <= tol and rep.recon_rel <= tol
    return rep


def cqrrpt(m, cfg: Optional[CqrrptConfig] = None) -> CqrrptOutput:
    """Drop-in for ``cqrrpt::cqrrpt(const DenseMatrix&, const CqrrptConfig&)``
    (cqrrpt.cc:317-328). ``m`` is not modified. Host input -> host outputs
    (numpy, column-major); CUDA input -> CUDA outputs."""
    cfg = cfg or CqrrptConfig()
    check_config(cfg)
    if cfg.measure_distortion:
        raise NotImplementedError("measure_distortion is a desk-scale SVD diagnostic, out of scope")
    torch = _torch()
    on_device = isinstance(m, torch.Tensor) and m.is_cuda
    mshape = tuple(m.shape)
    if len(mshape) != 2:
        raise InvalidArgument("expected a matrix")
    rows, n = mshape
    if n == 0:  # cqrrpt.cc:319-324
        q = torch.zeros((rows, 0), dtype=torch.float64, device="cuda") if on_device else np.zeros((rows, 0), order="F")
        r = torch.zeros((0, 0), dtype=torch.float64, device="cuda") if on_device else np.zeros((0, 0), order="F")
        return CqrrptOutput(PivotedQR(q, r, np.zeros(0, dtype=np.int64), 0))
    A = to_device_colmajor(m)  # working copy: Q is written in place
    src = A.clone() if cfg.validate_output else None
    # the default (fast-accept) stage 2 is exact; diagnostics=True fills
    # cond_m_pre with the value the reference's search reports
    res = dgeqpt(A, d_factor=cfg.gamma, nnz=cfg.nnz_per_col, seed=cfg.seed, eps_tol=cfg.eps_tol,
                 cond_method=int(cfg.cond_method), stage1=cfg.stage1_enabled,
                 diagnostics=True, timings=True,
                 sketch_family={SketchFamily.gaussian: "gaussian", SketchFamily.srft: "srft"}.get(cfg.family, "saso"))
    k = res.k
    q_dev = A[:, :k]
    r_dev = res.r
    piv = res.pivots.cpu().numpy().astype(np.int64)
    diag = _diagnostics_from(res.ctx)
    if on_device:
        q_out, r_out = q_dev, r_dev
    else:
        q_out = np.asfortranarray(q_dev.cpu().numpy())
        r_out = np.asfortranarray(r_dev.cpu().numpy())
    out = CqrrptOutput(PivotedQR(q_out, r_out, piv, k), k0=res.k0, k=k, diagnostics=diag)
    if cfg.validate_output:  # cqrrpt.cc:309-312
        tol = max(100.0 * n * UNIT_ROUNDOFF, 10.0 * cfg.eps_tol)
        out.diagnostics.validation = validate(PivotedQR(q_dev, r_dev, piv, k), src, tol)
    return out
