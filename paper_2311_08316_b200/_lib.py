"""ctypes binding of the sm_100a library (include/cqrrpt_gpu.h).

There is no fallback: if libcqrrpt_gpu.so is missing or fails to load, every
entry point raises. Device buffers are passed as raw pointers (torch is only
used by callers for allocation, streams and collectives).
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libcqrrpt_gpu.so")

_i64, _u64, _f64, _i32, _vp, _sz = (ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_int32,
                                    ctypes.c_void_p, ctypes.c_size_t)

ERR = {1: "CUDA error", 2: "NCCL error", 3: "singular preconditioner (zero diagonal)", 4: "out of device memory",
       5: "internal error"}
COND_DIAG_RATIO, COND_KRYLOV_BOUNDS, COND_IDENTITY_DEVIATION = 0, 1, 2
F_OUTPUTS_ON_HOST, F_EXACT_STAGE2, F_NO_STAGE1, F_DIAGNOSTICS, F_TIMINGS = 0x1, 0x2, 0x4, 0x8, 0x10
F_FAST_SKETCH = 0x20
F_NO_WAVEFRONT = 0x40
F_WAVEFRONT = 0x80
SKETCH_SASO, SKETCH_GAUSSIAN, SKETCH_SRFT = 0, 1, 2

ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_size_t, ctypes.c_void_p,
                                ctypes.c_void_p)


class Ctx(ctypes.Structure):
    """Mirror of cqrrpt_gpu_ctx (include/cqrrpt_gpu.h)."""
    _fields_ = [
        ("stream", _vp), ("rank", _i32), ("nranks", _i32), ("global_row_offset", _i64), ("comm", _vp),
        ("allreduce", ALLREDUCE_FN), ("allreduce_user", _vp), ("cond_method", _i32), ("flags", _i32),
        ("sketch_family", _i32), ("reserved0", _i32),
        ("d", _i64), ("k_sk", _i64), ("k0_final", _i64), ("retries", _i32), ("stage2_exact", _i32),
        ("cond_m_pre", _f64), ("cond_upper_bound", _f64), ("truncation_ratio", _f64), ("flop_estimate", _f64),
        ("timings_ms", _f64 * 8), ("sketch_rows", _i64),
    ]


SYMBOLS = {
    # name: (restype, argtypes)
    "cqrrpt_gpu_ctx_init": (None, [ctypes.POINTER(Ctx)]),
    "cqrrpt_gpu_dgeqpt": (ctypes.c_int, [_i64, _i64, _vp, _i64, _f64, _i64, _u64, _f64, _vp, _i64, _vp,
                                         ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(Ctx)]),
    "cqrrpt_gpu_dgeqpt_host": (ctypes.c_int, [_i64, _i64, _vp, _i64, _f64, _i64, _u64, _f64, _vp, _i64, _vp, _i64,
                                              _vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(Ctx)]),
    "cqrrpt_gpu_sketch_rows": (_i64, [_f64, _i64]),
    "cqrrpt_gpu_saso_plan": (ctypes.c_int, [_i64, _i64, _i64, _i64, _u64, _vp, _vp]),
    "cqrrpt_gpu_saso_sketch": (ctypes.c_int, [_i64, _i64, _vp, _i64, _i64, _i64, _u64, _i64, _vp, _i64, _vp]),
    "cqrrpt_gpu_srft_sketch": (ctypes.c_int, [_i64, _i64, _vp, _i64, _i64, _u64, _vp, _i64, _vp]),
    "cqrrpt_gpu_gaussian_sketch": (ctypes.c_int, [_i64, _i64, _vp, _i64, _i64, _u64, _i64, _vp, _i64, _vp]),
    "cqrrpt_gpu_saso_sketch_ex": (ctypes.c_int, [_i64, _i64, _vp, _i64, _i64, _i64, ctypes.c_uint64, _i64, _vp, _i64,
                                                   ctypes.c_uint32, _vp]),
    "cqrrpt_gpu_qrcp": (ctypes.c_int, [_i64, _i64, _vp, _i64, _f64, _vp, _i64, _vp, ctypes.POINTER(_i64), _vp]),
    "cqrrpt_gpu_rank_stage1": (ctypes.c_int, [_i64, _i64, _vp, _i64, ctypes.POINTER(_i64), _vp]),
    "cqrrpt_gpu_rank_stage2": (ctypes.c_int, [_i64, _i64, _vp, _i64, _vp, _i64, _f64, _i32, _i32, _vp, _i64, _vp, _i64,
                                              ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i32),
                                              ctypes.POINTER(_f64), _vp]),
    "cqrrpt_gpu_trsm_right": (ctypes.c_int, [_i64, _i64, _vp, _i64, _vp, _vp, _i64, _vp, _i64, _vp]),
    "cqrrpt_gpu_trsm_engine": (ctypes.c_int, [_i64, _i64]),
    "cqrrpt_gpu_gram": (ctypes.c_int, [_i64, _i64, _vp, _i64, _vp, _i64, _vp]),
    "cqrrpt_gpu_potrf": (ctypes.c_int, [_i64, _vp, _i64, ctypes.POINTER(_i64), _vp]),
    "cqrrpt_gpu_cond_estimate": (ctypes.c_int, [_i64, _vp, _i64, _i32, ctypes.POINTER(_f64), _vp]),
    "cqrrpt_gpu_cholesky_qr": (ctypes.c_int, [_i64, _i64, _vp, _i64, _vp, _i64, ctypes.c_int32,
                                              ctypes.POINTER(_i64), _vp]),
    "cqrrpt_gpu_trtri_upper": (ctypes.c_int, [_i64, _vp, _i64, _vp, _i64, _vp]),
    "cqrrpt_gpu_trmm_upper": (ctypes.c_int, [_i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp]),
    "cqrrpt_gpu_validate": (ctypes.c_int, [_i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp,
                                           ctypes.POINTER(_f64), ctypes.POINTER(_f64), ctypes.POINTER(_f64), _vp]),
    "cqrrpt_gpu_flop_model": (_f64, [_i64, _i64, _i64, _i64, _f64]),
    "cqrrpt_gpu_comm_unique_id": (ctypes.c_int, [ctypes.c_char_p]),
    "cqrrpt_gpu_comm_init": (ctypes.c_int, [_i32, _i32, ctypes.c_char_p, ctypes.POINTER(_vp)]),
    "cqrrpt_gpu_comm_allreduce": (ctypes.c_int, [_vp, _vp, _sz, _vp]),
    "cqrrpt_gpu_comm_destroy": (None, [_vp]),
    "cqrrpt_gpu_release_workspace": (None, []),
    "cqrrpt_gpu_add": (ctypes.c_int, [_vp, _vp, _sz, _vp]),
    "cqrrpt_gpu_copy": (ctypes.c_int, [_vp, _vp, _sz, _vp]),
    "cqrrpt_gpu_stream_sync": (ctypes.c_int, [_vp]),
    "cqrrpt_gpu_last_error": (ctypes.c_char_p, []),
    "cqrrpt_gpu_launch_count": (_i64, [_i32]),
}

_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    """Load the CUDA library; raise loudly if it is not built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"CUDA library not built: {LIB_PATH} (run __graft_entry__.build() or "
                               f"python paper_2311_08316_b200/build.py); there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SYMBOLS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    return load().cqrrpt_gpu_last_error().decode(errors="replace")


class InvalidArgument(ValueError):
    """The reference's std::invalid_argument (negative C-ABI return)."""


class DomainError(ArithmeticError):
    """The reference's std::domain_error (zero diagonal in trsm_right)."""


def check(rc: int, what: str) -> None:
    if rc == 0:
        return
    if rc < 0:
        raise InvalidArgument(f"{what}: invalid argument {-rc}: {last_error()}")
    if rc == 3:
        raise DomainError(f"{what}: {last_error()}")
    raise RuntimeError(f"{what}: {ERR.get(rc, rc)}: {last_error()}")


def new_ctx() -> Ctx:
    c = Ctx()
    load().cqrrpt_gpu_ctx_init(ctypes.byref(c))
    return c
