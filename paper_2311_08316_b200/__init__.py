"""B200-native CQRRPT (randomized CholeskyQR with column pivoting, arXiv
2311.08316) for tall FP64 matrices on sm_100a.

The compute path is the CUDA library built from ``csrc/`` (C ABI in
``include/cqrrpt_gpu.h``); this package is the host-side mirror of the
reference's ``cqrrpt()`` interface plus thin launch helpers.
"""
from .cqrrpt import (  # noqa: F401
    Comm,
    CondMethod,
    CqrrptConfig,
    CqrrptDiagnostics,
    CqrrptOutput,
    DeviceResult,
    DomainError,
    HostResult,
    InvalidArgument,
    PhaseTimings,
    PivotedQR,
    SketchFamily,
    ValidationReport,
    UNIT_ROUNDOFF,
    check_config,
    colmajor_empty,
    cqrrpt,
    dgeqpt,
    dgeqpt_host,
    flop_model,
    release_workspace,
    sketch_flops_saso,
    sketch_rows_for,
    to_device_colmajor,
    validate,
)
from . import kernels  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
