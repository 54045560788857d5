"""Row-sharded multi-GPU CQRRPT (one process per GPU).

The path shards by rows: rank r owns rows
[offset_r, offset_r + m_r) of the tall matrix. SASO column c of S depends
only on the GLOBAL row index c (sketch.cc:81), so every rank samples its own
block of S with no communication. The only cross-GPU data are the d x n
sketch partials and the k0 x k0 Gram partials, each combined by one
sum-allreduce (NCCL over NVLink/NVSwitch inside the library); QRCP, the rank
decisions, Cholesky and R are replicated bit-identically on every rank, and
each rank writes its own rows of Q in place.
"""
from __future__ import annotations

from typing import Optional, Tuple

from .cqrrpt import Comm, DeviceResult, dgeqpt


def shard_rows(m: int, nranks: int, rank: int) -> Tuple[int, int]:
    """Contiguous balanced row block of `rank`: (global offset, local rows)."""
    if nranks < 1 or not (0 <= rank < nranks):
        raise ValueError("bad rank / nranks")
    base, extra = divmod(m, nranks)
    count = base + (1 if rank < extra else 0)
    offset = rank * base + min(rank, extra)
    return offset, count


def cqrrpt_sharded(a_local, comm: Optional[Comm], global_row_offset: int, **kw) -> DeviceResult:
    """cqrrpt_gpu_dgeqpt on this rank's rows (column-major CUDA tensor).
    R, pivots, k, k0 come back identical on every rank; Q overwrites
    a_local[:, :k]."""
    return dgeqpt(a_local, comm=comm, global_row_offset=global_row_offset, **kw)
