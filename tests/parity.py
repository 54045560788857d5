"""Shared parity comparators (test infrastructure).

Tie rule (north_star "J and k must match exactly wherever the
sketch's pivot decisions are not within rounding of a tie"): the oracle's
instrumented QRCP (oracle/cqrrpt_oracle.c, bit-identical to qrcp.cc:35-97)
records, per step, the relative gap (w1 - w2)/w1 between the best and the
second-best working squared norm. A step is a near-tie when the gap is
<= 1e3 * u * n. J must equal the reference's exactly up to the first
near-tie step; beyond it only the set of the remaining pivots, k and the
residual / orthogonality metrics are compared. At N = 1 the device sketch
and QRCP are bit-exact, so on tie-free inputs this is full equality; at
N > 1 the allreduced sketch is summed in a different order and the rule is
what makes the comparison meaningful.
"""
from __future__ import annotations

import numpy as np

U = 1.1102230246251565e-16


def tie_bar(n: int) -> float:
    return 1e3 * U * n


def first_near_tie(gaps, n: int, k_sk: int | None = None) -> int:
    g = np.asarray(gaps, dtype=np.float64)
    if k_sk is not None:
        g = g[:k_sk]
    hit = np.nonzero(g <= tie_bar(n))[0]
    return int(hit[0]) if hit.size else int(g.size)


def assert_pivots_tie_rule(got, ref, first_tie: int, k_sk: int | None = None) -> int:
    """Assert J equality up to the first near-tie (full equality when there
    is none before k_sk); always assert `got` is a permutation of `ref`.
    Returns the length of the compared exact prefix."""
    got = np.asarray(got, dtype=np.int64)
    ref = np.asarray(ref, dtype=np.int64)
    n = ref.size
    assert got.size == n
    assert np.array_equal(np.sort(got), np.arange(n)), "pivots are not a permutation"
    k_sk = n if k_sk is None else k_sk
    if first_tie >= k_sk:
        # every decision is tie-free: positions beyond k_sk follow from the swaps
        bad = np.nonzero(got != ref)[0]
        assert bad.size == 0, f"J differs from the reference at {bad[:8].tolist()} (no near-tie)"
        return n
    bad = np.nonzero(got[:first_tie] != ref[:first_tie])[0]
    assert bad.size == 0, f"J differs at {bad[:8].tolist()} before the first near-tie {first_tie}"
    return first_tie


def fnv_pivots(piv) -> str:
    x = 1469598103934665603
    for v in np.asarray(piv, dtype=np.int64):
        x = ((x ^ (int(v) & 0xFFFFFFFFFFFFFFFF)) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{x:016x}"
