"""World-size-2 gloo test of the row-sharded decomposition (CPU).

Two processes each own a contiguous row block (paper_2311_08316_b200.
distributed.shard_rows), sample their block of S from GLOBAL row indices,
sketch locally, and combine the d x n sketch and the k0 x k0 Gram with one
sum-allreduce each — exactly the exchange the GPU path performs over NCCL.
The per-rank arithmetic runs on the CPU oracle (no GPU here); rank 0 checks
J, k and the factors against the single-process reference result.
"""
import os
import socket

import numpy as np
import pytest

from paper_2311_08316_b200.distributed import shard_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, n, gamma, nnz, seed, q):
    import torch
    import torch.distributed as dist
    from oracle.oracle import Oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = Oracle()
        full = orc.gen_gaussian(m, n, 5)
        full, _ = orc.c5_scale_columns(full, span=4.0, seed=1)
        off, cnt = shard_rows(m, world, rank)
        a = np.asfortranarray(full[off:off + cnt])
        d = orc.sketch_rows_for(gamma, n)
        # 1) local sketch partial from global row indices, then allreduce #1
        msk = orc.saso_apply(d, a, nnz, seed, c0=off)
        t = torch.from_numpy(np.ascontiguousarray(msk))
        dist.all_reduce(t)
        msk = np.asfortranarray(t.numpy())
        # 2) replicated QRCP + stage 1
        r_sk, piv, k_sk = orc.qrcp(msk)
        k0 = orc.rank_stage1(r_sk)
        # 3) local precondition + Gram partial, allreduce #2
        m_pre = orc.trsm_right(np.asfortranarray(a[:, piv[:k0]]), r_sk[:k0, :k0])
        g = orc.gram(m_pre)
        t = torch.from_numpy(np.ascontiguousarray(g))
        dist.all_reduce(t)
        g = t.numpy().copy()
        # 4) replicated Cholesky, local Q rows, replicated R
        r_pre, fi = orc.cholesky(g)
        q_loc = orc.trsm_right(m_pre, r_pre)
        r = orc.multiply_upper_triangular(r_pre, r_sk[:k0, :])
        gathered = [None] * world
        dist.all_gather_object(gathered, (off, q_loc, piv, k0, fi, r, msk))
        if rank == 0:
            q.put(gathered)
    finally:
        dist.destroy_process_group()


def test_row_shard_partition():
    for m, p in [(10, 3), (131072, 8), (7, 8), (1000, 2)]:
        blocks = [shard_rows(m, p, r) for r in range(p)]
        assert sum(c for _, c in blocks) == m
        assert all(blocks[r][0] + blocks[r][1] == (blocks[r + 1][0] if r + 1 < p else m) for r in range(p))
        assert max(c for _, c in blocks) - min(c for _, c in blocks) <= 1


def test_two_rank_gloo_decomposition_matches_single_process():
    import torch.multiprocessing as mp
    m, n, gamma, nnz, seed = 1500, 48, 1.25, 8, 7
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, gamma, nnz, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle.oracle import Oracle
    orc = Oracle()
    full = orc.gen_gaussian(m, n, 5)
    full, _ = orc.c5_scale_columns(full, span=4.0, seed=1)
    ref = orc.cqrrpt(full, gamma=gamma, nnz=nnz, seed=seed, want_sketch=True)
    off0, q0, piv0, k00, fi0, r0, msk0 = gathered[0]
    # the summed sketch equals the single-process sketch up to summation order
    assert np.max(np.abs(msk0 - ref.extra["m_sk"])) <= 1e-13 * np.linalg.norm(full)
    # replicated decisions identical on both ranks and equal to the reference
    for (_, _, piv, k0, fi, r, _) in gathered:
        assert np.array_equal(piv, piv0) and k0 == k00 and fi == fi0 and np.array_equal(r, r0)
    from parity import assert_pivots_tie_rule, first_near_tie
    _, _, k_sk, gaps = orc.qrcp(ref.extra["m_sk"], gaps=True)
    assert_pivots_tie_rule(piv0, ref.pivots, first_near_tie(gaps, n, k_sk), k_sk)
    assert k00 == ref.k0 and fi0 == 0 and ref.k == k00
    err = np.linalg.norm(r0 - ref.r, axis=0) / np.linalg.norm(ref.r, axis=0)
    assert np.max(err) <= 1e-10
    # stacked local Q rows reproduce the global Q
    q_all = np.vstack([g[1] for g in sorted(gathered, key=lambda t: t[0])])
    assert np.max(np.abs(q_all - ref.q)) <= 1e-10


def _bench_rows_worker(rank, world, port, q):
    """bench.py's N-rank input: rank r generates rows [r m/N, (r+1) m/N) of the
    one global matrix (tools/workloads.py tiles; C3's noise scale from the
    all-reduced ||AB||_F^2)."""
    import torch
    import torch.distributed as dist
    from tools.workloads import make_rows
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        for cfg in (dict(m=4 * 65536, n=6, gamma=1.25, kind="graded"),
                    dict(m=4 * 65536, n=6, gamma=1.25, kind="lowrank", rank=3, noise=1e-12)):
            ml = cfg["m"] // world
            a = make_rows(cfg, rank * ml, (rank + 1) * ml, "cpu", dist=dist)
            gathered = [None] * world
            dist.all_gather_object(gathered, a.numpy().copy())
            out[cfg["kind"]] = np.vstack(gathered)
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def test_two_rank_bench_rows_are_one_global_matrix():
    """The N-GPU bench factors the same matrix as the 1-GPU bench (strong
    scaling): the ranks' row blocks stack to the single-rank matrix exactly."""
    import torch.multiprocessing as mp
    from tools.workloads import make_rows
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_rows_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    stacked = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for cfg in (dict(m=4 * 65536, n=6, gamma=1.25, kind="graded"),
                dict(m=4 * 65536, n=6, gamma=1.25, kind="lowrank", rank=3, noise=1e-12)):
        whole = make_rows(cfg, 0, cfg["m"], "cpu").numpy()
        assert np.array_equal(stacked[cfg["kind"]], whole)
