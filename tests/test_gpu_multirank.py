"""The library's multi-rank path (row shards + two sum-allreduces) exercised on
one GPU: two host threads act as two ranks, each with its own stream, row
block and global row offset, joined by a caller-supplied allreduce (the
cqrrpt_gpu_allreduce_fn hook) that sums the device buffers in rank order.
No kernel waits on another: the ranks only meet in host code between phases.
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


class ThreadAllreduce:
    """Sum-allreduce between host-thread ranks; ``order`` is the rank order
    the partial buffers are added in (NCCL's ring/tree order differs from a
    single chain, which is what the tie rule is for)."""

    def __init__(self, nranks, order=None):
        from paper_2311_08316_b200 import _lib
        self.L = _lib.load()
        self.n = nranks
        self.order = list(order) if order is not None else list(range(nranks))
        self.bar = threading.Barrier(nranks)
        self.bufs = [None] * nranks

    def for_rank(self, rank):
        L = self.L

        def ar(ptr, count, stream):
            L.cqrrpt_gpu_stream_sync(stream)
            self.bufs[rank] = ptr
            self.bar.wait()
            first = self.order[0]
            if rank == first:
                for r in self.order[1:]:
                    assert L.cqrrpt_gpu_add(ptr, self.bufs[r], count, stream) == 0
                L.cqrrpt_gpu_stream_sync(stream)
            self.bar.wait()
            if rank != first:
                assert L.cqrrpt_gpu_copy(ptr, self.bufs[first], count * 8, stream) == 0
            self.bar.wait()
        return ar


@pytest.mark.parametrize("nranks,order", [(2, None), (3, None), (3, (2, 0, 1)), (4, (3, 2, 1, 0))])
def test_threaded_ranks_match_single_gpu(cuda, oracle, nranks, order):
    import torch
    from paper_2311_08316_b200.distributed import shard_rows
    from parity import assert_pivots_tie_rule, first_near_tie
    m, n = 9000, 96
    a = oracle.gen_gaussian(m, n, 17)
    ref = oracle.cqrrpt(a, gamma=1.25, nnz=8, seed=0, want_sketch=True)
    _, _, k_sk, gaps = oracle.qrcp(ref.extra["m_sk"], gaps=True)
    coll = ThreadAllreduce(nranks, order)
    results = [None] * nranks
    errors = []

    def run(rank):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            off, cnt = shard_rows(m, nranks, rank)
            with torch.cuda.stream(st):
                A = cuda.to_device_colmajor(np.asfortranarray(a[off:off + cnt]))
                st.synchronize()
                res = cuda.dgeqpt(A, d_factor=1.25, nnz=8, seed=0, stream=st, allreduce=coll.for_rank(rank),
                                  nranks=nranks, rank=rank, global_row_offset=off)
                st.synchronize()
                results[rank] = (off, A[:, : res.k].cpu().numpy(), res.r.cpu().numpy(),
                                 res.pivots.cpu().numpy(), res.k, res.k0)
        except Exception as exc:  # surfaced below
            errors.append(repr(exc))
            coll.bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errors, errors
    _, _, r0, p0, k_0, k00 = results[0]
    for (_, _, r, p, k, k0) in results:
        assert np.array_equal(p, p0) and k == k_0 and k0 == k00
        assert np.array_equal(r, r0)  # replicated phases are bit-identical across ranks
    # the allreduced sketch is summed in another order than the reference's
    # single chain: J equal up to the first near-tie (tests/parity.py)
    assert_pivots_tie_rule(p0, ref.pivots, first_near_tie(gaps, n, k_sk), k_sk)
    assert k_0 == ref.k and k00 == ref.k0
    q = np.vstack([x[1] for x in sorted(results, key=lambda t: t[0])])
    v = oracle.validate(a, np.asfortranarray(q), r0, p0)
    vr = oracle.validate(a, ref.q, ref.r, ref.pivots)
    assert v["orth_fro"] <= 10 * max(vr["orth_fro"], 1e-14)
    assert v["recon_rel"] <= 10 * max(vr["recon_rel"], 1e-15)


def test_threaded_ranks_int8_gram_size(cuda):
    """Two ranks with 70000 rows each and n = 1024: each rank's Gram runs on
    the INT8 engine (m_local >= 65536, k >= 1024) before the allreduce. J,
    k0, k follow the single-GPU run under the tie rule (gaps from the
    oracle's QRCP on the single-GPU sketch, which is the reference's sketch
    bit for bit); Q and R to rounding."""
    import torch
    from parity import assert_pivots_tie_rule, first_near_tie
    from paper_2311_08316_b200 import kernels
    m, n, nranks = 140000, 1024, 2
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn((n, m), dtype=torch.float64, device="cuda", generator=g).t()
    a *= (10.0 ** (-6.0 * torch.rand(n, dtype=torch.float64, device="cuda", generator=g)))[None, :]
    single = a.clone()
    ref = cuda.dgeqpt(single, d_factor=1.25, nnz=8, seed=0)
    sk = kernels.saso_sketch(a, cuda.sketch_rows_for(1.25, n), 8, 0).cpu().numpy()
    from oracle.oracle import Oracle
    _, _, k_sk, gaps = Oracle().qrcp(sk, gaps=True)
    coll = ThreadAllreduce(nranks)
    results = [None] * nranks
    errors = []

    def run(rank):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            off = rank * (m // nranks)
            with torch.cuda.stream(st):
                A = a[off:off + m // nranks].clone()
                st.synchronize()
                res = cuda.dgeqpt(A, d_factor=1.25, nnz=8, seed=0, stream=st, allreduce=coll.for_rank(rank),
                                  nranks=nranks, rank=rank, global_row_offset=off)
                st.synchronize()
                results[rank] = (A[:, : res.k].cpu().numpy(), res.r.cpu().numpy(), res.pivots.cpu().numpy(), res.k,
                                 res.k0)
        except Exception as exc:  # surfaced below
            errors.append(repr(exc))
            coll.bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errors, errors
    q0, r0, p0, k_0, k00 = results[0]
    assert np.array_equal(results[1][2], p0) and np.array_equal(results[1][1], r0)
    assert (k_0, k00) == (ref.k, ref.k0)
    assert_pivots_tie_rule(p0, ref.pivots.cpu().numpy(), first_near_tie(gaps, n, k_sk), k_sk)
    q = np.vstack([results[0][0], results[1][0]])
    qr_ref = single[:, : ref.k].cpu().numpy()
    if np.array_equal(p0, ref.pivots.cpu().numpy()):
        assert np.max(np.abs(q - qr_ref)) <= 1e-9
        rr = ref.r.cpu().numpy()
        assert np.max(np.abs(r0 - rr) / (np.abs(rr).max(axis=0) + 1e-300)) <= 1e-9


def test_nccl_communicator_single_rank(cuda):
    """The NCCL path of the library (libnccl dlopen'ed, cqrrpt_gpu_comm_*):
    unique id -> init -> in-place sum-allreduce on device data -> destroy,
    with one rank (one GPU per box); values must come back unchanged."""
    import ctypes
    import torch
    from paper_2311_08316_b200 import _lib
    L = _lib.load()
    buf = ctypes.create_string_buffer(128)
    if L.cqrrpt_gpu_comm_unique_id(buf) != 0:
        pytest.skip("NCCL not loadable here: " + L.cqrrpt_gpu_last_error().decode())
    h = _lib._vp()
    _lib.check(L.cqrrpt_gpu_comm_init(1, 0, buf.raw, ctypes.byref(h)), "comm_init")
    comm = cuda.Comm(h.value, 1, 0)
    try:
        x = torch.arange(1000, dtype=torch.float64, device="cuda") * 0.5
        y = x.clone()
        comm.allreduce(y)
        torch.cuda.synchronize()
        assert torch.equal(x, y)
    finally:
        comm.close()
