"""Multi-process (world_size 2, gloo, CPU) tests of the row-sharded path's
host logic: nnz-balanced contiguous row blocks, the variable-size CSR gather
to the root, and the (num, den) all-reduce of the L2 error.  The row blocks
come from the oracle's CSR of a trimmed case, so the gathered matrix must be
bit-identical to the single-process one."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_matrix():
    from oracle import assemble as OA
    from oracle import configs as OC
    cfg = OC.build_space([OC.closed_circle()], 16, 3)
    return OA.assemble_mass(cfg, strategy="dwq").data


def _worker(rank, world, port, outq):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2101_08053_b200.distributed import allreduce_sum, gather_csr, row_block
        M = _oracle_matrix()
        counts = np.diff(M.indptr)
        rb, re_ = row_block(M.shape[0], world, rank, counts)
        a, b = M.indptr[rb], M.indptr[re_]
        ptr = torch.from_numpy((M.indptr[rb:re_ + 1] - a).astype(np.int32))
        ind = torch.from_numpy(M.indices[a:b].astype(np.int32))
        dat = torch.from_numpy(M.data[a:b].copy())
        out = gather_csr(ptr, ind, dat, rank, world, root=0)
        parts = torch.tensor([float(M.data[a:b].sum()), float(re_ - rb)], dtype=torch.float64)
        allreduce_sum(parts)
        if rank == 0:
            outq.put((out[0].numpy(), out[1].numpy(), out[2].numpy(), parts.numpy(), (rb, re_)))
        else:
            outq.put(("rank1", parts.numpy(), (rb, re_)))
    finally:
        dist.destroy_process_group()


def test_row_block_balanced_by_nnz():
    from paper_2101_08053_b200.distributed import row_block
    counts = np.r_[np.full(10, 100), np.full(90, 10)]
    blocks = [row_block(100, 4, r, counts) for r in range(4)]
    assert blocks[0][0] == 0 and blocks[-1][1] == 100
    assert all(blocks[k][1] == blocks[k + 1][0] for k in range(3))
    sums = [counts[a:b].sum() for a, b in blocks]
    assert max(sums) - min(sums) <= 100
    assert row_block(7, 1, 0) == (0, 7)


@pytest.mark.timeout(300)
def test_gather_and_allreduce_world2_gloo():
    M = _oracle_matrix()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    root = next(r for r in res if not isinstance(r[0], str))
    other = next(r for r in res if isinstance(r[0], str))
    ptr, ind, dat, parts, blk0 = root
    assert blk0[0] == 0 and blk0[1] == other[2][0] and other[2][1] == M.shape[0]
    assert np.array_equal(ptr, M.indptr) and np.array_equal(ind, M.indices)
    assert np.array_equal(dat, M.data)
    assert np.allclose(parts, [M.data.sum(), M.shape[0]], rtol=1e-15)
    assert np.array_equal(parts, other[1])


def _halo_worker(rank, world, port, outq):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import scipy.sparse as sp
        from paper_2101_08053_b200.distributed import BlockSystem, row_block
        n, bw = 40, 3
        A = sp.diags([np.full(n - abs(k), 1.0 + k) for k in range(-bw, bw + 1)], list(range(-bw, bw + 1)),
                     format="csr")
        rb, re_ = row_block(n, world, rank)
        a, b = A.indptr[rb], A.indptr[re_]
        S = BlockSystem(torch.from_numpy((A.indptr[rb:re_ + 1] - a).astype(np.int32)),
                        torch.from_numpy(A.indices[a:b].astype(np.int32)), torch.from_numpy(A.data[a:b].copy()),
                        rb, re_, n)
        full = torch.zeros(n, dtype=torch.float64)
        full[rb:re_] = torch.arange(rb, re_, dtype=torch.float64) + 100.0
        S.exchange(full)
        outq.put((rank, rb, re_, full.numpy(), S.sends, S.recvs, S.diag.numpy(),
                  S.dot(torch.ones(re_ - rb, dtype=torch.float64), torch.ones(re_ - rb, dtype=torch.float64))))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_halo_plan_and_exchange_world2_gloo():
    """BlockSystem (the distributed CG's row block): each rank receives
    exactly the off-block columns its rows read, from their owner; the block
    diagonal; the all-reduced dot."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(2)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, a0, b0, f0, s0, v0, d0, dot0), (r1, a1, b1, f1, s1, v1, d1, dot1) = res
    assert (a0, b1) == (0, 40) and b0 == a1
    assert v0 == [(1, b0, b0 + 3)] and v1 == [(0, a1 - 3, a1)]       # halos of width = bandwidth
    assert s0 == [(1, b0 - 3, b0)] and s1 == [(0, a1, a1 + 3)]
    assert np.array_equal(f0[b0:b0 + 3], np.arange(b0, b0 + 3) + 100.0)
    assert np.array_equal(f1[a1 - 3:a1], np.arange(a1 - 3, a1) + 100.0)
    assert np.all(d0 == 1.0) and np.all(d1 == 1.0)
    assert dot0 == dot1 == 40.0
