"""The row-sharded path end to end with two ranks (VERDICT r1 'Next' #5, #9):
both ranks on cuda:0, gloo for the exchanges (one GPU per box here; the
ranks never wait on each other's kernels -- every exchange goes through the
host).  Against the single-process results on the same inputs:

* ``assemble_mass_distributed`` (nnz-balanced row blocks, batched p2p
  gather): the CSR bit-identical to ``assemble_mass``;
* ``l2_error_distributed`` (elements and cut points split, one all-reduce):
  within 1e-12 of ``l2_error``;
* ``solve_spd_distributed`` (row-sharded CG with a halo exchange of the
  search direction per iteration, src/projection.py:148-211): residual
  <= 1e-13, the same projection as the single-process solve in the M-norm,
  and the same L2 error to 1e-10 (src/cli.py:184-188 agreement).
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _space():
    from paper_2101_08053_b200 import cases as C
    return C.build_space(None, 64, 3, curves=[C.closed_circle()])


def _worker(rank, world, port, outq):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2101_08053_b200 as P
        from paper_2101_08053_b200 import cases as C
        from paper_2101_08053_b200 import distributed as D
        from paper_2101_08053_b200.projection import assemble_rhs_device
        b2d, cfg = _space()
        M = D.assemble_mass_distributed(b2d, cfg, None, strategy="dwq")
        prob = P.ProjectionProblem(C.f_config23, b2d, cfg, strategy="dwq")
        K = cfg.active_index()[0]["K"]
        x_ref = np.random.default_rng(7).standard_normal(K)
        e_dist = D.l2_error_distributed(x_ref, prob)
        # the solve on this rank's block
        f, csr = D.form_block(b2d, cfg, None, "dwq", rank, world)
        rb, re_ = csr.row_begin, csr.row_end
        S = D.BlockSystem(csr.indptr, csr.indices, csr.data, rb, re_, K)
        b_loc = assemble_rhs_device(prob, row_range=(rb, re_))
        st = {}
        x_loc = D.solve_spd_distributed(S, b_loc, stats=st)
        parts = [None] * world
        dist.all_gather_object(parts, (rb, re_, x_loc.cpu().numpy()))
        x = np.concatenate([p[2] for p in sorted(parts, key=lambda p: p[0])])
        if rank == 0:
            outq.put(dict(indptr=M.data.indptr, indices=M.data.indices, data=M.data.data, e_dist=e_dist,
                          x=x, st=st, blocks=[(p[0], p[1]) for p in sorted(parts, key=lambda p: p[0])]))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_row_sharded_formation_error_and_solve_world2():
    import paper_2101_08053_b200 as P
    from paper_2101_08053_b200 import cases as C
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=500)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    b2d, cfg = _space()
    M = P.assemble_mass(b2d, cfg, None, strategy="dwq")
    assert np.array_equal(res["indptr"], M.data.indptr)
    assert np.array_equal(res["indices"], M.data.indices)
    assert np.array_equal(res["data"], M.data.data)
    (a0, b0), (a1, b1) = res["blocks"]
    assert a0 == 0 and b0 == a1 and b1 == M.shape[0] and b0 > 0
    prob = P.ProjectionProblem(C.f_config23, b2d, cfg, strategy="dwq")
    x_ref = np.random.default_rng(7).standard_normal(M.shape[0])
    assert abs(res["e_dist"] - P.l2_error(x_ref, prob)) <= 1e-12
    # the solve
    assert res["st"]["residual"] <= 1e-13 and res["st"]["ranks"] == 2
    b = P.assemble_rhs(prob)
    x1 = P.solve_spd(M, b)
    x2 = res["x"]
    A = M.data
    assert np.linalg.norm(A @ x2 - b) / np.linalg.norm(b) <= 1e-13
    dx = x2 - x1
    assert np.sqrt(abs(dx @ (A @ dx))) <= 1e-8 * np.sqrt(x1 @ (A @ x1))
    assert abs(P.l2_error(x2, prob) - P.l2_error(x1, prob)) <= 1e-10
