"""Row-block formation (the multi-GPU sharding: each rank forms a contiguous
block of active rows and only the raw rows / cut-element groups / deep flags
its block reads).  Every block, eager and graph-captured, must be
bit-identical to the same rows of the full matrix."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _space(kind):
    from paper_2101_08053_b200 import cases as C
    if kind == "bspline":
        return C.build_space(None, 128, 3, curves=C.baseline_config(5)["curves"])
    if kind == "ccircle":
        return C.build_space(None, 64, 2, curves=[C.closed_circle()])
    return C.build_space(kind, 24, 4)


@pytest.mark.parametrize("kind,strategy", [("bspline", "dwq"), ("ccircle", "hybrid"), ("corner", "dwq"),
                                           ("line", "wq")])
@pytest.mark.parametrize("world", [1, 2, 5])
def test_row_blocks_match_full_matrix(kind, strategy, world):
    import torch
    from paper_2101_08053_b200.assembly import GraphFormation, form
    b2d, cfg = _space(kind)
    _, full = form(b2d, cfg, None, strategy)
    F = [t.cpu().numpy() for t in (full.indptr, full.indices, full.data)]
    K = cfg.active_index()[0]["K"]
    for rank in range(world):
        rb, re_ = (K * rank) // world, (K * (rank + 1)) // world
        _, blk = form(b2d, cfg, None, strategy, row_range=(rb, re_))
        gf = GraphFormation(b2d, cfg, None, strategy, row_range=(rb, re_))
        gf.run()
        gf.run()
        torch.cuda.synchronize()
        a, b = F[0][rb], F[0][re_]
        for csr in (blk, gf.csr):
            ptr, ind, dat = (t.cpu().numpy() for t in (csr.indptr, csr.indices, csr.data))
            assert np.array_equal(ptr, F[0][rb:re_ + 1] - a)
            assert np.array_equal(ind[: b - a], F[1][a:b])
            assert np.array_equal(dat[: b - a], F[2][a:b])
