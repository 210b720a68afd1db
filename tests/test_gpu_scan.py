"""Row-pointer scan (tq_scan_indptr, single-pass decoupled look-back) against
numpy's cumulative sum: empty and tiny inputs, every tile boundary case,
long look-back chains, unaligned pointers, and the int32 overflow error."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def scan(counts, capture=False, offset=0):
    from paper_2101_08053_b200 import _lib as L
    n = counts.size
    buf = torch.zeros(n + offset + 1, dtype=torch.int32, device="cuda")
    buf[offset:offset + n] = torch.from_numpy(counts.astype(np.int32)).cuda()
    out = torch.full((n + offset + 1,), -7, dtype=torch.int32, device="cuda")
    nnz = L.i64(0)
    L.call("tq_scan_indptr", L.ptr(buf[offset:]), n, L.ptr(out[offset:]), None if capture else L.C.byref(nnz),
           L.stream())
    torch.cuda.synchronize()
    return out[offset:offset + n + 1].cpu().numpy(), int(nnz.value)


@pytest.mark.parametrize("n", [0, 1, 3, 4, 5, 1023, 1024, 1025, 4096 + 7, 33 * 1024 + 1, 3_078_139])
def test_scan_matches_cumsum(n):
    rng = np.random.default_rng(n)
    counts = rng.integers(0, 100, size=n)
    got, nnz = scan(counts)
    ref = np.concatenate([[0], np.cumsum(counts)])
    assert np.array_equal(got, ref)
    assert nnz == ref[-1]


@pytest.mark.parametrize("offset", [1, 2, 3])
def test_scan_unaligned_pointers(offset):
    counts = np.random.default_rng(offset).integers(0, 9, size=5000)
    got, nnz = scan(counts, offset=offset)
    assert np.array_equal(got, np.concatenate([[0], np.cumsum(counts)]))


def test_scan_overflow_raises():
    counts = np.full(3, 2**30, dtype=np.int64)
    with pytest.raises(OverflowError):
        scan(counts)


def test_scan_repeatable_and_capture_mode():
    counts = np.random.default_rng(5).integers(0, 200, size=200_000)
    a, _ = scan(counts)
    b, _ = scan(counts, capture=True)       # no host read-back: same device result
    assert np.array_equal(a, b)


def scan_tiles(tile_sums, nrows):
    """tq_scan_tiles on given tile sums (tile mode of the row pointer)."""
    from paper_2101_08053_b200 import _lib as L
    tiles = torch.full((L.tile_ints(nrows),), -3, dtype=torch.int32, device="cuda")
    tiles[:len(tile_sums)] = torch.from_numpy(np.asarray(tile_sums, np.int32)).cuda()
    counts = torch.zeros(max(nrows, 1), dtype=torch.int32, device="cuda")
    indptr = torch.full((nrows + 1,), -7, dtype=torch.int32, device="cuda")
    ctx = L.RowCtx()
    ctx.row_begin, ctx.row_end = 5, 5 + nrows
    ctx.counts, ctx.tiles = L.ptr(counts), L.ptr(tiles)
    nnz = L.i64(0)
    L.call("tq_scan_tiles", ctx, L.ptr(indptr), L.C.byref(nnz), L.stream())
    torch.cuda.synchronize()
    return tiles[L.tile_pad(nrows):].cpu().numpy(), indptr.cpu().numpy(), int(nnz.value)


@pytest.mark.parametrize("nrows", [0, 1, 31, 32, 33, 4096, 4096 * 32 + 5, 3_078_139])
def test_scan_tiles_matches_cumsum(nrows):
    ntiles = (nrows + 31) // 32
    sums = np.random.default_rng(nrows).integers(0, 32 * 81, size=ntiles)
    tiles, indptr, nnz = scan_tiles(sums, nrows)
    ref = np.concatenate([[0], np.cumsum(sums)])
    assert np.array_equal(tiles[:ntiles], ref[:-1])       # exclusive bases
    assert indptr[nrows] == ref[-1] and nnz == ref[-1]


def test_scan_tiles_overflow_raises():
    with pytest.raises(OverflowError):
        scan_tiles(np.full(3, 2**30), 96)


def test_tiles_expect_flags_a_changed_total():
    """tq_tiles_expect + tq_scan_tiles: the total against the nnz a captured
    pass sized its output with -> flag word TQ_TILE_CTL + 4 (the
    replay guard must fire without the early scan)."""
    from paper_2101_08053_b200 import _lib as L
    nrows = 4096 * 3 + 7
    sums = np.random.default_rng(2).integers(0, 32 * 81, size=(nrows + 31) // 32)
    total = int(sums.sum())
    for expect, flag in ((total, 0), (total + 1, 1), (total - 32, 1)):
        tiles = torch.zeros((L.tile_ints(nrows),), dtype=torch.int32, device="cuda")
        tiles[:len(sums)] = torch.from_numpy(sums.astype(np.int32)).cuda()
        counts = torch.zeros(nrows, dtype=torch.int32, device="cuda")
        indptr = torch.empty(nrows + 1, dtype=torch.int32, device="cuda")
        ctx = L.RowCtx()
        ctx.row_begin, ctx.row_end = 0, nrows
        ctx.counts, ctx.tiles = L.ptr(counts), L.ptr(tiles)
        L.call("tq_tiles_expect", ctx, expect, L.stream())
        L.call("tq_scan_tiles", ctx, L.ptr(indptr), None, L.stream())
        assert int(tiles[L.tile_ctl(nrows) + 4].item()) == flag


def test_replayed_pass_with_another_nnz_writes_nothing_and_raises():
    """A pass run in capture mode with a wrong expected nnz (what a replay
    whose counts moved would see): the scan flags it, the fill kernels write
    nothing into the (captured-size) buffers, and check() raises."""
    from paper_2101_08053_b200 import assembly as A, cases as C, _lib as L
    c5 = C.baseline_config(5, nel=64)
    b2d, cfg = C.build_space(None, 64, 4, curves=c5["curves"])
    f0, csr0 = A.form(b2d, cfg, None, "dwq")
    nnz = csr0.nnz
    A.form(b2d, cfg, None, "dwq", capture={"nnz": nnz})                 # right count: no flag
    f1, csr1 = A.form(b2d, cfg, None, "dwq", capture={"nnz": nnz})
    torch.cuda.synchronize()
    assert int(f1._count_bufs[1][L.tile_ctl(f1._nrows) + 4].item()) == 0
    assert np.array_equal(csr1.data.cpu().numpy(), csr0.data.cpu().numpy())
    f2, csr2 = A.form(b2d, cfg, None, "dwq", capture={"nnz": nnz - 1})   # smaller buffers
    torch.cuda.synchronize()
    assert int(f2._count_bufs[1][L.tile_ctl(f2._nrows) + 4].item()) == 1

    class _G:
        pass
    g = _G()
    g.f = f2
    with pytest.raises(RuntimeError):
        A.GraphFormation.check(g)
