"""Specialised kernels against their generic counterparts, bit for bit: the
degree-templated c == 1 element-Gauss part of the raw rows
(k_raw_gauss_sep<P>) against the generic k_raw_regular<1>, through the whole
formation (the generic path is forced with TQ_RAW_GAUSS_GENERIC, read when
the library loads -- hence the subprocesses)."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
from paper_2101_08053_b200 import cases as C
from paper_2101_08053_b200.assembly import form
kind, nel, p, strategy = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
if kind == "bspline":
    b2d, cfg = C.build_space(None, nel, p, curves=C.baseline_config(5)["curves"])
else:
    b2d, cfg = C.build_space(kind, nel, p)
_, csr = form(b2d, cfg, None, strategy)
np.savez(sys.argv[5], *[t.cpu().numpy() for t in (csr.indptr, csr.indices, csr.data)])
"""


@pytest.mark.parametrize("kind,nel,p,strategy", [("bspline", 96, 4, "dwq"), ("bspline", 64, 3, "hybrid"),
                                                 ("corner", 24, 2, "hybrid"), ("bspline", 48, 6, "dwq")])
def test_gauss_part_specialisation_bit_identical(tmp_path, kind, nel, p, strategy):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for mode in ("sep", "generic"):
        env = dict(os.environ)
        env.pop("TQ_RAW_GAUSS_GENERIC", None)
        if mode == "generic":
            env["TQ_RAW_GAUSS_GENERIC"] = "1"
        f = tmp_path / f"{mode}.npz"
        subprocess.run([sys.executable, "-c", _SCRIPT.format(root=root), kind, str(nel), str(p), strategy, str(f)],
                       check=True, env=env, timeout=600)
        z = np.load(f)
        out[mode] = [z[k] for k in ("arr_0", "arr_1", "arr_2")]
    for a, b in zip(out["sep"], out["generic"]):
        assert np.array_equal(a, b)


def _count_state(f, ctx_fn, call):
    """Run one count-pass-1 variant into fresh buffers; returns the per-row
    outputs (lists sorted: their append order is scheduling-dependent)."""
    import torch
    from paper_2101_08053_b200 import _lib as L
    K = f.K
    counts = torch.full((K,), -7, dtype=torch.int32, device=f.dev)
    work = torch.zeros(2 * K + 2, dtype=torch.int32, device=f.dev)
    tiles = torch.zeros(L.tile_ints(K), dtype=torch.int32, device=f.dev)
    f.rowfast = torch.full((K,), 9, dtype=torch.int8, device=f.dev)
    ctx = ctx_fn()
    ctx.counts, ctx.tiles = L.ptr(counts), L.ptr(tiles)
    call(ctx, counts, work)
    torch.cuda.synchronize()
    w = work.cpu().numpy()
    na, nb = int(w[0]), int(w[1])
    la = np.sort(w[2:2 + na])
    lb = np.sort(w[2 + K:2 + K + nb])
    deep = np.ones(K, bool)
    deep[la] = False
    c = counts.cpu().numpy()
    ctl = L.tile_ctl(K)
    t = tiles.cpu().numpy()
    return dict(counts=c[deep], la=la, lb=lb, rowfast=f.rowfast.cpu().numpy(), tiles=t[:(K + 31) // 32],
                ctl=t[ctl:ctl + 2])


@pytest.mark.parametrize("kind,nel,p", [("bspline", 96, 4), ("corner", 24, 2)])
@pytest.mark.parametrize("spoil", [False, True])
def test_speculative_count_pass(kind, nel, p, spoil):
    """tq_row_counts_spec + tq_row_counts_verify against tq_row_counts_geo:
    identical rows, lists, tile sums and first/last list-A words -- with all
    lines positive (no redo) and with a factor entry zeroed (the device-side
    redo runs)."""
    import torch
    from paper_2101_08053_b200 import _lib as L, cases as C
    from paper_2101_08053_b200.assembly import form
    if kind == "bspline":
        b2d, cfg = C.build_space(None, nel, p, curves=C.baseline_config(5)["curves"])
    else:
        b2d, cfg = C.build_space(kind, nel, p)
    f, _ = form(b2d, cfg, None, "dwq")
    assert f.a1 is not None and f.deep is not None
    if spoil:        # one non-positive line: the speculation is wrong there
        f.a1 = f.a1.clone()
        f.a1[f.b1.n // 2, f.b1.p + 1] = 0.0
    pos = torch.empty(f.b1.n + f.b2.n, dtype=torch.int8, device=f.dev)
    bad = torch.empty(1, dtype=torch.int32, device=f.dev)
    ref = _count_state(f, f.rowctx, lambda ctx, c, w: L.call(
        "tq_row_counts_geo", ctx, L.ptr(f.deep), L.ptr(pos), L.ptr(c), L.ptr(w), L.stream()))

    def spec(ctx, c, w):
        L.call("tq_row_counts_spec", ctx, L.ptr(f.deep), L.ptr(c), L.ptr(w), L.stream())
        L.call("tq_row_counts_verify", ctx, L.ptr(f.deep), L.ptr(pos), L.ptr(bad), L.ptr(c), L.ptr(w), L.stream())
    got = _count_state(f, f.rowctx, spec)
    assert (int(bad.item()) > 0) == spoil
    for k in ref:
        assert np.array_equal(ref[k], got[k]), k



def test_tiled_coefficient_grid_matches_pointwise(tmp_path):
    """k_coeff_grid_tiled (line tables in shared memory, direction-2
    contraction first) against the per-point detj kernel (TQ_COEFF_POINTWISE,
    read when the library loads) on ragged grid sizes, including points on
    knots: equal to rounding (1e-13)."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2101_08053_b200 import cases as C, assembly as A
rng = np.random.default_rng(3)
geo = C.geometry_map(np.random.default_rng(0))
x1 = torch.tensor(np.sort(np.concatenate([rng.uniform(0, 1, 37), np.linspace(0, 1, 9)])), device="cuda")
x2 = torch.tensor(np.sort(np.concatenate([rng.uniform(0, 1, 301), [0.0, 0.5, 1.0]])), device="cuda")
np.save(sys.argv[1], geo.grid_device(x1, x2).cpu().numpy())
""".format(root=root)
    out = {}
    for mode in ("tiled", "pointwise"):
        env = dict(os.environ)
        env.pop("TQ_COEFF_POINTWISE", None)
        if mode == "pointwise":
            env["TQ_COEFF_POINTWISE"] = "1"
        f = tmp_path / f"{mode}.npy"
        subprocess.run([sys.executable, "-c", script, str(f)], check=True, env=env, timeout=600)
        out[mode] = np.load(f)
    assert out["tiled"].shape == (46, 304)
    # the tiled kernel contracts direction 2 first: same terms, another order
    np.testing.assert_allclose(out["tiled"], out["pointwise"], rtol=1e-13,
                               atol=1e-13 * np.max(np.abs(out["pointwise"])))


@pytest.mark.parametrize("kind,nel,p,strategy", [("bspline", 48, 6, "dwq"), ("bspline", 32, 8, "hybrid"),
                                                 ("corner", 12, 7, "hybrid")])
def test_wide_cut_blocks_bit_identical(tmp_path, kind, nel, p, strategy):
    """Block-per-group cut-element blocks (k_cut_blocks_wide, q2 >= 7)
    against the warp-per-group kernel (forced with TQ_CUT_BLOCKS_WIDE_FROM,
    read when the library loads): the whole formation, bit for bit."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for mode in ("wide", "warp"):
        env = dict(os.environ)
        env.pop("TQ_CUT_BLOCKS_WIDE_FROM", None)
        if mode == "warp":
            env["TQ_CUT_BLOCKS_WIDE_FROM"] = "99"
        f = tmp_path / f"{mode}.npz"
        subprocess.run([sys.executable, "-c", _SCRIPT.format(root=root), kind, str(nel), str(p), strategy, str(f)],
                       check=True, env=env, timeout=600)
        z = np.load(f)
        out[mode] = [z[k] for k in ("arr_0", "arr_1", "arr_2")]
    for a, b in zip(out["wide"], out["warp"]):
        assert np.array_equal(a, b)


_CUTCELL_SNIPPET = """
import hashlib, sys
sys.path.insert(0, {root!r})
import numpy as np
from paper_2101_08053_b200 import cases as C, assembly as A
for nel in (96, 256):
    c5 = C.baseline_config(5, nel=nel)
    b2d, cfg = C.build_space(None, nel, 4, curves=c5["curves"])
    for s in ("dwq", "hybrid", "wq"):
        M = A.assemble_mass(b2d, cfg, None, strategy=s).data
        h = hashlib.sha256()
        for a in (M.indptr, M.indices, M.data):
            h.update(np.ascontiguousarray(a).tobytes())
        print(nel, s, M.nnz, h.hexdigest())
"""


def test_cutcell_rows_over_group_lists_bit_identical():
    """k_raw_cutcells_list (default: per-row group lists built once per plan)
    against the element-window scan of k_raw_cutcells (TQ_CUTCELL_LISTS=0,
    read once per process): the same additions in the same order, so the
    CSR is bit-identical (config-5 recipe, three strategies)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for v in ("0", "1"):
        env = dict(os.environ, TQ_CUTCELL_LISTS=v)
        r = subprocess.run([sys.executable, "-c", _CUTCELL_SNIPPET.format(root=root)], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(r.stdout)
    assert outs[0] == outs[1] and len(outs[0].splitlines()) == 6
