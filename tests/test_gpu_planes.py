"""The all-raw formation path in the planes layout (csrc/planes.cu,
csrc/cutrows.cu): strips of interior rows, element-centric cut rows in pair
form, and the one-pass symmetrise / zero-drop / CSR.  Checked against the
row-major path (TQ_PLANES=0 semantics: the per-row kernels and the two
count passes) on the same formation -- pattern identical, values to 1e-13 --
and against itself by row blocks (bit-identical) and graph replays.  The
reference parity of this path is tests/test_gpu_trimmed.py (config 4 goldens
and the bspline_detj cases run through it by default)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _case(nel, p, detj=True):
    from paper_2101_08053_b200 import cases as C
    c4 = C.baseline_config(4, p=p, nel=nel)
    b2d, cfg = C.build_space(None, nel, p, curves=c4["curves"])
    return b2d, cfg, (c4["coeff"] if detj else None)


def _both(b2d, cfg, coeff, strategy):
    import paper_2101_08053_b200 as P
    from paper_2101_08053_b200 import _rawrows as R
    out = {}
    saved = R.PLANES
    try:
        for pl in (False, True):
            R.PLANES = pl
            out[pl] = P.assemble_mass(b2d, cfg, coeff, strategy=strategy).data
    finally:
        R.PLANES = saved
    return out[False], out[True]


@pytest.mark.parametrize("nel,p,strategy,detj", [(48, 3, "dwq", True), (64, 4, "dwq", True), (64, 4, "hybrid", True),
                                                 (64, 4, "wq", True), (32, 3, "reference", False),
                                                 (32, 3, "reference", True), (96, 6, "dwq", True),
                                                 (96, 8, "dwq", True), (40, 2, "hybrid", True)])
def test_planes_path_matches_row_major_path(nel, p, strategy, detj):
    from paper_2101_08053_b200 import _rawrows as R
    b2d, cfg, coeff = _case(nel, p, detj)
    a, b = _both(b2d, cfg, coeff, strategy)
    assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
    # different summation orders (strips contract direction 1 first, cut rows
    # sum pair-form element blocks): rounding-level differences only
    assert np.max(np.abs(a.data - b.data)) <= 1e-13 * np.max(np.abs(a.data))
    assert np.allclose(a.data, b.data, rtol=1e-12, atol=1e-14 * np.max(np.abs(a.data)))


def test_planes_path_used_for_non_separable_formations():
    from paper_2101_08053_b200 import _rawrows as R, assembly as A
    b2d, cfg, coeff = _case(48, 4)
    f, _ = A.form(b2d, cfg, coeff, "dwq")
    assert R.planes(f) and R.pairs_mode(f)
    assert f.raw.shape[0] == (2 * 4 + 1) ** 2           # planes: one row per window entry
    assert int(f._planes_status.item()) == 0


@pytest.mark.parametrize("strategy", ["dwq", "hybrid"])
@pytest.mark.parametrize("world", [2, 3])
def test_planes_row_blocks_bit_identical(strategy, world):
    import torch
    from paper_2101_08053_b200.assembly import GraphFormation, form
    b2d, cfg, coeff = _case(64, 4)
    _, full = form(b2d, cfg, coeff, strategy)
    F = [t.cpu().numpy() for t in (full.indptr, full.indices, full.data)]
    K = cfg.active_index()[0]["K"]
    for rank in range(world):
        rb, re_ = (K * rank) // world, (K * (rank + 1)) // world
        _, blk = form(b2d, cfg, coeff, strategy, row_range=(rb, re_))
        gf = GraphFormation(b2d, cfg, coeff, strategy, row_range=(rb, re_))
        gf.run()
        gf.run()
        torch.cuda.synchronize()
        gf.check()
        a, b = F[0][rb], F[0][re_]
        for csr in (blk, gf.csr):
            ptr, ind, dat = (t.cpu().numpy() for t in (csr.indptr, csr.indices, csr.data))
            assert np.array_equal(ptr, F[0][rb:re_ + 1] - a)
            assert np.array_equal(ind[: b - a], F[1][a:b])
            assert np.array_equal(dat[: b - a], F[2][a:b])


def test_planes_graph_replay_matches_eager():
    import torch
    from paper_2101_08053_b200.assembly import GraphFormation, form
    b2d, cfg, coeff = _case(96, 6)
    _, eager = form(b2d, cfg, coeff, "dwq")
    gf = GraphFormation(b2d, cfg, coeff, "dwq")
    for _ in range(3):
        gf.run()
    torch.cuda.synchronize()
    gf.check()
    for x, y in zip((eager.indptr, eager.indices, eager.data), (gf.csr.indptr, gf.csr.indices, gf.csr.data)):
        assert torch.equal(x, y)


def _host_ders(kn, p, u):
    """Cox-de Boor values and first derivatives (NURBS book A2.2 / A2.3)."""
    n = len(kn) - p - 1
    s = int(np.searchsorted(kn, u, side="right") - 1)
    s = min(max(s, p), n - 1)

    def vals(q):
        N = np.zeros(q + 1)
        N[0] = 1.0
        left, right = np.zeros(q + 1), np.zeros(q + 1)
        for j in range(1, q + 1):
            left[j] = u - kn[s + 1 - j]
            right[j] = kn[s + j] - u
            saved = 0.0
            for r in range(j):
                t = N[r] / (right[r + 1] + left[j - r])
                N[r] = saved + right[r + 1] * t
                saved = left[j - r] * t
            N[j] = saved
        return N

    N, Nl = vals(p), vals(p - 1)
    D = np.zeros(p + 1)
    for k in range(p + 1):
        i = s - p + k
        if k >= 1 and kn[i + p] > kn[i]:
            D[k] += p / (kn[i + p] - kn[i]) * Nl[k - 1]
        if k <= p - 1 and kn[i + p + 1] > kn[i + 1]:
            D[k] -= p / (kn[i + p + 1] - kn[i + 1]) * Nl[k]
    return s, N, D


@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_geometry_line_tables(p):
    """tq_geo_lines (degree-templated derivatives) against the host formula --
    the regression for the runtime-degree derivative helper that nvcc
    miscompiles for sm_100a in that kernel (scripts/probes/bt.cu)."""
    import torch
    from paper_2101_08053_b200 import _lib as L, _rawrows as R
    from paper_2101_08053_b200.assembly import GeometryMap
    from paper_2101_08053_b200.splines import make_uniform_knots
    R._bind()
    kn = make_uniform_knots(8, p).knots
    n = kn.size - p - 1
    gm = GeometryMap(kn, p, np.zeros((n, n)), np.zeros((n, n)))
    u = np.random.default_rng(p).uniform(0, 1, 64)
    X = torch.tensor(u, dtype=torch.float64, device="cuda")
    sp = torch.empty(64, dtype=torch.int32, device="cuda")
    nd = torch.empty(64 * 2 * (p + 1), dtype=torch.float64, device="cuda")
    L.call("tq_geo_lines", gm.device(), L.ptr(X), 64, L.ptr(sp), L.ptr(nd), L.stream())
    sp, nd = sp.cpu().numpy(), nd.cpu().numpy().reshape(64, 2, p + 1)
    for t in range(64):
        s, N, D = _host_ders(kn, p, u[t])
        assert sp[t] == s
        np.testing.assert_allclose(nd[t, 0], N, rtol=1e-13, atol=1e-15)
        np.testing.assert_allclose(nd[t, 1], D, rtol=1e-12, atol=1e-12 * np.max(np.abs(D)))


@pytest.mark.parametrize("p", [2, 3, 5])
def test_coefficient_kernels_against_host_det_j(p):
    """det J of a perturbed B-spline map from tq_coeff_grid / tq_coeff_points
    (runtime-degree derivatives) and from the Gauss pair blocks' line tables,
    against the host formula: guards every det J kernel against the sm_100a
    miscompile of the runtime-degree helper."""
    import torch
    from paper_2101_08053_b200.assembly import GeometryMap
    from paper_2101_08053_b200.splines import make_uniform_knots
    rng = np.random.default_rng(10 + p)
    kn = make_uniform_knots(6, p).knots
    n = kn.size - p - 1
    g = np.array([kn[i + 1: i + p + 1].mean() for i in range(n)])
    X = np.repeat(g[:, None], n, axis=1) + rng.normal(0, 0.01, (n, n))
    Y = np.repeat(g[None, :], n, axis=0) + rng.normal(0, 0.01, (n, n))
    gm = GeometryMap(kn, p, X, Y)
    u, v = rng.uniform(0, 1, 7), rng.uniform(0, 1, 5)

    def host(uu, vv):
        s1, N1, D1 = _host_ders(kn, p, uu)
        s2, N2, D2 = _host_ders(kn, p, vv)
        Xw, Yw = X[s1 - p: s1 + 1, s2 - p: s2 + 1], Y[s1 - p: s1 + 1, s2 - p: s2 + 1]
        xu, xv = D1 @ Xw @ N2, N1 @ Xw @ D2
        yu, yv = D1 @ Yw @ N2, N1 @ Yw @ D2
        return xu * yv - xv * yu

    ref = np.array([[host(a, b) for b in v] for a in u])
    grid = gm.grid_device(torch.tensor(u, device="cuda"), torch.tensor(v, device="cuda")).cpu().numpy()
    np.testing.assert_allclose(grid, ref, rtol=1e-12)
    P = np.stack(np.meshgrid(u, v, indexing="ij"), axis=-1).reshape(-1, 2)
    pts = gm.at_host(P).reshape(7, 5)
    np.testing.assert_allclose(pts, ref, rtol=1e-12)


_GATHER_SNIPPET = """
import hashlib, sys
sys.path.insert(0, {root!r})
import numpy as np
from paper_2101_08053_b200 import cases as C, assembly as A
for p, nel in ((4, 48), (6, 64), (8, 64)):
    c4 = C.baseline_config(4, p=p, nel=nel)
    b2d, cfg = C.build_space(None, nel, p, curves=c4["curves"])
    for s in ("dwq", "hybrid"):
        M = A.assemble_mass(b2d, cfg, c4["coeff"], strategy=s).data
        h = hashlib.sha256()
        for a in (M.indptr, M.indices, M.data):
            h.update(np.ascontiguousarray(a).tobytes())
        print(p, s, M.nnz, h.hexdigest())
"""


def test_cut_row_gather_element_major_bit_identical():
    """k_cut_rows_gather_em (default) against the entry-major kernel
    (TQ_GATHER_EM=0, read once per process): the same additions in the same
    order per entry, so the CSR is bit-identical (p = 4, 6, 8; dwq and hybrid)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = _GATHER_SNIPPET.format(root=root)
    outs = []
    for em in ("0", "1"):
        env = dict(os.environ, TQ_GATHER_EM=em)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(r.stdout)
    assert outs[0] == outs[1] and len(outs[0].splitlines()) == 6
