"""Edge cases of the formation path against the oracle (bars as in
tests/test_gpu_parity.py): single-element and two-element meshes, degree 1,
a knot vector with a repeated interior knot (C^0 line inside a trimmed
space), and a trim that leaves no active function.  The naive `wq`
strategy on trimmed spaces imports the oracle's weight tables."""

import numpy as np
import pytest

from tests.test_gpu_parity import assert_matrix_close

pytestmark = pytest.mark.gpu

KNOTS = [0, 0, 0, 0.2, 0.55, 0.55, 0.8, 1, 1, 1]     # reference test_cli custom knots (degree 2)


def _pair(case, nel, p, knots=None):
    import paper_2101_08053_b200 as P
    from paper_2101_08053_b200 import cases as C
    from oracle import bspline as OB, configs as OC, trim as OT
    kv = None if knots is None else P.KnotVector(np.array(knots, float), p)
    b2d, cfg = C.build_space(case, nel, p, kv, kv)
    if knots is None:
        ocfg = OC.build_space([OC.case_curve(case)], nel, p)
    else:
        ocfg = OT.classify(OB.Space1D(knots, p), OB.Space1D(knots, p), [OC.case_curve(case)])
    return P, b2d, cfg, ocfg


def _imported(b2d, ocfg):
    from oracle import assemble as OA
    from paper_2101_08053_b200.quadrature import rules_from_arrays
    r1, r2, dwq = OA.build_rules(OA._Run(ocfg, OA.Coeff()), True)

    def conv(basis, rs, d, u=None):
        k0, wptr, w = rs.packed()
        return rules_from_arrays(basis, rs.layout.points, rs.layout.offsets, k0, wptr, w, d, u)

    b1, b2 = b2d.dir
    return conv(b1, r1, 0), conv(b2, r2, 1), {(d, u): conv((b1, b2)[d], rs, d, u) for (d, u), rs in dwq.items()}


def _check(P, b2d, cfg, ocfg, strategy):
    from oracle import assemble as OA
    assert np.array_equal(cfg.element_class, ocfg.element_class)
    assert np.array_equal(cfg.func_class, ocfg.func_class)
    R = OA.assemble_mass(ocfg, strategy=strategy).data
    rules = _imported(b2d, ocfg) if strategy == "wq" and cfg.has_cuts() else None
    M = P.assemble_mass(b2d, cfg, strategy=strategy, rules=rules).data
    assert_matrix_close(M, R)


@pytest.mark.parametrize("strategy", ["reference", "wq", "hybrid", "dwq"])
@pytest.mark.parametrize("nel,p", [(1, 1), (1, 3), (2, 2), (3, 1)])
def test_tiny_meshes(nel, p, strategy):
    P, b2d, cfg, ocfg = _pair("line", nel, p)
    _check(P, b2d, cfg, ocfg, strategy)


@pytest.mark.parametrize("strategy", ["reference", "wq", "hybrid", "dwq"])
def test_repeated_interior_knot(strategy):
    P, b2d, cfg, ocfg = _pair("circle", 7, 2, KNOTS)
    _check(P, b2d, cfg, ocfg, strategy)


def test_no_active_functions():
    """A trim whose valid side holds no element: empty 0 x 0 matrix, as the
    oracle, and an empty load vector."""
    import paper_2101_08053_b200 as P
    from paper_2101_08053_b200 import cases as C, trimming as T
    from oracle import assemble as OA, configs as OC, trim as OTr
    # valid side of a line below the whole domain: nothing is active
    b2d, cfg = C.build_space(None, 4, 2, curves=[T.LineTrim((1.0, -1.0), (0.0, -1.0))])
    ocfg = OC.build_space([OTr.LineTrim((1.0, -1.0), (0.0, -1.0))], 4, 2)
    assert np.array_equal(cfg.element_class, ocfg.element_class)
    assert (cfg.element_class == 2).all()
    for strategy in ("reference", "wq", "hybrid", "dwq"):
        R = OA.assemble_mass(ocfg, strategy=strategy).data
        M = P.assemble_mass(b2d, cfg, strategy=strategy).data
        assert M.shape == R.shape == (0, 0) and M.nnz == R.nnz == 0


def _inject_oracle_cut_rule(cfg, ocfg, q):
    """The oracle's cut-cell points in place of the native ones (the
    per-entry bars are for the kernels; the native decomposition differs
    by ulps, which sliver sub-cells amplify -- DESIGN §3)."""
    from paper_2101_08053_b200._classify import CutCellRule
    orule = ocfg.cut_cell_rule(q)
    keys = sorted(orule.rules)
    el = np.array(keys, np.int64).reshape(-1, 2)
    pts = [orule.rules[k][0] for k in keys]
    ptr = np.concatenate([[0], np.cumsum([x.shape[0] for x in pts])]).astype(np.int64)
    P = np.vstack(pts) if pts else np.empty((0, 2))
    W = np.concatenate([orule.rules[k][1] for k in keys]) if keys else np.empty(0)
    cfg._cut_rules[q] = CutCellRule(q, el, ptr, P, W, np.zeros(len(keys), np.int32))


@pytest.mark.parametrize("nel,p", [(24, 2), (48, 3)])
def test_corner_bezier_larger_meshes(nel, p):
    """The cubic-Bezier case on the device classifier beyond the golden
    sizes: classes and u_disc bit-exact, dwq values against the oracle
    (native cut cells: rel-Frobenius; oracle cut cells injected: per entry)."""
    from oracle import assemble as OA
    P, b2d, cfg, ocfg = _pair("corner", nel, p)
    assert np.array_equal(cfg.element_class, ocfg.element_class)
    assert np.array_equal(cfg.func_class, ocfg.func_class)
    assert np.array_equal(cfg.u_disc[0], ocfg.u_disc[0]) and np.array_equal(cfg.u_disc[1], ocfg.u_disc[1])
    R = OA.assemble_mass(ocfg, strategy="dwq").data
    M = P.assemble_mass(b2d, cfg, strategy="dwq").data
    assert np.array_equal(M.indptr, R.indptr) and np.array_equal(M.indices, R.indices)
    assert np.linalg.norm(M.data - R.data) <= 1e-12 * np.linalg.norm(R.data)
    _inject_oracle_cut_rule(cfg, ocfg, p)
    assert_matrix_close(P.assemble_mass(b2d, cfg, strategy="dwq").data, R)


def test_cli_mass_corner(tmp_path):
    from tests.test_cli import read_csv
    from paper_2101_08053_b200.cli import main
    assert main(["mass", "--case", "corner", "--degrees", "2", "--meshes", "8", "--out", str(tmp_path)]) == 0
    _, rows = read_csv(tmp_path / "mass_corner_n8.csv")
    assert float(rows[0][4]) <= 1e-12 and float(rows[0][5]) <= 1e-12
