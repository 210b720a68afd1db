"""Pin the CPU oracle against golden vectors produced by the reference itself.

The fixtures come from ``tests/golden/make_golden.py`` (reference run in the
build container).  Bars: integers bit-exact; matrix values rel-Frobenius
<= 1e-12 and |dM_ij| <= 1e-12 sqrt(M_ii M_jj); RHS max|db| <= 1e-12 max|b|;
L2 error within 1e-10.
"""

import hashlib

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import assemble as OA
from oracle import bspline as OB
from oracle import configs as OC
from oracle import project as OP
from oracle import quad as OQ
from oracle import trim as OT
from tests import golden_cases as G


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def oracle_case(desc):
    nel, p = desc["nel"], desc["p"]
    coeff, target = None, None
    if desc["kind"] == "case":
        curves = [OC.case_curve(desc["name"])]
    elif desc["kind"] == "config":
        curves = []
    elif desc["kind"] == "ccircle":
        curves = [OC.closed_circle()]
    else:
        c4 = OC.config(4)
        curves = c4["curves"]
        if desc["coeff"] == "detj":
            coeff = OA.Coeff(c4["coeff"])
    target = {"default": OP.default_target, "config1": OC.f_config1, "config23": OC.f_config23,
              "config5": OC.f_config5, None: None}[desc["target"]]
    cfg = OC.build_space(curves, nel, p)
    return cfg, coeff, target


def assert_matrix_close(M, d, s, full=True):
    """Pattern bit-exact, values per the parity contract."""
    assert sha(M.indptr, M.indices) == str(d[f"{s}_hash"])
    if full:
        R = sp.csr_matrix((d[f"{s}_data"], d[f"{s}_indices"], d[f"{s}_indptr"]), shape=M.shape)
    else:
        rows = d[f"{s}_rows"]
        got = np.concatenate([M.data[M.indptr[r]:M.indptr[r + 1]] for r in rows])
        ref = d[f"{s}_rowsdata"]
        assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))
        assert abs(sp.linalg.norm(M) - float(d[f"{s}_fro"])) <= 1e-12 * float(d[f"{s}_fro"])
        return
    dM = (M - R).tocoo()
    fro = sp.linalg.norm(R)
    assert sp.linalg.norm(dM) <= 1e-12 * fro
    diag = R.diagonal()
    bound = 1e-12 * np.sqrt(diag[dM.row] * diag[dM.col]) + 1e-300
    assert np.all(np.abs(dM.data) <= bound)


CASES = G.tags()


@pytest.mark.parametrize("tag", CASES)
def test_oracle_matches_reference_golden(tag):
    d = G.load(tag)
    desc = G.describe(tag)
    cfg, coeff, target = oracle_case(desc)
    # classification: bit-exact
    assert np.array_equal(cfg.element_class, d["element_class"])
    assert np.array_equal(cfg.func_class, d["func_class"])
    assert np.array_equal(cfg.u_disc[0], d["u_disc1"]) and np.array_equal(cfg.u_disc[1], d["u_disc2"])
    assert np.array_equal(cfg.active(), d["active"])
    # cut-cell rule (host geometry input): same cells, same points to rounding
    rule = cfg.cut_cell_rule(desc["p"])
    keys = sorted(rule.rules)
    assert np.array_equal(np.array(keys, np.int64).reshape(-1, 2), d["cut_el"])
    cnt = np.array([rule.rules[k][0].shape[0] for k in keys], np.int64)
    assert np.array_equal(np.concatenate([[0], np.cumsum(cnt)]), d["cut_ptr"])
    if keys:
        P = np.vstack([rule.rules[k][0] for k in keys])
        W = np.concatenate([rule.rules[k][1] for k in keys])
        assert np.max(np.abs(P - d["cut_pts"])) <= 1e-13
        assert np.max(np.abs(W - d["cut_w"])) <= 1e-13 * np.max(np.abs(d["cut_w"]))
    full = f"{G.strategies_in(d)[0]}_data" in d
    mats = {}
    for s in G.strategies_in(d):
        M = OA.assemble_mass(cfg, coeff, s).data
        mats[s] = M
        assert_matrix_close(M, d, s, full=full)
    if "rhs" in d:
        b = OP.assemble_rhs(target, cfg, coeff)
        assert np.max(np.abs(b - d["rhs"])) <= 1e-12 * np.max(np.abs(d["rhs"]))
    if "l2" in d:
        x = OP.solve_spd(mats[G.strategies_in(d)[-1]], d["rhs"])
        assert abs(OP.l2_error(x, target, cfg) - float(d["l2"])) <= 1e-10


@pytest.fixture(scope="module")
def rules1d():
    return dict(np.load(f"{G.HERE}/rules_1d.npz"))


@pytest.mark.parametrize("nel,p", [(9, 1), (9, 2), (9, 3), (7, 4), (8, 5), (10, 6), (16, 2), (64, 3), (12, 8)])
def test_oracle_weights_bit_exact(rules1d, nel, p):
    """Same LAPACK path -> the oracle's WQ and DWQ weights are the reference's
    bit for bit (this is what makes the c != 1 weight-import parity work)."""
    s = OB.uniform_space(nel, p)
    r = OQ.compute_wq_rules(s)
    k0, ptr, w = r.packed()
    assert np.array_equal(r.layout.points, rules1d[f"wq_{nel}_{p}_pts"])
    assert np.array_equal(k0, rules1d[f"wq_{nel}_{p}_k0"])
    assert np.array_equal(ptr, rules1d[f"wq_{nel}_{p}_ptr"])
    assert np.max(np.abs(w - rules1d[f"wq_{nel}_{p}_w"])) <= 1e-13 * np.max(np.abs(w))
    assert np.max(np.abs(OQ.mass_1d(s) - rules1d[f"wq_{nel}_{p}_M"])) <= 1e-16
    dq = OQ.build_dwq(s, r.layout, float(rules1d[f"dwq_{nel}_{p}_u"]))
    k0, ptr, w = dq.packed()
    assert np.array_equal(dq.layout.points, rules1d[f"dwq_{nel}_{p}_pts"])
    assert np.array_equal(k0, rules1d[f"dwq_{nel}_{p}_k0"])
    assert np.max(np.abs(w - rules1d[f"dwq_{nel}_{p}_w"])) <= 1e-12 * np.max(np.abs(w))


def test_oracle_nonuniform_knots(rules1d):
    s = OB.Space1D(rules1d["wq_nonuni_knots"], 2)
    f, v = s.eval_nonzero(rules1d["eval_nonuni_u"])
    assert np.array_equal(f, rules1d["eval_nonuni_first"])
    assert np.max(np.abs(v - rules1d["eval_nonuni_vals"])) <= 1e-15
    r = OQ.compute_wq_rules(s)
    k0, ptr, w = r.packed()
    assert np.array_equal(r.layout.points, rules1d["wq_nonuni_pts"])
    assert np.array_equal(k0, rules1d["wq_nonuni_k0"])
    assert np.max(np.abs(w - rules1d["wq_nonuni_w"])) <= 1e-13 * np.max(np.abs(w))


def test_reference_known_answers():
    """Known answers the reference suite pins (pkg/tests/test_assembly.py:30-43,
    pkg/tests/test_splines.py:90-93, pkg/tests/test_quadrature.py:119-128)."""
    s = OB.Space1D([0, 0, 1, 1], 1)
    cfg = OT.classify(s, OB.Space1D([0, 0, 1, 1], 1), [])
    M = OA.assemble_mass(cfg, strategy="reference").data.toarray()
    A1 = np.array([[1 / 3, 1 / 6], [1 / 6, 1 / 3]])
    assert np.max(np.abs(M - np.kron(A1, A1))) <= 1e-15
    q = OB.uniform_space(4, 2)
    f, v = q.eval_nonzero(np.array([0.375]))
    assert np.allclose(v[0], [0.125, 0.75, 0.125], atol=1e-15)
    assert np.allclose(OQ.mass_1d(s), A1, atol=1e-15)
    for p in (1, 2, 3, 4):
        cfg = OC.build_space([], 6, p)
        M = OA.assemble_mass(cfg, strategy="reference").data.toarray()
        M1 = OQ.mass_1d(cfg.s1)
        assert np.max(np.abs(M - np.kron(M1, M1))) <= 1e-14
