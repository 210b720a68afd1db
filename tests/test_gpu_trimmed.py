"""GPU parity on trimmed spaces against the reference's golden vectors.

Integers (element/function classes, u_disc, active order, CSR pattern) are
bit-exact; values rel-Frobenius and per-entry <= 1e-12 (sqrt(M_ii M_jj)
scaled).  The GPU's own weights are used throughout: its pivoted-QR fits
choose LAPACK dgeqp3's pivots (wq.cu), so even where the matrix depends on
the particular weights -- c != 1, and the naive ``wq`` strategy on trimmed
spaces -- it matches the reference (p = 8 at 1e-10, see below).
Those cases are also checked with the reference's weight tables imported
(the oracle reproduces them bit for bit,
tests/test_oracle_golden.py::test_oracle_weights_bit_exact), which isolates
the row kernels at 1e-12.
"""

import hashlib

import numpy as np
import pytest
import scipy.sparse as sp

from tests import golden_cases as G
from tests.test_gpu_parity import assert_matrix_close

pytestmark = pytest.mark.gpu

TAGS = list(G.tags())


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def product_case(desc):
    import paper_2101_08053_b200 as P
    from paper_2101_08053_b200 import cases as C
    nel, p = desc["nel"], desc["p"]
    coeff = None
    if desc["kind"] == "case":
        curves = [C.make_case(desc["name"]).curve()]
    elif desc["kind"] == "config":
        curves = []
    elif desc["kind"] == "ccircle":
        curves = [C.closed_circle()]
    else:
        cfg4 = C.baseline_config(4)
        curves = cfg4["curves"]
        if desc["coeff"] == "detj":
            coeff = cfg4["coeff"]
    b2d, cfg = C.build_space(None, nel, p, curves=curves)
    return b2d, cfg, coeff


def imported_rules(b2d, desc):
    """The reference weights (via the pinned oracle) as product rule sets."""
    from oracle import assemble as OA
    from paper_2101_08053_b200.quadrature import rules_from_arrays
    from tests.test_oracle_golden import oracle_case
    ocfg, ocoeff, _ = oracle_case(desc)
    run = OA._Run(ocfg, ocoeff or OA.Coeff())
    r1, r2, dwq = OA.build_rules(run, True)

    def conv(basis, rs, d, u=None):
        k0, wptr, w = rs.packed()
        return rules_from_arrays(basis, rs.layout.points, rs.layout.offsets, k0, wptr, w, d, u)

    b1, b2 = b2d.dir
    pd = {(d, u): conv((b1, b2)[d], rs, d, u) for (d, u), rs in dwq.items()}
    return conv(b1, r1, 0), conv(b2, r2, 1), pd


def golden_rows(M, d, s):
    rows = d[f"{s}_rows"]
    got = np.concatenate([M.data[M.indptr[r]:M.indptr[r + 1]] for r in rows])
    return got, d[f"{s}_rowsdata"]


@pytest.mark.parametrize("tag", TAGS)
def test_trimmed_matches_reference(tag):
    import paper_2101_08053_b200 as P
    d = G.load(tag)
    desc = G.describe(tag)
    b2d, cfg, coeff = product_case(desc)
    # classification: bit-exact
    assert np.array_equal(cfg.element_class, d["element_class"])
    assert np.array_equal(cfg.func_class, d["func_class"])
    assert np.array_equal(cfg.u_disc[0], d["u_disc1"]) and np.array_equal(cfg.u_disc[1], d["u_disc2"])
    assert np.array_equal(cfg.active_functions(), d["active"])
    # host-native cut-cell rule
    if d["cut_el"].size:
        rule = cfg.cut_cell_rule(desc["p"])
        assert np.array_equal(rule.elements, d["cut_el"])
        assert np.array_equal(rule.ptr, d["cut_ptr"])
        assert np.max(np.abs(rule.points - d["cut_pts"])) <= 1e-13
        # host geometry input: weights of sliver sub-cells inherit ulp-level
        # point differences amplified by their small Jacobian (measured up to
        # 5.5e-10 relative on 1e-9-sized weights at 128^2, p=4)
        assert np.max(np.abs(rule.weights - d["cut_w"])) <= 1e-12 * np.max(np.abs(d["cut_w"]))
        assert np.max(np.abs(rule.weights - d["cut_w"]) / np.abs(d["cut_w"])) <= 1e-8
    full = f"{G.strategies_in(d)[0]}_data" in d
    trimmed = d["cut_el"].size > 0
    for s in G.strategies_in(d):
        weight_sensitive = s != "reference" and (coeff is not None or (s == "wq" and trimmed))
        # (a) the product path as shipped: the GPU's OWN weights (k_wq_solve
        #     pivots exactly as LAPACK dgeqp3, wq.cu) and the native cut-cell
        #     rule -- pattern exact, values within 1e-12.  Weight-sensitive
        #     matrices at p = 8 get 1e-10 on the sampled rows: the p = 8 moment
        #     systems reach condition 7e8, which amplifies the last-bit
        #     differences between OpenBLAS's kernel arithmetic and the GPU's
        #     into ~1e-11 of a few weights (pivots identical; measured max
        #     1.3e-11, scripts/probes/weights_gap.py).
        tol = 1e-10 if (weight_sensitive and desc["p"] >= 8) else 1e-12
        M = P.assemble_mass(b2d, cfg, coeff, strategy=s).data
        assert sha(M.indptr, M.indices) == str(d[f"{s}_hash"]), s
        if full:
            R = sp.csr_matrix((d[f"{s}_data"], d[f"{s}_indices"], d[f"{s}_indptr"]), shape=M.shape)
            assert np.linalg.norm(M.data - R.data) <= tol * np.linalg.norm(R.data)
        else:
            got, ref = golden_rows(M, d, s)
            assert np.max(np.abs(got - ref)) <= tol * np.max(np.abs(ref))
            assert abs(sp.linalg.norm(M) - float(d[f"{s}_fro"])) <= 1e-12 * float(d[f"{s}_fro"])
        rules = imported_rules(b2d, desc) if weight_sensitive else None
        if rules is not None:
            # (a') kernels alone: the reference's weight tables imported, 1e-12
            M = P.assemble_mass(b2d, cfg, coeff, strategy=s, rules=rules).data
            if full:
                assert np.linalg.norm(M.data - R.data) <= 1e-12 * np.linalg.norm(R.data)
            else:
                got, ref = golden_rows(M, d, s)
                assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))
        # (b) kernels alone: the reference's own cut-cell points injected,
        #     per-entry bar |dM_ij| <= 1e-12 sqrt(M_ii M_jj)
        if full and trimmed:
            inject_golden_cut_rule(cfg, d, desc["p"])
            M2 = P.assemble_mass(b2d, cfg, coeff, strategy=s, rules=rules).data
            cfg._cut_rules.clear()
            assert_matrix_close(M2, R)
        elif full:
            assert_matrix_close(M, R)


def inject_golden_cut_rule(cfg, d, q):
    from paper_2101_08053_b200._classify import CutCellRule
    ncell = np.zeros(d["cut_el"].shape[0], np.int32)
    cfg._cut_rules[q] = CutCellRule(q, d["cut_el"], d["cut_ptr"], d["cut_pts"], d["cut_w"], ncell)


def product_target(desc):
    from paper_2101_08053_b200 import cases as C
    from paper_2101_08053_b200.projection import default_target
    return {"default": default_target, "config1": C.f_config1, "config23": C.f_config23,
            "config5": C.f_config5}[desc["target"]]


RHS_TAGS = [t for t in TAGS if "rhs" in G.load(t)]


@pytest.mark.parametrize("tag", RHS_TAGS)
def test_rhs_and_l2_error_match_reference(tag):
    """assemble_rhs: max|db| <= 1e-12 max|b| and |db_i| <= 1e-12 sum_j |M_ij|;
    l2_error of the reference's own solution within 1e-10
    (src/projection.py:101-145, 221-260)."""
    import paper_2101_08053_b200 as P
    d = G.load(tag)
    desc = G.describe(tag)
    b2d, cfg, coeff = product_case(desc)
    target = product_target(desc)
    prob = P.ProjectionProblem(target, b2d, cfg, coeff=coeff)
    b = P.assemble_rhs(prob)
    ref = d["rhs"]
    assert np.max(np.abs(b - ref)) <= 1e-12 * np.max(np.abs(ref))
    s = G.strategies_in(d)[-1]
    if f"{s}_data" in d:
        # per-entry bar with the reference's own cut-cell points (kernels alone)
        if d["cut_el"].size:
            inject_golden_cut_rule(cfg, d, desc["p"])
            b = P.assemble_rhs(prob)
            cfg._cut_rules.clear()
        R = sp.csr_matrix((d[f"{s}_data"], d[f"{s}_indices"], d[f"{s}_indptr"]), shape=(ref.size, ref.size))
        rowabs = np.asarray(abs(R).sum(axis=1)).ravel()
        assert np.all(np.abs(b - ref) <= 1e-12 * rowabs + 1e-300)
    if "l2" in d:
        e = P.l2_error(d["x"], prob)
        assert abs(e - float(d["l2"])) <= 1e-10


def test_rhs_host_callable_target_matches_device_target():
    """A plain Python callable target (evaluated on the host at the Gauss
    points) gives the same load vector as the in-kernel separable target."""
    import paper_2101_08053_b200 as P
    from paper_2101_08053_b200 import cases as C
    b2d, cfg = C.build_space(None, 16, 3, curves=[C.closed_circle()])
    dev_t = C.f_config5
    host_t = lambda Q: np.sin(2 * np.pi * Q[:, 0]) * np.cos(3 * np.pi * Q[:, 1])
    b1 = P.assemble_rhs(P.ProjectionProblem(dev_t, b2d, cfg))
    b2 = P.assemble_rhs(P.ProjectionProblem(host_t, b2d, cfg))
    assert np.max(np.abs(b1 - b2)) <= 1e-13 * np.max(np.abs(b1))


def test_project_reproduces_spline_target():
    """pkg/tests/test_projection.py:57-73 analogue: a member of the trimmed
    space projects onto itself (L2 error <= 1e-12)."""
    import paper_2101_08053_b200 as P
    from paper_2101_08053_b200 import cases as C
    b2d, cfg = C.build_space("line", 8, 2)
    b1, b2 = b2d.dir
    rng = np.random.default_rng(12)
    coeffs = rng.standard_normal((b1.n, b2.n))

    def spline(Q):
        Q = np.atleast_2d(Q)
        return np.einsum("ki,kj,ij->k", b1.collocation(Q[:, 0]), b2.collocation(Q[:, 1]), coeffs)

    prob = P.ProjectionProblem(spline, b2d, cfg, strategy="hybrid")
    x, M, _ = P.project(prob)
    assert P.l2_error(x, prob, active=M.active) <= 1e-12
