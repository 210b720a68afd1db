"""Known-answer properties the reference's own test suite asserts
(pkg/tests/test_assembly.py, test_projection.py, test_splines.py,
test_quadrature.py), run on the GPU product path: Kronecker structure of the
untrimmed matrix, partition-of-unity row sums, exact symmetry, strategy
agreement, basis and moment values, and the L2-projection convergence
rates with strategy agreement <= 1e-10."""

import math

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu


def _P():
    import paper_2101_08053_b200 as P
    from paper_2101_08053_b200 import cases as C
    return P, C


@pytest.mark.parametrize("strategy", ["reference", "wq", "hybrid", "dwq"])
def test_untrimmed_matrix_is_kron_of_1d_mass(strategy):
    P, C = _P()
    b2d, cfg = C.build_space(None, 6, 2, curves=[])
    M = P.assemble_mass(b2d, cfg, strategy=strategy).data.toarray()
    A1 = P.mass_matrix_1d(b2d.dir[0])
    assert np.max(np.abs(M - np.kron(A1, A1))) <= 1e-15


def test_uniform_quadratic_midpoint_values():
    P, _ = _P()
    b = P.make_uniform_basis(4, 2)
    first, vals = b.eval_nonzero_batch(np.array([0.375]))        # midpoint of element 1
    assert int(first[0]) == 1
    assert np.allclose(vals[0], [0.125, 0.75, 0.125], atol=1e-15)


def test_exact_moments_known_values():
    P, _ = _P()
    lin = P.make_uniform_basis(1, 1)                                 # [0,1], degree 1
    assert np.allclose(P.mass_matrix_1d(lin), [[1 / 3, 1 / 6], [1 / 6, 1 / 3]], atol=1e-15)
    quad = P.make_uniform_basis(1, 2)
    assert abs(P.mass_matrix_1d(quad)[0, 0] - 0.2) <= 1e-15         # int (1-x)^4 = 1/5


@pytest.mark.parametrize("case", ["line", "circle", "corner"])
def test_row_sums_equal_loads_of_one(case):
    P, C = _P()
    b2d, cfg = C.build_space(case, 10, 2)
    M = P.assemble_mass(b2d, cfg, strategy="reference").data
    ones = lambda X: np.ones(np.atleast_2d(X).shape[0])
    b = P.assemble_rhs(P.ProjectionProblem(ones, b2d, cfg))
    assert np.max(np.abs(np.asarray(M.sum(axis=1)).ravel() - b)) <= 1e-12


@pytest.mark.parametrize("strategy", ["reference", "hybrid", "dwq", "wq"])
@pytest.mark.parametrize("case", ["line", "circle", "corner", "bspline"])
def test_symmetry_and_positive_definiteness(strategy, case):
    P, C = _P()
    if case == "bspline":
        b2d, cfg = C.build_space(None, 64, 3, curves=C.baseline_config(5)["curves"])
    else:
        b2d, cfg = C.build_space(case, 10, 3)
    M = P.assemble_mass(b2d, cfg, strategy=strategy).data
    D = (M - M.T).tocsr()
    D.eliminate_zeros()
    assert D.nnz == 0                                     # exactly symmetric (reference bound: 1e-12 ||M||)
    # positive definiteness: Gauss-exact strategies (naive WQ on trimmed
    # spaces is the paper's failure case: the reference's own wq matrix of the
    # line case at 10^2, p = 3 has eigenvalues down to -0.04 after scaling,
    # and so does this one now that the fits pivot as LAPACK does; the
    # reference checks `reference` only)
    if M.shape[0] <= 4000 and strategy != "wq":
        A = M.toarray()
        s = 1.0 / np.sqrt(np.diag(A))
        np.linalg.cholesky(0.5 * (A + A.T) * np.outer(s, s))


def test_fast_strategies_agree_with_reference():
    P, C = _P()
    for case in ("line", "circle", "corner"):
        b2d, cfg = C.build_space(case, 12, 3)
        R = P.assemble_mass(b2d, cfg, strategy="reference").data
        for s in ("hybrid", "dwq"):
            M = P.assemble_mass(b2d, cfg, strategy=s).data
            assert sp.linalg.norm(M - R) <= 1e-12 * sp.linalg.norm(R), (case, s)


@pytest.mark.timeout(600)
def test_line_p3_convergence_rate_and_agreement():
    P, _ = _P()
    recs = P.run_convergence_study("line", ["reference", "hybrid", "dwq"], [3], [5, 10, 20, 40])
    by = {}
    for r in recs:
        by.setdefault(r.strategy, []).append(r)
    for strategy, rs in by.items():
        rs = sorted(rs, key=lambda r: r.mesh)
        assert abs(rs[-1].rate - 4.0) <= 0.2, strategy
        errs = [r.l2_rel for r in rs]
        assert all(e2 < e1 for e1, e2 in zip(errs, errs[1:]))
    ref = {r.mesh: r.l2_rel for r in by["reference"]}
    for s in ("hybrid", "dwq"):
        for r in by[s]:
            assert abs(r.l2_rel - ref[r.mesh]) <= 1e-10


def test_untrimmed_p2_projection_rate():
    P, C = _P()
    errs = []
    for nel in (5, 10, 20, 40):
        b2d, cfg = C.build_space(None, nel, 2, curves=[])
        prob = P.ProjectionProblem(P.projection.default_target, b2d, cfg)
        x, M, _ = P.project(prob)
        errs.append(P.l2_error(x, prob, active=M.active))
    rate = math.log(errs[-2] / errs[-1]) / math.log(2)
    assert abs(rate - 3.0) <= 0.2
