"""Behaviours the reference's own tests assert (pkg/tests/test_assembly.py,
test_trimming.py), on the GPU drop-in: identical patterns across strategies,
hybrid == wq without cuts, constant-coefficient scaling, the naive-WQ error
confined to cut rows, the report's components and Gauss footprint, and the
error conventions (floating curve, cut-cell degree)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

STRATEGIES = ("reference", "wq", "hybrid", "dwq")


def _P():
    import paper_2101_08053_b200 as P
    from paper_2101_08053_b200 import cases as C
    return P, C


@pytest.mark.parametrize("name", ["line", "circle", "corner"])
def test_sparsity_pattern_identical_across_strategies(name):
    P, C = _P()
    b2d, cfg = C.build_space(name, 8, 2)
    mats = [P.assemble_mass(b2d, cfg, strategy=s).data for s in STRATEGIES]
    for M in mats[1:]:
        assert np.array_equal(M.indptr, mats[0].indptr) and np.array_equal(M.indices, mats[0].indices)


def test_hybrid_equals_wq_when_untrimmed():
    P, C = _P()
    b2d, cfg = C.build_space(None, 5, 2, curves=[])
    Mh = P.assemble_mass(b2d, cfg, strategy="hybrid").data
    Mw = P.assemble_mass(b2d, cfg, strategy="wq").data
    assert (Mh != Mw).nnz == 0


@pytest.mark.parametrize("strategy", ["reference", "dwq"])
def test_constant_coefficient_scales(strategy):
    P, C = _P()
    b2d, cfg = C.build_space(None, 5, 2, curves=[])
    M1 = P.assemble_mass(b2d, cfg, strategy=strategy).toarray()
    c = P.CoefficientField(lambda X: np.full(np.atleast_2d(X).shape[0], 2.5))
    M2 = P.assemble_mass(b2d, cfg, coeff=c, strategy=strategy).toarray()
    assert np.max(np.abs(M2 - 2.5 * M1)) <= 1e-14


def test_wq_failure_is_localized_to_cut_rows():
    P, C = _P()
    from paper_2101_08053_b200.trimming import ElementClass
    b2d, cfg = C.build_space("line", 10, 3)
    ref = P.assemble_mass(b2d, cfg, strategy="reference")
    M = P.assemble_mass(b2d, cfg, strategy="wq")
    diff = (M.data - ref.data).toarray()
    fclass = cfg.func_class[M.active[:, 0], M.active[:, 1]]
    interior = fclass == ElementClass.INTERIOR
    assert np.max(np.abs(diff[np.ix_(interior, interior)])) <= 1e-12
    assert np.max(np.abs(diff)) > 1e-6


def test_report_components_and_reference_weight_setup():
    P, C = _P()
    b2d, cfg = C.build_space("line", 8, 3)
    for s in STRATEGIES:
        _, rep = P.form_with_timings(s, b2d, cfg)
        assert all(t >= 0 for t in rep.components())
        assert rep.t_total >= sum(rep.components()) - 1e-9
        assert rep.t_total <= sum(rep.components()) + 0.25 * rep.t_total + 0.05
    _, rep = P.form_with_timings("reference", b2d, cfg)
    assert rep.n_wq_points == 0


def test_gauss_footprint_grows_with_degree():
    P, C = _P()
    counts = {}
    for p in (2, 6):
        b2d, cfg = C.build_space("circle", 8, p)
        _, rep = P.form_with_timings("hybrid", b2d, cfg)
        counts[p] = rep.n_gauss_elements
        if p == 6:
            assert rep.n_gauss_elements == len(cfg.interior_elements)
    assert counts[6] >= counts[2]


def test_floating_curve_is_rejected():
    P, _ = _P()
    from paper_2101_08053_b200.trimming import CircleTrim, TrimmingConfigurationError
    basis = P.make_uniform_basis(2, 1)
    with pytest.raises(TrimmingConfigurationError):
        P.classify_elements(P.TensorBasis2D(basis, basis), [CircleTrim((0.25, 0.25), 0.1, 0.0, 0.4)])


def test_cut_cell_degree_out_of_range():
    P, C = _P()
    b2d, cfg = C.build_space("circle", 6, 2)
    with pytest.raises(ValueError):
        cfg.cut_cell_rule(0)
    with pytest.raises(ValueError):
        cfg.cut_cell_rule(11, cache=False)
