"""Cut-cell decomposition on the device (tq_cutcell_device) against the host
C++ decomposition it restates (and, through tests/test_gpu_trimmed.py, the
reference's golden rules): same elements, offsets and sub-cell counts; points
and weights identical up to libm-vs-CUDA ulps in the curve transcendentals."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _space(kind, nel, p):
    from paper_2101_08053_b200 import cases as C
    if kind == "ccircle":
        return C.build_space(None, nel, p, curves=[C.closed_circle()])
    if kind == "bspline":
        return C.build_space(None, nel, p, curves=C.baseline_config(5)["curves"])
    return C.build_space(kind, nel, p)


@pytest.mark.parametrize("kind,nel,q", [("line", 10, 3), ("circle", 12, 2), ("corner", 10, 3), ("corner", 40, 6),
                                        ("ccircle", 64, 3), ("bspline", 128, 4), ("bspline", 32, 8)])
def test_device_matches_host_decomposition(kind, nel, q):
    from paper_2101_08053_b200 import _classify as K
    b2d, cfg = _space(kind, nel, min(q, 6))
    rd = K.cut_cell_rule_device(cfg, q)
    rh = K.cut_cell_rule(cfg, q, host_only=True)
    assert np.array_equal(rd.elements, rh.elements)
    assert np.array_equal(rd.ptr, rh.ptr)
    assert np.array_equal(rd._ncells, rh._ncells)
    # the golden-rule tolerances of tests/test_gpu_trimmed.py
    assert np.max(np.abs(rd.points - rh.points), initial=0.0) <= 1e-13
    assert np.max(np.abs(rd.weights - rh.weights), initial=0.0) <= 1e-12 * max(np.max(np.abs(rh.weights), initial=0), 1e-300)
    if kind in ("line", "bspline"):        # no transcendental functions on these paths
        assert np.array_equal(rd.points, rh.points) and np.array_equal(rd.weights, rh.weights)


def test_product_uses_device_rule():
    b2d, cfg = _space("ccircle", 32, 3)
    rule = cfg.cut_cell_rule(3)
    assert getattr(rule, "dev", None) is not None and rule.total_points() > 0
    # valid area = interior elements + cut cells (q = 3 cells interpolate the circle: ~1e-7)
    assert abs(rule.weights.sum() - (1.0 - np.pi * 0.09) - _interior_area(cfg)) < 1e-6


def _interior_area(cfg):
    b1, b2 = cfg.basis2d.dir
    h1, h2 = np.diff(b1.breakpoints), np.diff(b2.breakpoints)
    area_int = float(np.sum(np.outer(h1, h2)[cfg.element_class == 0]))
    return -area_int
