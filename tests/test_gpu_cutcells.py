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


@pytest.mark.parametrize("slot_cells", [1, 2])
@pytest.mark.parametrize("kind,nel,q", [("corner", 10, 3), ("bspline", 128, 4), ("ccircle", 64, 3)])
def test_slot_overflow_matches_two_pass(kind, nel, q, slot_cells):
    """Small slots force the re-decomposition of overflowing elements
    (tq_cutcell_device_pack, any_overflow); the packed rule equals the
    two-pass schedule (tq_cutcell_device) bit for bit."""
    import ctypes as Ct
    import torch
    from paper_2101_08053_b200 import _classify as K, _lib as L
    b2d, cfg = _space(kind, nel, min(q, 6))
    rd = K.cut_cell_rule_device(cfg, q, slot_cells=slot_cells)
    d = rd.dev
    n = np.diff(rd.ptr)
    assert slot_cells > 1 or n.max() > (q + 1) ** 2          # some element overflowed its slot
    # two-pass schedule on the same elements
    b1, b2 = cfg.basis2d.dir
    el = d["el"]
    ncut = el.shape[0]
    arr, keep = K.curve_array(cfg.curves)
    tabs = K.cell_tables(q)
    bp1, bp2 = b1.device_arrays()["bp"], b2.device_arrays()["bp"]
    ptr = torch.zeros(ncut + 1, dtype=torch.int64, device=el.device)
    nc = torch.zeros(ncut, dtype=torch.int32, device=el.device)
    st = torch.zeros(ncut, dtype=torch.int32, device=el.device)
    args = (arr, len(cfg.curves), L.ptr(bp1), L.ptr(bp2), L.ptr(el), ncut, q, tabs.ctypes.data_as(L.vp))
    L.call("tq_cutcell_device", *args, L.ptr(ptr), None, None, L.ptr(nc), L.ptr(st), L.stream())
    ptr[1:] = torch.cumsum(ptr[1:], 0)
    npts = int(ptr[-1])
    P = torch.empty((npts, 2), dtype=torch.float64, device=el.device)
    W = torch.empty(npts, dtype=torch.float64, device=el.device)
    L.call("tq_cutcell_device", *args, L.ptr(ptr), L.ptr(P), L.ptr(W), L.ptr(nc), L.ptr(st), L.stream())
    assert int(st.abs().sum()) == 0
    assert np.array_equal(rd.ptr, ptr.cpu().numpy())
    assert np.array_equal(rd._ncells, nc.cpu().numpy())
    assert np.array_equal(rd.points, P.cpu().numpy()) and np.array_equal(rd.weights, W.cpu().numpy())


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
