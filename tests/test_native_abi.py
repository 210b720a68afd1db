"""CPU-side checks of the native library and the host logic (no GPU).

* the in-tree library loads and exports every entry point include/*.h
  declares (no compute call is made);
* the host-native cut-cell decomposition (C++, runs on the CPU) reproduces
  the reference's cut-cell rules on the golden cases;
* the host point-layout / knot-insertion / DWQ-layout logic of the product
  matches the oracle restatement bit for bit.
"""

import os
import re

import numpy as np
import pytest

from tests import golden_cases as G

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "trimquad_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|void\*|void|int64_t|long long|const char\*)\s+(tq_\w+)\s*\(",
                                 text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2101_08053_b200 import _lib
    lib = _lib.lib()
    names = declared_functions()
    assert len(names) >= 29
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.tq_version() >= 1


def test_library_is_sm100a_only():
    """The fatbin carries sm_100a SASS (cross-compiled here, no GPU)."""
    import subprocess
    from paper_2101_08053_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


class _HostConfig:
    """Just what the host cut-cell builder reads from a TrimConfiguration."""

    def __init__(self, basis2d, element_class, curves):
        self.basis2d = basis2d
        self.element_class = element_class
        self.curves = curves


def _product_curves(desc):
    from paper_2101_08053_b200 import cases as C
    if desc["kind"] == "case":
        return [C.make_case(desc["name"]).curve()]
    if desc["kind"] == "ccircle":
        return [C.closed_circle()]
    if desc["kind"] == "bspline":
        return C.baseline_config(4)["curves"]
    return []


@pytest.mark.parametrize("tag", list(G.tags()))
def test_host_cut_cell_rule_matches_reference(tag):
    import paper_2101_08053_b200 as P
    from paper_2101_08053_b200 import _classify
    d = G.load(tag)
    if d["cut_el"].size == 0:
        pytest.skip("untrimmed")
    desc = G.describe(tag)
    b = P.make_uniform_basis(desc["nel"], desc["p"])
    b2d = P.TensorBasis2D(b, P.make_uniform_basis(desc["nel"], desc["p"]))
    rule = _classify.cut_cell_rule(_HostConfig(b2d, d["element_class"], _product_curves(desc)), desc["p"])
    assert np.array_equal(rule.elements, d["cut_el"])
    assert np.array_equal(rule.ptr, d["cut_ptr"])
    assert np.max(np.abs(rule.points - d["cut_pts"])) <= 1e-13
    assert np.max(np.abs(rule.weights - d["cut_w"])) <= 1e-12 * np.max(np.abs(d["cut_w"]))


@pytest.mark.parametrize("nel,p", [(9, 1), (16, 2), (64, 3), (12, 8), (128, 4)])
def test_host_layouts_and_dwq_geometry_match_oracle(nel, p):
    import paper_2101_08053_b200 as P
    from paper_2101_08053_b200 import quadrature as Q
    from oracle import bspline as OB
    from oracle import quad as OQ
    b = P.make_uniform_basis(nel, p)
    s = OB.uniform_space(nel, p)
    lay = P.place_wq_points(b)
    olay = OQ.place_wq_points(s)
    assert np.array_equal(lay.points, olay.points) and np.array_equal(lay.offsets, olay.offsets)
    for u in (float(b.breakpoints[nel // 2]), float(b.breakpoints[1])):
        refined, S, aug = Q.dwq_layout(b, lay, u)
        oref, oS, oaug = OQ.dwq_layout(s, olay, u)
        assert np.array_equal(refined.kv.knots, oref.knots)
        assert np.array_equal(aug.points, oaug.points) and np.array_equal(aug.offsets, oaug.offsets)
        assert abs(S.matrix - oS).max() == 0.0


def test_knot_vector_validation_errors():
    import paper_2101_08053_b200 as P
    with pytest.raises(ValueError):
        P.KnotVector([0, 0, 1, 1], 2)
    with pytest.raises(ValueError):
        P.KnotVector([0, 0, 0.5, 0.2, 1, 1], 1)
    with pytest.raises(ValueError):
        P.KnotVector([0, 0, 0.5, 0.5, 0.5, 1, 1], 1)
    kv = P.KnotVector([0, 0, 0, 0.25, 0.5, 0.5, 0.75, 1, 1, 1], 2)
    assert kv.multiplicity_of(0.5) == 2 and kv.num_elements == 4
    with pytest.raises(ValueError):
        kv.find_spans(np.array([1.5]))
