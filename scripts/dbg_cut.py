import sys; sys.path.insert(0, "/root/repo")
import numpy as np
from tests import golden_cases as G
from paper_2101_08053_b200 import _classify, cases as C
from paper_2101_08053_b200.splines import make_uniform_basis, TensorBasis2D
tag, nel, p = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
d = G.load(tag)
class Cfg: pass
cfg = Cfg()
b = make_uniform_basis(nel, p)
cfg.basis2d = TensorBasis2D(b, make_uniform_basis(nel, p))
cfg.element_class = d["element_class"]
cfg.curves = [C.closed_circle()] if "config3" in tag or "ccircle" in tag or "config2" in tag else C.baseline_config(4)["curves"]
rule = _classify.cut_cell_rule(cfg, p)
print("ptr equal", np.array_equal(rule.ptr, d["cut_ptr"]))
dw = np.abs(rule.weights - d["cut_w"])
dp = np.max(np.abs(rule.points - d["cut_pts"]), axis=1)
k = np.argmax(dw)
el = np.searchsorted(rule.ptr, k, side="right") - 1
print("max dw", dw[k], "w", d["cut_w"][k], rule.weights[k], "at elem", rule.elements[el], "pt", rule.points[k], d["cut_pts"][k], "maxdp", dp.max())
bad = np.unique(np.searchsorted(rule.ptr, np.nonzero(dw > 1e-15)[0], side="right") - 1)
print("bad elems", [tuple(rule.elements[e]) for e in bad[:10]], len(bad))
