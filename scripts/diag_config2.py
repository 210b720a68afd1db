import sys; sys.path.insert(0, ".")
import numpy as np, scipy.sparse as sp
from tests import golden_cases as G
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import cases as C
d = G.load("config2")
b2d, cfg = C.build_space(None, 64, 3, curves=[C.closed_circle()])
rule = cfg.cut_cell_rule(3)
print("cut pts maxdiff", np.max(np.abs(rule.points - d["cut_pts"])), "w maxrel", np.max(np.abs(rule.weights - d["cut_w"]) / np.abs(d["cut_w"])))
for s in ("hybrid", "dwq"):
    M = P.assemble_mass(b2d, cfg, strategy=s).data
    R = sp.csr_matrix((d[f"{s}_data"], d[f"{s}_indices"], d[f"{s}_indptr"]), shape=M.shape)
    dd = M.data - R.data
    diag = R.diagonal()
    rows = np.repeat(np.arange(R.shape[0]), np.diff(R.indptr))
    sc = np.sqrt(np.abs(diag[rows] * diag[R.indices]))
    ratio = np.abs(dd) / sc
    k = np.argmax(ratio)
    print(s, "relfro", np.linalg.norm(dd) / np.linalg.norm(R.data), "max ratio", ratio[k], "at", rows[k], R.indices[k],
          "val", R.data[k], "diag", diag[rows[k]], diag[R.indices[k]], "n>1e-12", int(np.sum(ratio > 1e-12)))
    fc = cfg.func_class[cfg.active_functions()[:, 0], cfg.active_functions()[:, 1]]
    print("  classes of worst", fc[rows[k]], fc[R.indices[k]])
