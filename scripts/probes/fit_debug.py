"""GPU fit vs the LAPACK emulation on one uniform space: basis values at the
layout points (bit equality) and the active sets of differing rows."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import _lib as L
from oracle import bspline as B, quad as Q
nel, p = int(sys.argv[1]), int(sys.argv[2])
b = P.make_uniform_basis(nel, p)
r = P.compute_wq_rules(b)
sp_ = B.uniform_space(nel, p)
lay = Q.place_wq_points(sp_)
assert np.array_equal(lay.points, r.layout.points)
f_o, V_o = sp_.eval_nonzero(lay.points)
f_g, V_g = b.eval_device(L.dev(lay.points, torch.float64), check=False)
f_g, V_g = f_g.cpu().numpy(), V_g.cpu().numpy()
print("first equal", np.array_equal(f_o, f_g), "vals bit-equal", np.array_equal(V_o, V_g),
      "max diff", np.max(np.abs(V_o - V_g)))
o = Q.compute_wq_rules(sp_, lay)
for i in range(b.n):
    kk, ww = r.row(i)
    ref = o.rows[i][1]
    if np.max(np.abs(ww - ref)) > 1e-12 * np.max(np.abs(ref)):
        print(i, "gpu nz", np.nonzero(ww)[0], "ref nz", np.nonzero(ref)[0])
