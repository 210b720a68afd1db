"""Host profile of form() on a fresh configuration (dev aid)."""
import sys, time, cProfile, pstats; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import cases as C, trimming as T
from paper_2101_08053_b200.assembly import form
c5 = C.baseline_config(5)
knots = P.make_uniform_knots(2048, 4).knots.copy(); ctrl = c5["curves"][0].ctrl.copy()
def fresh():
    bb = P.TensorBasis2D(P.Basis1D(P.KnotVector(knots, 4)), P.Basis1D(P.KnotVector(knots, 4)))
    cf = P.classify_elements(bb, [T.PeriodicBSplineTrim(ctrl)])
    torch.cuda.synchronize()
    return bb, cf
for _ in range(2):
    bb, cf = fresh(); form(bb, cf, None, "dwq")
bb, cf = fresh()
pr = cProfile.Profile(); pr.enable()
f, csr = form(bb, cf, None, "dwq"); torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
