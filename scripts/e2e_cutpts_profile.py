"""cProfile of _rawrows.cut_point_tables and _Setup.__init__ inside a fresh config-5 call (dev aid)."""
import cProfile, pstats, sys, time; sys.path.insert(0, ".")
import torch
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import cases as C, trimming as T, _rawrows as R
pr = cProfile.Profile()
def prof(mod, name):
    fn = getattr(mod, name)
    def w(*a, **k):
        pr.enable()
        try: return fn(*a, **k)
        finally: pr.disable()
    setattr(mod, name, w)
prof(R._Setup, "__init__")
c5 = C.baseline_config(5)
knots = P.make_uniform_knots(2048, 4).knots.copy(); ctrl = c5["curves"][0].ctrl.copy()
def call():
    bb = P.TensorBasis2D(P.Basis1D(P.KnotVector(knots.copy(), 4)), P.Basis1D(P.KnotVector(knots.copy(), 4)))
    cf = P.classify_elements(bb, [T.PeriodicBSplineTrim(ctrl.copy())])
    return P.assemble_mass(bb, cf, None, strategy="dwq")
for _ in range(3): call()
pr.clear()
for _ in range(5): call()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(35)
st.sort_stats("cumulative").print_stats(30)
