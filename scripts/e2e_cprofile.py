"""cProfile of one fresh-configuration public-API call (classify + form +
host CSR) on config 5 after warm-up -- dev aid for the e2e path.
``split``: classification and the cut-cell rule outside the profile, so
it shows assemble_mass alone."""
import cProfile, pstats, sys, time; sys.path.insert(0, ".")
import torch
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import cases as C, trimming as T
c5 = C.baseline_config(5)
knots = P.make_uniform_knots(2048, 4).knots.copy(); ctrl = c5["curves"][0].ctrl.copy()
split = "split" in sys.argv
def prep():
    bb = P.TensorBasis2D(P.Basis1D(P.KnotVector(knots.copy(), 4)), P.Basis1D(P.KnotVector(knots.copy(), 4)))
    cf = P.classify_elements(bb, [T.PeriodicBSplineTrim(ctrl.copy())])
    return bb, cf
def call(bb=None, cf=None):
    if bb is None:
        bb, cf = prep()
    M = P.assemble_mass(bb, cf, None, strategy="dwq")
    torch.cuda.synchronize()
    return M
for _ in range(3):
    call()
args = ()
if split:
    args = prep()
    args[1].cut_cell_rule(4)
    torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter(); pr.enable(); call(*args); pr.disable(); print("call %.1f ms" % ((time.perf_counter() - t0) * 1e3))
st = pstats.Stats(pr); st.sort_stats("cumulative").print_stats(70)
st.sort_stats("tottime").print_stats(50)
