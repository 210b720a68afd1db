"""cProfile of one fresh-configuration public-API call (classify + form +
host CSR) on config 5 after warm-up -- dev aid for the e2e path."""
import cProfile, pstats, sys, time; sys.path.insert(0, ".")
import torch
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import cases as C, trimming as T
c5 = C.baseline_config(5)
knots = P.make_uniform_knots(2048, 4).knots.copy(); ctrl = c5["curves"][0].ctrl.copy()
def call():
    bb = P.TensorBasis2D(P.Basis1D(P.KnotVector(knots.copy(), 4)), P.Basis1D(P.KnotVector(knots.copy(), 4)))
    cf = P.classify_elements(bb, [T.PeriodicBSplineTrim(ctrl.copy())])
    M = P.assemble_mass(bb, cf, None, strategy="dwq")
    torch.cuda.synchronize()
    return M
for _ in range(3):
    call()
pr = cProfile.Profile()
t0 = time.perf_counter(); pr.enable(); call(); pr.disable(); print("call %.1f ms" % ((time.perf_counter() - t0) * 1e3))
st = pstats.Stats(pr); st.sort_stats("cumulative").print_stats(45)
st.sort_stats("tottime").print_stats(30)
