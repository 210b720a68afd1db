"""One fresh-configuration public-API call (classify + cut cells + form +
host CSR) on config 5 inside a profiler range, after warm calls (for
`ncu --profile-from-start off`) -- dev aid for the e2e path."""
import sys, time; sys.path.insert(0, ".")
import torch
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import cases as C, trimming as T
c5 = C.baseline_config(5)
knots = P.make_uniform_knots(2048, 4).knots.copy(); ctrl = c5["curves"][0].ctrl.copy()
def call():
    t0 = time.perf_counter()
    bb = P.TensorBasis2D(P.Basis1D(P.KnotVector(knots.copy(), 4)), P.Basis1D(P.KnotVector(knots.copy(), 4)))
    cf = P.classify_elements(bb, [T.PeriodicBSplineTrim(ctrl.copy())])
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    cf.cut_cell_rule(4)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    M = P.assemble_mass(bb, cf, None, strategy="dwq")
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    return M, (round(t1 - t0, 4), round(t2 - t1, 4), round(t3 - t2, 4))
for _ in range(2):
    call()
import numpy as np
ts = np.array([call()[1] for _ in range(12)])
print("classify / cut cells / assemble_mass s: median", np.median(ts, 0), "min", ts.min(0))
if "prof" in sys.argv:
    torch.cuda.cudart().cudaProfilerStart()
    call()
    torch.cuda.cudart().cudaProfilerStop()
