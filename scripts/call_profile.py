"""Per-entry-point host time of _lib.call during form() on a fresh
configuration (dev aid)."""
import sys, time, collections; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import cases as C, trimming as T, _lib as L
from paper_2101_08053_b200.assembly import form
c5 = C.baseline_config(5)
knots = P.make_uniform_knots(2048, 4).knots.copy(); ctrl = c5["curves"][0].ctrl.copy()
def fresh():
    bb = P.TensorBasis2D(P.Basis1D(P.KnotVector(knots, 4)), P.Basis1D(P.KnotVector(knots, 4)))
    cf = P.classify_elements(bb, [T.PeriodicBSplineTrim(ctrl)])
    torch.cuda.synchronize()
    return bb, cf
orig = L.call
acc = collections.defaultdict(float); cnt = collections.Counter()
def timed(name, *a):
    t = time.perf_counter(); orig(name, *a); acc[name] += time.perf_counter() - t; cnt[name] += 1
for _ in range(2):
    bb, cf = fresh(); form(bb, cf, None, "dwq")
bb, cf = fresh()
L.call = timed
import paper_2101_08053_b200._rawrows as R, paper_2101_08053_b200.assembly as A, paper_2101_08053_b200.quadrature as Q, paper_2101_08053_b200.splines as S
for m in (R, A, Q, S):
    if hasattr(m, "L"): m.L.call = timed
t0 = time.perf_counter(); f, csr = form(bb, cf, None, "dwq"); torch.cuda.synchronize(); T0 = time.perf_counter() - t0
for k, v in sorted(acc.items(), key=lambda x: -x[1])[:15]:
    print(f"{v*1e3:8.2f} ms x{cnt[k]:3d} {k}")
print(f"form total {T0*1e3:.1f} ms")
