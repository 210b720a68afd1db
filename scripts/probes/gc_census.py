"""gc-tracked objects alive after the public-API e2e loop, and what a full
collection costs (dev aid for the e2e step spikes)."""
import collections, gc, sys, time; sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import cases as C
c5 = C.baseline_config(5)
knots = np.ascontiguousarray(P.make_uniform_knots(2048, 4).knots)
ctrl = np.ascontiguousarray(c5["curves"][0].ctrl)
def census(tag):
    objs = gc.get_objects()
    t = time.perf_counter(); n = gc.collect(); dt = time.perf_counter() - t
    cnt = collections.Counter(type(o).__name__ for o in objs)
    print(tag, "tracked", len(objs), "collect_ms", round(1e3 * dt, 1), "freed", n, cnt.most_common(12), flush=True)
census("import")
for k in range(3):
    bb = P.TensorBasis2D(P.Basis1D(P.KnotVector(knots.copy(), 4)), P.Basis1D(P.KnotVector(knots.copy(), 4)))
    cf = P.classify_elements(bb, [P.trimming.PeriodicBSplineTrim(ctrl.copy())])
    M = P.assemble_mass(bb, cf, None, strategy="dwq")
    del M
    census(f"step{k}")
gc.freeze()
t = time.perf_counter(); gc.collect(); print("after freeze collect_ms", round(1e3 * (time.perf_counter() - t), 1))
