"""Breakdown of the end-to-end public-API path on config 5 (dev aid)."""
import sys, time; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import cases as C, trimming as T
from paper_2101_08053_b200.assembly import form
c5 = C.baseline_config(5)
knots = P.make_uniform_knots(2048, 4).knots.copy(); ctrl = c5["curves"][0].ctrl.copy()
def run():
    t = [time.perf_counter()]
    bb = P.TensorBasis2D(P.Basis1D(P.KnotVector(knots, 4)), P.Basis1D(P.KnotVector(knots, 4)))
    cf = P.classify_elements(bb, [T.PeriodicBSplineTrim(ctrl)]); torch.cuda.synchronize(); t.append(time.perf_counter())
    if "sync" in sys.argv:
        cf.cut_cell_rule(4)
    t.append(time.perf_counter())    # cut cells: built inside form (worker thread) unless "sync"
    f, csr = form(bb, cf, None, "dwq"); torch.cuda.synchronize(); t.append(time.perf_counter())
    h = csr.to_host(); t.append(time.perf_counter())
    import scipy.sparse as sp
    M = sp.csr_matrix((h[2], h[1], h[0]), shape=(f.K, f.K)); t.append(time.perf_counter())
    act = cf.active_functions(); t.append(time.perf_counter())
    r = f.report
    print("  phases: weights %.1f interior %.1f cut %.1f cutel %.1f finish %.1f ms" % (
        r.t_weights * 1e3, r.t_interior * 1e3, r.t_cut_regular * 1e3, r.t_cut_elements * 1e3, r.t_finish * 1e3))
    return np.diff(t)
for k in range(3):
    d = run()
import gc
gct = []
_t = [0.0]
def _cb(phase, info):
    if phase == "start": _t[0] = time.perf_counter()
    else: gct.append((info["generation"], time.perf_counter() - _t[0]))
gc.callbacks.append(_cb)
tot = []
for k in range(6):
    d = run(); tot.append(d.sum())
    print("classify %.3f cutcells %.3f form %.3f d2h %.3f scipy %.3f active %.3f total %.3f" % (*d, d.sum()))
print("median total %.1f ms" % (1e3 * np.median(tot)))
print("gc pauses (gen, ms):", [(g, round(1e3 * d, 1)) for g, d in gct if d > 1e-3])
