"""Per-call split of the e2e path (bench loop, gc frozen): form, pinned
allocation, copy launch, final sync -- where do the slow steps come from?"""
import gc, sys, time; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import assembly as A, cases as C, trimming as T
rec = {}
from paper_2101_08053_b200 import _rawrows as R, quadrature as Q
def wrap(mod, name):
    fn = getattr(mod, name)
    def w(*a, **k):
        t = time.perf_counter(); c = time.thread_time()
        try: return fn(*a, **k)
        finally:
            rec[name] = rec.get(name, 0.0) + time.perf_counter() - t
            rec[name + ".cpu"] = rec.get(name + ".cpu", 0.0) + time.thread_time() - c
    setattr(mod, name, w)
for m, n in [(R, "build_all_rules"), (R, "run_phase"), (A.Formation, "finish"), (A.Formation, "_alloc_out"),
             (R, "DwqPlan"), (R, "fit_sets_async"), (Q, "compute_wq_rules"), (Q, "build_dwq"), (R._Setup, "__init__")]:
    wrap(m, n)
gcs = []
def gccb(phase, info):
    if phase == "start": gcs.append([info["generation"], time.perf_counter()])
    else: gcs[-1][1] = time.perf_counter() - gcs[-1][1]
gc.callbacks.append(gccb)
_form = A.form
def form(*a, **k):
    t = time.perf_counter(); r = _form(*a, **k); rec["form"] = time.perf_counter() - t; return r
A.form = form
def to_host(self):
    t0 = time.perf_counter(); out = []
    hs = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in (self.indptr, self.indices, self.data)]
    t1 = time.perf_counter()
    torch.cuda.current_stream().synchronize()
    t2 = time.perf_counter()
    for h, t in zip(hs, (self.indptr, self.indices, self.data)):
        h.copy_(t, non_blocking=True)
    t3 = time.perf_counter()
    torch.cuda.current_stream().synchronize()
    t4 = time.perf_counter()
    rec.update(pin=t1 - t0, gpu_tail=t2 - t1, launch=t3 - t2, d2h=t4 - t3)
    return tuple(h.numpy() for h in hs)
A.DeviceCSR.to_host = to_host
c5 = C.baseline_config(5)
knots = P.make_uniform_knots(2048, 4).knots.copy(); ctrl = c5["curves"][0].ctrl.copy()
gc.collect(); gc.freeze()
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 24):
    rec.clear(); gcs.clear(); ms0 = torch.cuda.memory_stats()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    bb = P.TensorBasis2D(P.Basis1D(P.KnotVector(knots.copy(), 4)), P.Basis1D(P.KnotVector(knots.copy(), 4)))
    cf = P.classify_elements(bb, [T.PeriodicBSplineTrim(ctrl.copy())])
    t1 = time.perf_counter()
    M = P.assemble_mass(bb, cf, None, strategy="dwq")
    t2 = time.perf_counter()
    del M; torch.cuda.synchronize()
    t3 = time.perf_counter()
    print("%2d total %6.1f classify %5.1f assemble %6.1f release %4.1f | " % (i, 1e3 * (t3 - t0), 1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2))
          + " ".join("%s %.1f" % (k, 1e3 * v) for k, v in rec.items())
          + " | gc " + " ".join("g%d:%.1f" % (g, 1e3 * d) for g, d in gcs if d > 5e-4)
          + " | dalloc %d dfree %d retries %d seg %d" % tuple(torch.cuda.memory_stats().get(k, 0) - ms0.get(k, 0) for k in ("num_device_alloc", "num_device_free", "num_alloc_retries", "segment.all.allocated")))
