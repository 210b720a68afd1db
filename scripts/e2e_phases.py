"""Host wall time per public-API phase of one fresh-configuration call on
config 5 (wrapped entry points, no added syncs: host time, with the GPU
running behind) -- dev aid for the e2e path."""
import collections, functools, sys, time; sys.path.insert(0, ".")
import torch
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import cases as C, trimming as T, assembly as A, _rawrows as R, quadrature as Q
from paper_2101_08053_b200 import _classify as K, splines as S
acc = collections.defaultdict(float)
def wrap(mod, name, label=None):
    fn = getattr(mod, name)
    @functools.wraps(fn)
    def w(*a, **k):
        t = time.perf_counter()
        try:
            return fn(*a, **k)
        finally:
            acc[label or name] += time.perf_counter() - t
    setattr(mod, name, w)
for mod, name in [(A, "form"), (R, "build_all_rules"), (R, "run_phase"), (A.Formation, "finish"),
                  (A.DeviceCSR, "to_scipy"), (K, "cut_cell_rule_device"), (Q, "dwq_layout"), (R, "prelaunch_geometry"), (A, "SparseMatrix"), (T.TrimConfiguration, "active_functions"), (R, "cut_point_tables"), (R, "_plan"),
                  (A.Formation, "interior_products"), (Q, "_solve_rows_async"), (Q, "dwq_solve_async")]:
    wrap(mod, name)
c5 = C.baseline_config(5)
knots = P.make_uniform_knots(2048, 4).knots.copy(); ctrl = c5["curves"][0].ctrl.copy()
def call():
    t0 = time.perf_counter()
    bb = P.TensorBasis2D(P.Basis1D(P.KnotVector(knots.copy(), 4)), P.Basis1D(P.KnotVector(knots.copy(), 4)))
    t1 = time.perf_counter()
    cf = P.classify_elements(bb, [T.PeriodicBSplineTrim(ctrl.copy())])
    t2 = time.perf_counter()
    M = P.assemble_mass(bb, cf, None, strategy="dwq")
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    return dict(basis=t1 - t0, classify=t2 - t1, assemble=t3 - t2)
for _ in range(3):
    call()
acc.clear()
n = 5
tot = collections.defaultdict(float)
for _ in range(n):
    for k, v in call().items():
        tot[k] += v
for k, v in list(tot.items()) + sorted(acc.items(), key=lambda x: -x[1]):
    print(f"{k:28s} {1e3 * v / n:8.2f} ms")
