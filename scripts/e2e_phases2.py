"""Finer host wall time per function of one fresh-configuration call on
config 5 (inclusive times; wrappers nest) -- dev aid for the e2e path."""
import collections, functools, sys, time; sys.path.insert(0, ".")
import torch
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import cases as C, trimming as T, assembly as A, _rawrows as R, quadrature as Q
from paper_2101_08053_b200 import _classify as K, splines as S, _lib as L
acc = collections.defaultdict(float); cnt = collections.defaultdict(int)
def wrap(mod, name, label=None):
    fn = getattr(mod, name)
    lab = label or (getattr(mod, "__name__", "").split(".")[-1] + "." + name)
    @functools.wraps(fn)
    def w(*a, **k):
        t = time.perf_counter()
        try:
            return fn(*a, **k)
        finally:
            acc[lab] += time.perf_counter() - t; cnt[lab] += 1
    setattr(mod, name, w)
for mod, names in [
    (A, ["form"]), (A.Formation, ["__init__", "finish", "build_weights", "interior_products", "_alloc_out", "rowctx"]),
    (A.DeviceCSR, ["to_host"]),
    (R, ["build_all_rules", "run_phase", "dwq_keys", "cut_point_tables", "_plan", "_plan_uncached", "_cut_tables",
         "_elem_tables", "route_cut_rows", "cut_rows_host", "element_points", "_desc_dev", "_FitPlan",
         "fit_sets_async", "combine_sets_async", "DwqPlan", "place_wq_points", "_key_index", "active_host"]),
    (R._Setup, ["__init__"]),
    (Q, ["dwq_layout", "_augment_nested", "_required_counts", "refine_to_c_minus_1", "_row_lengths"]),
    (Q.DwqPlan, ["_finalize"]),
    (S, ["_repeated_insertion"]), (S.Basis1D, ["__init__", "device"]), (S.KnotVector, ["__init__"]),
    (L, ["dev", "dev_many", "eval_many"]),
    (K, ["cut_cell_rule_device", "classify_device"]),
    (T.TrimConfiguration, ["active_functions", "cut_cell_rule_async"]),
]:
    for n in names:
        if hasattr(mod, n):
            wrap(mod, n)
        else:
            print("missing", mod, n)
_call = L.call
def call_named(name, *a):
    t = time.perf_counter()
    try:
        return _call(name, *a)
    finally:
        acc["call:" + name] += time.perf_counter() - t; cnt["call:" + name] += 1
for m in (L, A, R, Q, K, S, T):
    if getattr(m, "call", None) is _call:
        m.call = call_named
L.call = call_named
c5 = C.baseline_config(5)
knots = P.make_uniform_knots(2048, 4).knots.copy(); ctrl = c5["curves"][0].ctrl.copy()
def call():
    bb = P.TensorBasis2D(P.Basis1D(P.KnotVector(knots.copy(), 4)), P.Basis1D(P.KnotVector(knots.copy(), 4)))
    cf = P.classify_elements(bb, [T.PeriodicBSplineTrim(ctrl.copy())])
    t2 = time.perf_counter()
    M = P.assemble_mass(bb, cf, None, strategy="dwq")
    return time.perf_counter() - t2
for _ in range(3):
    call()
acc.clear(); cnt.clear()
n = 6
tot = sum(call() for _ in range(n))
print(f"assemble_mass {1e3 * tot / n:8.2f} ms")
for k, v in sorted(acc.items(), key=lambda x: -x[1]):
    print(f"{k:40s} {1e3 * v / n:8.3f} ms  x{cnt[k] / n:.0f}")
