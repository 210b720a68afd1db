"""Device bytes still allocated after each public-API call returns and its
result is dropped, with the cyclic collector disabled (0 = freed by
refcount; anything else waits for the collector) -- dev aid."""
import gc, sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import cases as C
def fresh(idx, **kw):
    c = C.baseline_config(idx, **kw)
    b2d, cfg = C.build_space(None, c["nel"], c["p"], curves=c["curves"])
    return c, b2d, cfg
def run(name, fn):
    for _ in range(2): fn()
    gc.collect(); torch.cuda.synchronize(); base = torch.cuda.memory_allocated()
    gc.disable(); fn(); torch.cuda.synchronize()
    left = torch.cuda.memory_allocated() - base
    gc.enable(); n = gc.collect()
    print("%-44s left %8.2f MB   (collector then freed %d objects)" % (name, left / 1e6, n))
def mass(idx, strategy, **kw):
    def f():
        c, b2d, cfg = fresh(idx, **kw)
        P.assemble_mass(b2d, cfg, c["coeff"], strategy=strategy)
    return f
def rhs(idx, **kw):
    def f():
        c, b2d, cfg = fresh(idx, **kw)
        P.assemble_rhs(P.ProjectionProblem(c["target"], b2d, cfg))
    return f
def l2(idx, **kw):
    def f():
        c, b2d, cfg = fresh(idx, **kw)
        K = cfg.active_functions().shape[0]
        P.l2_error(np.ones(K), P.ProjectionProblem(c["target"], b2d, cfg))
    return f
def proj(idx, **kw):
    def f():
        c, b2d, cfg = fresh(idx, **kw)
        P.project(P.ProjectionProblem(c["target"], b2d, cfg, strategy=c["strategy"]) if "strategy" in P.ProjectionProblem.__init__.__code__.co_varnames else P.ProjectionProblem(c["target"], b2d, cfg))
    return f
for strat in ("reference", "wq", "hybrid", "dwq"):
    run("assemble_mass config2 %s" % strat, mass(2, strat))
run("assemble_mass config1 wq (untrimmed)", mass(1, "wq"))
run("assemble_mass config4 p=6 nel=64 dwq c=detJ", mass(4, "dwq", nel=64))
run("assemble_mass config5 nel=512 dwq", mass(5, "dwq", nel=512))
run("assemble_rhs config2", rhs(2)); run("assemble_rhs config5 nel=512", rhs(5, nel=512))
run("l2_error config2", l2(2)); run("l2_error config5 nel=512", l2(5, nel=512))
try:
    run("project config2", proj(2))
except Exception as e:
    print("project probe failed:", repr(e)[:200])
