"""Which objects of a fresh-configuration call are only freed by the cyclic
collector?  (They keep device tensors alive past the call; dev aid.)"""
import collections, gc, sys; sys.path.insert(0, ".")
import torch
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import cases as C, trimming as T
c5 = C.baseline_config(5)
knots = P.make_uniform_knots(2048, 4).knots.copy(); ctrl = c5["curves"][0].ctrl.copy()
def call():
    bb = P.TensorBasis2D(P.Basis1D(P.KnotVector(knots.copy(), 4)), P.Basis1D(P.KnotVector(knots.copy(), 4)))
    cf = P.classify_elements(bb, [T.PeriodicBSplineTrim(ctrl.copy())])
    M = P.assemble_mass(bb, cf, None, strategy="dwq")
    return M.shape
for _ in range(2): call()
gc.collect(); torch.cuda.synchronize()
base = torch.cuda.memory_allocated()
gc.disable()
call(); torch.cuda.synchronize()
print("device bytes still allocated after the call (before gc): %.1f MB" % ((torch.cuda.memory_allocated() - base) / 1e6))
gc.set_debug(gc.DEBUG_SAVEALL)
n = gc.collect()
print("collected", n, "garbage", len(gc.garbage))
cnt = collections.Counter(type(o).__module__ + "." + type(o).__name__ for o in gc.garbage)
for k, v in cnt.most_common(40): print("%6d %s" % (v, k))
tb = sum(o.numel() * o.element_size() for o in gc.garbage if isinstance(o, torch.Tensor) and o.is_cuda)
print("cuda tensor bytes in garbage: %.1f MB" % (tb / 1e6))
for o in gc.garbage:
    m = type(o).__module__
    if m.startswith("paper_2101"):
        refs = [type(r).__name__ for r in gc.get_referrers(o) if r is not gc.garbage][:6]
        print("  ", type(o).__name__, "<-", refs)
