"""Where do slow dev_many calls spend their time? (instrumented copy)"""
import sys, time; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import _lib as L, cases as C, trimming as T, splines as S, quadrature as Q
log = []
def dev_many(items):
    t = [time.perf_counter()]
    arrs = [np.ascontiguousarray(x, dtype=L._NP_DTYPE.get(dt)) for x, dt in items]
    offs, total = [], 0
    for a in arrs:
        offs.append(total); total += (a.nbytes + 255) & ~255
    d = L.device(); ring = L._RINGS.get(d.index)
    if ring is None:
        ring = L._RINGS[d.index] = L._StagingRing()
    t.append(time.perf_counter())
    head0 = ring.head
    lo = ring.reserve(total)
    t.append(time.perf_counter())
    if lo is None:
        log.append(("fallback", total)); return [L.dev(a, dt) for a, (_, dt) in zip(arrs, items)]
    for a, o in zip(arrs, offs):
        if a.nbytes:
            ring.host[lo + o: lo + o + a.nbytes] = a.reshape(-1).view(np.uint8)
    t.append(time.perf_counter())
    block = torch.empty(total, dtype=torch.uint8, device=d)
    t.append(time.perf_counter())
    block.copy_(ring.buf[lo: lo + total], non_blocking=True)
    t.append(time.perf_counter())
    ring.done(None)
    t.append(time.perf_counter())
    out = [block[o: o + a.nbytes].view(dt).view(a.shape) if a.size else torch.empty(a.shape, dtype=dt, device=d)
           for a, o, (_, dt) in zip(arrs, offs, items)]
    t.append(time.perf_counter())
    log.append((total, head0, lo, [round(1e6 * (b - a)) for a, b in zip(t, t[1:])]))
    return out
L.dev_many = dev_many
c5 = C.baseline_config(5)
knots = P.make_uniform_knots(2048, 4).knots.copy(); ctrl = c5["curves"][0].ctrl.copy()
def call():
    bb = P.TensorBasis2D(P.Basis1D(P.KnotVector(knots.copy(), 4)), P.Basis1D(P.KnotVector(knots.copy(), 4)))
    cf = P.classify_elements(bb, [T.PeriodicBSplineTrim(ctrl.copy())])
    t2 = time.perf_counter()
    M = P.assemble_mass(bb, cf, None, strategy="dwq")
    return time.perf_counter() - t2
for i in range(10):
    log.clear()
    dt = call()
    tot = sum(sum(e[3]) for e in log if e[0] != "fallback")
    print("call %d: %.1f ms, dev_many total %.2f ms, n=%d" % (i, dt * 1e3, tot / 1e3, len(log)))
    for e in log:
        if e[0] == "fallback" or sum(e[3]) > 500:
            print("   slow:", e)
