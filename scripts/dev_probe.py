"""Micro-timing of the small-upload helpers (dev x7 vs dev_many of 7)."""
import sys, time; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2101_08053_b200 import _lib as L
L.device()
arrs = [(np.random.rand(2060), torch.float64), (np.random.rand(2049), torch.float64)] + \
       [(np.arange(2052, dtype=np.int64), torch.int32) for _ in range(5)]
def t(fn, n=200):
    for _ in range(20): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): fn()
    dt = (time.perf_counter() - t0) / n * 1e6; torch.cuda.synchronize(); return dt
print("dev x7      %.1f us" % t(lambda: [L.dev(a, d) for a, d in arrs]))
print("dev_many(7) %.1f us" % t(lambda: L.dev_many(arrs)))
print("ascontig x7 %.1f us" % t(lambda: [np.ascontiguousarray(a, dtype=L._NP_DTYPE[d]) for a, d in arrs]))
ring = L._RINGS[torch.cuda.current_device()]
print("reserve     %.1f us" % t(lambda: ring.reserve(100000)))
print("empty       %.1f us" % t(lambda: torch.empty(100000, dtype=torch.uint8, device="cuda")))
blk = torch.empty(100000, dtype=torch.uint8, device="cuda")
print("copy_       %.1f us" % t(lambda: blk.copy_(ring.buf[:100000], non_blocking=True)))
print("event       %.1f us" % t(lambda: ring.done(None)))
print("capturing   %.1f us" % t(lambda: torch.cuda.is_current_stream_capturing()))
print("device()    %.1f us" % t(lambda: L.device()))
