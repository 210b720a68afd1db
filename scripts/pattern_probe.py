"""Store-pattern probe for the fill kernel (dev aid)."""
import sys; sys.path.insert(0, ".")
import torch
from paper_2101_08053_b200 import _lib as L
lib = L.lib()
lib.tq_debug_pattern.argtypes = [L.i32, L.i32, L.i32, L.vp, L.vp, L.vp]
nrows = 3_078_139
idx = torch.empty(nrows * 81, dtype=torch.int32, device="cuda")
dat = torch.empty(nrows * 81, dtype=torch.float64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rpw in (1, 2, 4, 16, 64):
    for bps in (2, 4, 8):
        for _ in range(2):
            lib.tq_debug_pattern(nrows, rpw, bps, L.ptr(idx), L.ptr(dat), L.stream())
        torch.cuda.synchronize(); best = 1e9
        for _ in range(5):
            e0.record(); lib.tq_debug_pattern(nrows, rpw, bps, L.ptr(idx), L.ptr(dat), L.stream()); e1.record()
            torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
        print(f"rows/warp {rpw:3d} blocks/SM {bps}: {best:.3f} ms  {nrows*81*12/best/1e6:.0f} GB/s")
