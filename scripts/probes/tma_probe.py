"""Drive tma_probe.so (dev aid): bandwidth of TMA bulk CSR writes."""
import ctypes as C, os, sys, torch
lib = C.CDLL(os.path.join(os.path.dirname(__file__), "tma_probe.so"))
nrows = 3_078_139
idx = torch.empty(nrows * 81 + 8_000_000, dtype=torch.int32, device="cuda")
dat = torch.empty(nrows * 81 + 8_000_000, dtype=torch.float64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
import sys
touches = (1,) if "quick" in sys.argv else (0, 1)
for touch in touches:
    for ch in ((8,) if "quick" in sys.argv else (2, 4, 8, 16)):
        for ns in ((2,) if "quick" in sys.argv else (2, 3, 4)):
            for wpb, bps in ((6, 2), (8, 1)) if "quick" in sys.argv else ((8, 1), (8, 2), (4, 4), (16, 1)):
              for un in ((0, 4, 16) if "quick" in sys.argv else (0, 1)):
                args = (nrows, ch, ns, wpb, bps, touch, C.c_void_p(idx.data_ptr()), C.c_void_p(dat.data_ptr()), un)
                if lib.probe(*args) != 0:
                    continue
                torch.cuda.synchronize(); best = 1e9
                for _ in range(5):
                    e0.record(); lib.probe(*args); e1.record(); torch.cuda.synchronize()
                    best = min(best, e0.elapsed_time(e1))
                print(f"touch {touch} ch {ch:2d} ns {ns} wpb {wpb:2d} bps {bps} unaligned {un}: {best:.3f} ms {nrows*81*12/best/1e6:5.0f} GB/s", flush=True)
