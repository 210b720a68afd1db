"""Write bandwidth of incompressible vs constant data (dev aid)."""
import torch
n = 2 * 2**30 // 8
src_c = torch.full((n,), 1.0, dtype=torch.float64, device="cuda")
src_r = torch.rand(n, dtype=torch.float64, device="cuda")
dst = torch.empty(n, dtype=torch.float64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
def t(fn, nbytes, name):
    for _ in range(3): fn()
    torch.cuda.synchronize(); best = 1e9
    for _ in range(10):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    print(f"{name}: {nbytes/best/1e6:.0f} GB/s")
t(lambda: dst.copy_(src_c), 16 * n, "copy constant")
t(lambda: dst.copy_(src_r), 16 * n, "copy random")
t(lambda: dst.fill_(0.37), 8 * n, "fill constant")
t(lambda: torch.mul(src_r, 1.0000001, out=dst), 16 * n, "scale random (read+write)")
