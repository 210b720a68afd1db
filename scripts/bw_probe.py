"""Write-bandwidth ceiling probe: torch fill_ / copy_ on ~3 GB (dev aid)."""
import torch
n = 3 * 2**30 // 8
a = torch.empty(n, dtype=torch.float64, device="cuda")
b = torch.empty(n, dtype=torch.float64, device="cuda")
i32 = torch.empty(n, dtype=torch.int32, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn, bytes_ in (("fill f64", lambda: a.fill_(1.0), 8 * n), ("copy f64", lambda: b.copy_(a), 16 * n),
                         ("fill i32", lambda: i32.fill_(3), 4 * n)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name}: {bytes_ / best / 1e6:.0f} GB/s ({best:.3f} ms)")
