"""Measured FP64 peaks on this B200 (dev aid): DFMA loop (vector pipe) and
cuBLAS DGEMM through torch.matmul (float64)."""
import ctypes as C, json, os, torch
lib = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "fp64_peak.so"))
out = torch.empty(148 * 64 * 1024, dtype=torch.float64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 0.0
for blocks_per_sm in (4, 8):
    for threads in (256, 512):
        blocks, iters = 148 * blocks_per_sm, 4096
        lib.dfma(C.c_void_p(out.data_ptr()), blocks, threads, iters); torch.cuda.synchronize()
        e0.record(); lib.dfma(C.c_void_p(out.data_ptr()), blocks, threads, iters); e1.record(); torch.cuda.synchronize()
        fl = 2.0 * 8 * iters * blocks * threads
        best = max(best, fl / (e0.elapsed_time(e1) * 1e-3) / 1e12)
gemm = 0.0
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    torch.matmul(a, b); torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        torch.matmul(a, b)
    e1.record(); torch.cuda.synchronize()
    gemm = max(gemm, 5 * 2.0 * n ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
print(json.dumps({"dfma_tflops": best, "dgemm_tflops": gemm}))
