"""Probe: untrimmed formation timing on the GPU (development aid)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2101_08053_b200 as P

nel = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
p = int(sys.argv[2]) if len(sys.argv) > 2 else 4
b = P.make_uniform_basis(nel, p)
b2d = P.TensorBasis2D(b, P.make_uniform_basis(nel, p))
t0 = time.perf_counter(); cfg = P.classify_elements(b2d, []); torch.cuda.synchronize()
print("classify", time.perf_counter() - t0)
from paper_2101_08053_b200.assembly import form
for it in range(3):
    f, csr = form(b2d, cfg, None, "wq")
    r = f.report
    print(f"it{it} nnz={csr.nnz} weights={r.t_weights*1e3:.2f}ms interior={r.t_interior*1e3:.2f}ms finish={r.t_finish*1e3:.2f}ms total={r.t_total*1e3:.2f}ms")
# kernel-only timing of count/scan/fill
ctx = f.rowctx()
from paper_2101_08053_b200 import _lib as L
counts = torch.empty(f.K, dtype=torch.int32, device="cuda")
e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
print("deep rows", int(f.deep.sum().item()) if f.deep is not None else None)
for rep in range(3):
    e[0].record(); L.call("tq_row_counts", ctx, L.ptr(counts), L.stream()); e[1].record()
    L.call("tq_fill_rows", ctx, L.ptr(csr.indptr), L.ptr(csr.indices), L.ptr(csr.data), L.stream()); e[2].record()
    torch.cuda.synchronize()
    tc, tf = e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])
    print(f"counts {tc:.3f} ms  fill {tf:.3f} ms  fill GB/s {(12*csr.nnz + 4*f.K)/tf/1e6:.1f}")
