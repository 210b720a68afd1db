"""Config-5 RHS and L2-error timing (device events around the native calls
on resident inputs; dev aid for the bench's secondary line)."""
import sys, time; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import cases as C, projection as PR
nel = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
c5 = C.baseline_config(5, nel=nel)
b2d, cfg = C.build_space(None, nel, 4, curves=c5["curves"])
cfg.cut_cell_rule(4)
prob = P.ProjectionProblem(C.f_config5, b2d, cfg, strategy="dwq")
K = cfg.active_index()[0]["K"]
x = torch.randn(K, dtype=torch.float64, device="cuda")
for _ in range(2):
    b = PR.assemble_rhs_device(prob); nd = PR.l2_error_parts_device(x, prob)
torch.cuda.synchronize()
ts, tl = [], []
for _ in range(10):
    t0 = time.perf_counter(); b = PR.assemble_rhs_device(prob); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    t0 = time.perf_counter(); nd = PR.l2_error_parts_device(x, prob); torch.cuda.synchronize(); tl.append(time.perf_counter() - t0)
print(f"rhs call {1e3*np.median(ts):.3f} ms, l2 call {1e3*np.median(tl):.3f} ms (wall, median of 10)")
