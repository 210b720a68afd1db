"""Projection solve timings: device CG vs the reference's scipy path (dev aid)."""
import sys, time; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import cases as C
from oracle import project as OP
for nel, curves, scipy_too in ((128, [C.closed_circle()], True), (512, [C.closed_circle()], True),
                               (2048, C.baseline_config(5)["curves"], False)):
    b2d, cfg = C.build_space(None, nel, 4, curves=curves)
    prob = P.ProjectionProblem(P.projection.default_target, b2d, cfg, strategy="dwq")
    M = P.assemble_mass(b2d, cfg, strategy="dwq")
    b = P.assemble_rhs(prob)
    P.solve_spd(M, b)                      # warm
    torch.cuda.synchronize(); t = time.perf_counter()
    st = {}
    x = P.solve_spd(M, b, stats=st)
    tg = time.perf_counter() - t
    line = f"nel {nel}: n {M.shape[0]} nnz {M.data.nnz}  device CG {tg*1e3:.1f} ms iters {st['cg_iterations']} resid {st['residual']:.1e}"
    if scipy_too:
        t = time.perf_counter(); xr = OP.solve_spd(M.data, b); ts = time.perf_counter() - t
        line += f"  scipy {ts*1e3:.0f} ms  err diff {abs(P.l2_error(x, prob, M.active) - P.l2_error(xr, prob, M.active)):.1e}"
    print(line, flush=True)
