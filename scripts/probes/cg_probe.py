"""One device CG solve at 512^2 (ncu target; dev aid)."""
import sys; sys.path.insert(0, ".")
import torch
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import cases as C
b2d, cfg = C.build_space(None, 512, 4, curves=[C.closed_circle()])
prob = P.ProjectionProblem(P.projection.default_target, b2d, cfg, strategy="dwq")
M = P.assemble_mass(b2d, cfg, strategy="dwq")
b = P.assemble_rhs(prob)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
P.solve_spd(M, b)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
