"""Profile one config-5 formation step (host side) -- development aid."""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import torch
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import cases as C
from paper_2101_08053_b200.assembly import form
nel = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
c5 = C.baseline_config(5, nel=nel)
b2d, cfg = C.build_space(None, nel, 4, curves=c5["curves"])
cfg.cut_cell_rule(4)
for _ in range(3):
    f, csr = form(b2d, cfg, None, "dwq")
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
f, csr = form(b2d, cfg, None, "dwq")
torch.cuda.synchronize()
pr.disable()
r = f.report
print(f"weights {r.t_weights*1e3:.1f} interior {r.t_interior*1e3:.1f} cut {r.t_cut_regular*1e3:.1f} cutel {r.t_cut_elements*1e3:.1f} finish {r.t_finish*1e3:.1f}")
pstats.Stats(pr).sort_stats("cumtime").print_stats(35)
