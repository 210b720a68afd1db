"""Kernel-node priority census of the captured config-5 / config-4 graphs
(dev aid: do the capture streams' priorities reach the graph nodes?)."""
import sys; sys.path.insert(0, ".")
from paper_2101_08053_b200 import cases as C, assembly as A
c5 = C.baseline_config(5, nel=512)
b2d, cfg = C.build_space(None, 512, 4, curves=c5["curves"])
gf = A.GraphFormation(b2d, cfg, None, "dwq")
print("config5 512^2", gf.node_priorities())
c4 = C.baseline_config(4, p=6, nel=64)
b2d, cfg = C.build_space(None, 64, 6, curves=c4["curves"])
gf = A.GraphFormation(b2d, cfg, c4["coeff"], "dwq")
print("config4 p6 64^2", gf.node_priorities())
print("config4 node types", gf.node_types())
c5 = C.baseline_config(5, nel=2048)
b2d, cfg = C.build_space(None, 2048, 4, curves=c5["curves"])
gf = A.GraphFormation(b2d, cfg, None, "dwq")
print("config5 2048^2 node types", gf.node_types(), gf.node_priorities())
