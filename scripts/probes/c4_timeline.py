"""Device-timer stamps inside one replayed config-4 graph (critical path of
the c != 1 pass) -- dev aid.  python scripts/probes/c4_timeline.py [p] [nel]"""
import sys; sys.path.insert(0, ".")
import torch
from paper_2101_08053_b200 import cases as C, _lib as L, assembly as A
p = int(sys.argv[1]) if len(sys.argv) > 1 else 8
nel = int(sys.argv[2]) if len(sys.argv) > 2 else 256
c4 = C.baseline_config(4, p=p, nel=nel)
b2d, cfg = C.build_space(None, nel, p, curves=c4["curves"])
gf = A.GraphFormation(b2d, cfg, c4["coeff"], "dwq")
del gf
A.STAMPS = L.Stamps()
gf = A.GraphFormation(b2d, cfg, c4["coeff"], "dwq")
names = A.STAMPS.names
k = len(names) - 1 - names[::-1].index("start")
for _ in range(5):
    gf.run()
torch.cuda.synchronize()
t = A.STAMPS.buf.cpu().numpy()
base = int(t[k])
for i in range(k, len(names)):
    print(f"{names[i]:18s} {(int(t[i]) - base) / 1e3:8.1f} us")
