"""Strip launch classes of config 4 (rows per strip, strips, rule-row
capacities, union width, shared bytes, blocks per SM) -- dev aid."""
import sys; sys.path.insert(0, ".")
import numpy as np
from paper_2101_08053_b200 import cases as C, assembly as A, _rawrows as R
p = int(sys.argv[1]) if len(sys.argv) > 1 else 8
c4 = C.baseline_config(4, p=p, nel=256)
b2d, cfg = C.build_space(None, 256, p, curves=c4["curves"])
f, _ = A.form(b2d, cfg, c4["coeff"], "dwq")
pg = R.planes_geo(f)
cl = R.strip_classes(f, pg, f._setup.sets[0][0].layout, f._setup.sets[1][0].layout)
WP = 3 * ((2 * p + 3) // 3)
for ts, sd, ns, n1m, n2m, nu, b2cap in cl:
    gs = (n1m * WP + 1) & ~1
    glen = (nu + 3) & ~1
    b2 = gs + n1m * glen
    m = (n2m * WP + 1) // 2
    sb = 2 * (m | 1)
    buf = b2 + ts * sb
    tot = 2 * buf + nu * (WP | 1)
    print(f"ts={ts} strips={ns} n1m={n1m} n2m={n2m} nu={nu}  smem={8 * tot / 1024:.1f} KB  (B2 stage {8 * ts * sb / 1024:.1f} KB/buffer)")
print("nmax std", f._setup.nmax_std)
