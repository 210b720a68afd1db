"""Product (GPU) weight rows vs the reference's (oracle, bit-exact with
LAPACK) for one golden case: which rule sets / rows differ and by how much."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from tests import golden_cases as G
from tests.test_gpu_trimmed import product_case
from tests.test_oracle_golden import oracle_case
from oracle import assemble as OA
from paper_2101_08053_b200 import _rawrows
from paper_2101_08053_b200.assembly import Formation

tag = sys.argv[1] if len(sys.argv) > 1 else "bspline_detj_24_2"
desc = G.describe(tag)
b2d, cfg, coeff = product_case(desc)
f = Formation(b2d, cfg, coeff, "dwq")
r1, r2, dwq = _rawrows.build_all_rules(f)
ocfg, ocoeff, _ = oracle_case(desc)
run = OA._Run(ocfg, ocoeff or OA.Coeff())
o1, o2, odwq = OA.build_rules(run, True)


def cmp(name, pr, orr):
    k0, wptr, w = orr.packed()
    pts_same = np.array_equal(pr.layout.points, orr.layout.points)
    bad = []
    for i in range(len(orr.rows)):
        if orr.rows[i] is None:
            continue
        kk, ww = pr.row(i)
        ref = orr.rows[i][1]
        err = np.max(np.abs(ww - ref)) / max(np.max(np.abs(ref)), 1e-300) if ww.size == ref.size else np.inf
        if kk != orr.rows[i][0] or err > 1e-12:
            bad.append((i, err))
    print(f"{name}: layout same {pts_same}, rows {sum(r is not None for r in orr.rows)}, differing {len(bad)}: "
          + ", ".join(f"{i}:{e:.1e}" for i, e in sorted(bad, key=lambda x: -x[1])[:8]))


cmp("r1", r1, o1)
cmp("r2", r2, o2)
for key in sorted(odwq):
    cmp(f"dwq{key}", dwq[key], odwq[key])
