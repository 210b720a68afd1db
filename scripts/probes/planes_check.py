"""Planes path (tq_sf_strips + tq_planes_csr) against the row-major path on
the same formation: pattern identical, values within 1e-13 (dev aid)."""
import sys, time; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2101_08053_b200 import cases as C, assembly as A, _rawrows as R
import paper_2101_08053_b200 as P

def run(nel, p, strategy, detj=True):
    c4 = C.baseline_config(4, p=p, nel=nel)
    b2d, cfg = C.build_space(None, nel, p, curves=c4["curves"])
    coeff = c4["coeff"] if detj else None
    out = {}
    for pl in (False, True):
        R.PLANES = pl
        M = P.assemble_mass(b2d, cfg, coeff, strategy=strategy).data
        out[pl] = M
    a, b = out[False], out[True]
    same = np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
    d = np.max(np.abs(a.data - b.data)) / np.max(np.abs(a.data)) if same else float("nan")
    print(f"nel={nel} p={p} {strategy} detj={detj}: nnz {a.nnz} {b.nnz} pattern_same={same} maxrel={d:.3e}", flush=True)
    return same and d < 1e-13

ok = True
for args in [(48, 3, "dwq"), (64, 4, "dwq"), (64, 4, "hybrid"), (64, 4, "wq"), (32, 3, "reference", False),
             (32, 3, "reference"), (256, 6, "dwq"), (256, 8, "dwq")]:
    ok &= run(*args)
print("ALL_OK" if ok else "MISMATCH")
