"""sha256 of the config-4 CSR (dev aid: bit-identity of kernel variants
selected by environment knobs).  python scripts/probes/c4_hash.py p nel"""
import hashlib, sys; sys.path.insert(0, ".")
import numpy as np
from paper_2101_08053_b200 import cases as C, assembly as A
p = int(sys.argv[1]); nel = int(sys.argv[2])
c4 = C.baseline_config(4, p=p, nel=nel)
b2d, cfg = C.build_space(None, nel, p, curves=c4["curves"])
for strat in ("dwq", "hybrid"):
    M = A.assemble_mass(b2d, cfg, c4["coeff"], strategy=strat).data
    h = hashlib.sha256()
    for a in (M.indptr, M.indices, M.data):
        h.update(np.ascontiguousarray(a).tobytes())
    print(strat, p, nel, M.nnz, h.hexdigest()[:16])
