"""sha256 of the config-5-recipe CSR at a reduced mesh (dev aid: bit-identity
of kernel variants selected by environment knobs).  python c5_hash.py nel"""
import hashlib, sys; sys.path.insert(0, ".")
import numpy as np
from paper_2101_08053_b200 import cases as C, assembly as A
nel = int(sys.argv[1])
c5 = C.baseline_config(5, nel=nel)
b2d, cfg = C.build_space(None, nel, 4, curves=c5["curves"])
for strat in ("dwq", "hybrid", "wq"):
    M = A.assemble_mass(b2d, cfg, None, strategy=strat).data
    h = hashlib.sha256()
    for a in (M.indptr, M.indices, M.data):
        h.update(np.ascontiguousarray(a).tobytes())
    print(strat, nel, M.nnz, h.hexdigest()[:16])
