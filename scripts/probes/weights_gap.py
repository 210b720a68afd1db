"""c != 1 parity with the GPU's OWN weights (no rules= import): rel-Frobenius
gap to the reference goldens, and how many WQ/DWQ weight rows equal the
reference's (LAPACK dgeqp3) rows -- development probe."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, scipy.sparse as sp
import paper_2101_08053_b200 as P
from tests import golden_cases as G
from tests.test_gpu_trimmed import product_case, golden_rows

for tag in ("bspline_detj_24_2", "bspline_detj_32_3", "config4_p6", "config4_p8"):
    d = G.load(tag); desc = G.describe(tag)
    b2d, cfg, coeff = product_case(desc)
    for s in G.strategies_in(d):
        if s == "reference":
            continue
        M = P.assemble_mass(b2d, cfg, coeff, strategy=s).data
        if f"{s}_data" in d:
            R = sp.csr_matrix((d[f"{s}_data"], d[f"{s}_indices"], d[f"{s}_indptr"]), shape=M.shape)
            rel = np.linalg.norm(M.data - R.data) / np.linalg.norm(R.data)
            print(f"{tag:20s} {s:6s} rel-Frobenius {rel:.3e}", flush=True)
        else:
            got, ref = golden_rows(M, d, s)
            fro = float(d[f"{s}_fro"])
            print(f"{tag:20s} {s:6s} |dfro|/fro {abs(sp.linalg.norm(M) - fro) / fro:.3e} sampled max rel "
                  f"{np.max(np.abs(got - ref)) / np.max(np.abs(ref)):.3e}", flush=True)

R1 = G.load("rules_1d")
tot = same = 0
for key in [k[:-3] for k in R1 if k.endswith("_k0") and k.startswith(("wq_", "dwq_")) and "nonuni" not in k]:
    kind, nel, p = key.split("_")
    nel, p = int(nel), int(p)
    b = P.make_uniform_basis(nel, p)
    if kind == "wq":
        r = P.compute_wq_rules(b)
    else:
        r = P.build_dwq(b, P.place_wq_points(b), float(R1[f"{key}_u"]))
    k0, ptr, w = R1[f"{key}_k0"], R1[f"{key}_ptr"], R1[f"{key}_w"]
    n_same = 0
    for i in range(b.n):
        if k0[i] < 0:
            continue
        kk, ww = r.row(i)
        ref = w[ptr[i]:ptr[i + 1]]
        ok = kk == k0[i] and ww.size == ref.size and np.max(np.abs(ww - ref)) <= 1e-12 * np.max(np.abs(ref))
        n_same += ok
        tot += 1
    same += n_same
    print(f"{key:10s} rows equal to LAPACK's: {n_same}/{int((k0 >= 0).sum())}", flush=True)
print(f"total {same}/{tot}")
