"""Diagnose config-5 value differences: product (device cut cells) vs the
reference's cut-cell points injected, vs the golden's sampled rows."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, scipy.sparse as sp
import paper_2101_08053_b200 as P
from tests import golden_cases as G
from tests.test_gpu_headline import headline_space, inject_golden_cut_rule

tag = sys.argv[1] if len(sys.argv) > 1 else "config5"
s = sys.argv[2] if len(sys.argv) > 2 else "dwq"
d = G.load(tag)
b2d, cfg = headline_space(tag)
M = P.assemble_mass(b2d, cfg, None, strategy=s).data
saved = dict(cfg._cut_rules)
inject_golden_cut_rule(cfg, d)
M2 = P.assemble_mass(b2d, cfg, None, strategy=s).data
fro = float(d[f"{s}_fro"])
D = M.data - M2.data
print("fro golden", fro, "fro M", sp.linalg.norm(M), "fro M2", sp.linalg.norm(M2))
print("rel |fro(M)-fro| ", abs(sp.linalg.norm(M) - fro) / fro, " rel |fro(M2)-fro|", abs(sp.linalg.norm(M2) - fro) / fro)
print("||M-M2||/fro", np.linalg.norm(D) / fro)
k = np.argsort(-np.abs(D))[:10]
rows = np.searchsorted(M.indptr, k, side="right") - 1
act = cfg.active_functions()
fc = cfg.func_class
for kk, r in zip(k, rows):
    c = M.indices[kk]
    print(f"  row {r} {tuple(act[r])} fc {fc[tuple(act[r])]} col {c} {tuple(act[c])} M {M.data[kk]:.6e} M2 {M2.data[kk]:.6e} d {D[kk]:.3e}")
# sampled rows of M2 vs golden
rws = d[f"{s}_rows"]
got = np.concatenate([M2.data[M2.indptr[r]:M2.indptr[r + 1]] for r in rws])
ref = d[f"{s}_rowsdata"]
print("sampled rows M2 max rel", np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
got = np.concatenate([M.data[M.indptr[r]:M.indptr[r + 1]] for r in rws])
print("sampled rows M  max rel", np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
# sum of squares split: rows of cut functions vs others
isc = (fc[act[:, 0], act[:, 1]] == 1)
rr = np.repeat(np.arange(M.shape[0]), np.diff(M.indptr))
print("||D|| on cut-function rows", np.linalg.norm(D[isc[rr]]) / fro, "others", np.linalg.norm(D[~isc[rr]]) / fro)
