"""Config-4 row census: cut rows by mode, Gauss elements, cut groups/points (dev aid)."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2101_08053_b200 import cases as C, assembly as A, _rawrows as R
for p in (6, 8):
    c4 = C.baseline_config(4, p=p, nel=256)
    b2d, cfg = C.build_space(None, 256, p, curves=c4["curves"])
    f, csr = A.form(b2d, cfg, c4["coeff"], "dwq")
    desc, nint = R._plan(f)
    cut = desc[nint:]
    modes = np.bincount(cut[:, 1], minlength=3)
    ng = R.gauss_element_count(f)
    cu = f._setup.cut
    gp = cu["grp_pts"].cpu().numpy()
    print(f"p={p} rows {f.K} interior {nint} cut {cut.shape[0]} modes(G,BOX,MASK) {modes.tolist()} "
          f"gauss_elements {ng} groups {cu['ngroups']} points {int(gp[-1])} pts/group {np.diff(gp).mean():.0f} "
          f"cut elements {cu['grp_ptr'].numel() - 1}")
