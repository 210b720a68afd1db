"""Row census of config 5: deep / regular-tile / irregular rows (dev aid)."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2101_08053_b200 import cases as C
from paper_2101_08053_b200.assembly import form
c5 = C.baseline_config(5)
b2d, cfg = C.build_space(None, 2048, 4, curves=c5["curves"])
f, csr = form(b2d, cfg, None, "dwq")
K = f.K
act = f.active[:K].cpu().numpy()
deep = f.deep.cpu().numpy()[act] != 0
fast = f.rowfast[:K].cpu().numpy() != 0
n2 = b2d.shape[1]
nt = K // 32
reg = 0
for t in range(nt):
    a = act[32 * t: 32 * t + 32]
    if fast[32 * t: 32 * t + 32].all() and a[-1] - a[0] == 31 and a[0] // n2 == a[-1] // n2:
        reg += 1
print(f"rows {K} deep {deep.sum()} fast {fast.sum()} cut-rows {len(f.raw_list)} tiles {nt} regular {reg} ({reg/nt:.3f})")
