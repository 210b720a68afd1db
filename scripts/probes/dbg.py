import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2101_08053_b200 import cases as C, assembly as A, _rawrows as R, _lib as L
c4 = C.baseline_config(4, p=3, nel=48)
b2d, cfg = C.build_space(None, 48, 3, curves=c4["curves"])
f, csr = A.form(b2d, cfg, c4["coeff"], "dwq")
eg, em = f._setup.eg, f._setup.em
E1, _ = R._gauss_pairs(f, eg, em)
# inline path: call with null line tables
ge = R.gauss_elements(f)
ctx = R._gauss_ctx(f, eg, em, None, R._desc_dev(f)[0], torch.empty(1, dtype=torch.float64, device=f.dev), 0)
geo = c4["coeff"]._device
E2 = torch.empty_like(E1)
L.call("tq_gauss_pairs", ctx, geo.device(), L.ptr(eg[0][3]), L.ptr(eg[1][3]), L.ptr(ge["gel"]), ge["n"], 0,
       L.ptr(E2), 0, 0, 0, 0, L.stream())
torch.cuda.synchronize()
d = (E1 - E2).abs().max().item()
print("n", ge["n"], "maxdiff", d, "max", E2.abs().max().item())
i = int((E1 - E2).abs().argmax().item()); print(i, E1[i].item(), E2[i].item(), i // 100)
