import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2101_08053_b200 import cases as C, _lib as L, _rawrows as R
R._bind()
c4 = C.baseline_config(4, p=3, nel=48)
geo = c4["coeff"]._device
X = torch.tensor([0.0014465, 0.0068752, 0.3, 0.77], dtype=torch.float64, device="cuda")
sp = torch.empty(4, dtype=torch.int32, device="cuda")
nd = torch.zeros(4 * 8, dtype=torch.float64, device="cuda")
L.call("tq_geo_lines", geo.device(), L.ptr(X), 4, L.ptr(sp), L.ptr(nd), L.stream())
torch.cuda.synchronize()
print("knots", geo.knots, "p", geo.p, "n", geo.n)
print(sp.cpu().numpy()); print(nd.cpu().numpy().reshape(4, 8))
