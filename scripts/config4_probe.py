"""Config 4 (B-spline trim, c = det J of the perturbed geometry map, DWQ,
256^2, p = 6 / 8): one formation pass captured as a CUDA graph and
replayed (L2 flushed), plus the algorithmic roofline of SURVEY §8(d):
B_alg = 12 nnz + 4 (rows+1) + 8 N1 N2 (coefficient grid), F_alg = 2 sum over
interior rows of sum_factor_op_count -- dev aid / evidence for the c != 1
path.  Usage: python scripts/config4_probe.py [p] [nel] [prof]"""
import json, sys, time; sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2101_08053_b200 import cases as C, assembly as A
p = int(sys.argv[1]) if len(sys.argv) > 1 else 6
nel = int(sys.argv[2]) if len(sys.argv) > 2 else 256
c4 = C.baseline_config(4, p=p, nel=nel)
b2d, cfg = C.build_space(None, nel, p, curves=c4["curves"])
coeff = c4["coeff"]
gf = A.GraphFormation(b2d, cfg, coeff, "dwq")
K = cfg.active_index()[0]["K"]
flush = torch.empty(256 * 2**20 // 8, dtype=torch.float64, device="cuda")
for _ in range(3):
    gf.run()
torch.cuda.synchronize()
if "prof" in sys.argv:
    torch.cuda.cudart().cudaProfilerStart()
    A.form(b2d, cfg, coeff, "dwq", capture={"nnz": gf.nnz})
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    sys.exit(0)
ts = []
for _ in range(20):
    flush.fill_(1.0)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); gf.run(); e.record(); torch.cuda.synchronize()
    gf.check()
    ts.append(s.elapsed_time(e))
ms = float(np.median(ts))
# algorithmic figures
f = gf.f
r1, r2 = f.rules[0], f.rules[1]
act = cfg.active_functions()
fc = cfg.func_class
n1g, n2g = r1.layout.num_points, r2.layout.num_points
interior = act[fc[act[:, 0], act[:, 1]] == 0]
ops = 0
for i1, i2 in interior:
    ops += A.sum_factor_op_count(int(i1), int(i2), r1, r2)
F = 2.0 * ops
B = 12.0 * gf.nnz + 4.0 * (K + 1) + 8.0 * n1g * n2g
peaks = json.load(open("MEASURED_PEAKS.json"))
fp64 = json.load(open("profiles/fp64_peaks.json"))
bw = float(peaks.get("hbm_gbs", 6537.6)) * 1e9
pf = max(float(v) for k, v in fp64.items() if isinstance(v, (int, float)) and "tflop" in k.lower()) * 1e12
T = max(B / bw, F / pf)
print(json.dumps({"config": f"config4 p={p} nel={nel} dwq c=detJ", "rows": K, "nnz": gf.nnz,
                  "step_ms": ms, "nnz_per_s": gf.nnz / (ms / 1e3), "B_alg": B, "F_alg": F,
                  "T_hbm_us": 1e6 * B / bw, "T_fp64_us": 1e6 * F / pf, "T_star_us": 1e6 * T,
                  "step_frac_of_roofline": T / (ms / 1e3), "interior_rows": int(interior.shape[0])}))
