"""Device vs host cut-cell decomposition at config 5 (dev aid)."""
import sys, time; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2101_08053_b200 import cases as C, _classify as K
c5 = C.baseline_config(5)
b2d, cfg = C.build_space(None, 2048, 4, curves=c5["curves"])
K.cut_cell_rule_device(cfg, 4); torch.cuda.synchronize()
t = time.perf_counter(); rd = K.cut_cell_rule_device(cfg, 4); torch.cuda.synchronize(); td = time.perf_counter() - t
t = time.perf_counter(); rh = K.cut_cell_rule(cfg, 4, host_only=True); th = time.perf_counter() - t
print(f"device {td*1e3:.1f} ms  host C++ {th*1e3:.1f} ms  points {rd.total_points()} / {rh.total_points()}")
assert np.array_equal(rd.ptr, rh.ptr) and np.array_equal(rd.elements, rh.elements)
print("max |dP|", np.abs(rd.points - rh.points).max(), "max rel |dW|", (np.abs(rd.weights - rh.weights) / np.abs(rh.weights)).max(),
      "bit-identical P", np.array_equal(rd.points, rh.points), "W", np.array_equal(rd.weights, rh.weights))
