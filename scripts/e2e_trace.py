"""torch.profiler (CUPTI) trace of one fresh-configuration public-API call
on config 5 after warm-up: host API calls (syncs, mallocs, copies) and
device activity on one timeline -- dev aid for the e2e path.  Writes
gpurun_out/e2e_trace.json and prints the top runtime calls."""
import sys, time; sys.path.insert(0, ".")
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import cases as C, trimming as T
c5 = C.baseline_config(5)
knots = P.make_uniform_knots(2048, 4).knots.copy(); ctrl = c5["curves"][0].ctrl.copy()
def call():
    bb = P.TensorBasis2D(P.Basis1D(P.KnotVector(knots.copy(), 4)), P.Basis1D(P.KnotVector(knots.copy(), 4)))
    cf = P.classify_elements(bb, [T.PeriodicBSplineTrim(ctrl.copy())])
    M = P.assemble_mass(bb, cf, None, strategy="dwq")
    torch.cuda.synchronize()
    return M
for _ in range(3):
    M = call(); del M
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    M = call()
    print("call ms", 1e3 * (time.perf_counter() - t0))
prof.export_chrome_trace("gpurun_out/e2e_trace.json")
print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=30))
