"""e2e step spikes: per-step phase clocks of the bench's public-API loop,
gc activity and host-allocator stats (dev aid)."""
import gc, sys, time, json; sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import cases as C, assembly as A
c5 = C.baseline_config(5)
knots = np.ascontiguousarray(P.make_uniform_knots(2048, 4).knots)
ctrl = np.ascontiguousarray(c5["curves"][0].ctrl)
tohost = [0.0]
orig = A.DeviceCSR.to_host
def wrapped(self):
    t = time.perf_counter(); r = orig(self); tohost[0] += time.perf_counter() - t; return r
A.DeviceCSR.to_host = wrapped
gcev = []
gc.callbacks.append(lambda ph, info: gcev.append((ph, info.get("generation"), time.perf_counter())))
mode = sys.argv[1] if len(sys.argv) > 1 else "plain"
if mode == "nogc":
    gc.disable()
for k in range(12):
    torch.cuda.synchronize()
    tohost[0] = 0.0; gcev.clear()
    t0 = time.perf_counter()
    bb = P.TensorBasis2D(P.Basis1D(P.KnotVector(knots.copy(), 4)), P.Basis1D(P.KnotVector(knots.copy(), 4)))
    cf = P.classify_elements(bb, [P.trimming.PeriodicBSplineTrim(ctrl.copy())])
    t1 = time.perf_counter()
    M = P.assemble_mass(bb, cf, None, strategy="dwq")
    t2 = time.perf_counter()
    del M
    if mode == "collect":
        gc.collect()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    try:
        hs = torch.cuda.host_memory_stats()
        hst = {k2: hs[k2] for k2 in hs if ("allocated_bytes.current" in k2 or "reserved_bytes.current" in k2 or k2 in ("num_host_alloc", "num_host_free", "host_alloc_time.total", "host_free_time.total"))}
    except Exception as e:
        hst = str(e)
    gens = [g for ph, g, _ in gcev if ph == "start"]
    print(json.dumps({"k": k, "total": round(t3 - t0, 4), "classify": round(t1 - t0, 4), "assemble": round(t2 - t1, 4),
                      "to_host": round(tohost[0], 4), "release": round(t3 - t2, 4), "gc": gens,
                      "dev_reserved_GB": round(torch.cuda.memory_reserved() / 1e9, 2), "host": hst}), flush=True)
