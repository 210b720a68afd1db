"""Catch slow device allocations in the public-API e2e loop (dev aid): every
torch.empty/zeros call above 2 ms is printed with its size, caller and the
allocator's cudaMalloc/cudaFree counters."""
import sys, time, traceback, json; sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2101_08053_b200 as P
from paper_2101_08053_b200 import cases as C
c5 = C.baseline_config(5)
knots = np.ascontiguousarray(P.make_uniform_knots(2048, 4).knots)
ctrl = np.ascontiguousarray(c5["curves"][0].ctrl)
for name in ("empty", "zeros", "full", "arange"):
    orig = getattr(torch, name)
    def mk(orig, name):
        def w(*a, **k):
            t = time.perf_counter()
            r = orig(*a, **k)
            dt = time.perf_counter() - t
            if dt > 2e-3:
                ms = torch.cuda.memory_stats()
                fr = traceback.extract_stack(limit=4)[-2]
                print(json.dumps({"fn": name, "ms": round(1e3 * dt, 2), "bytes": r.numel() * r.element_size(),
                                  "dev": str(r.device), "at": f"{fr.filename.split('/')[-1]}:{fr.lineno}",
                                  "mallocs": ms.get("num_device_alloc"), "frees": ms.get("num_device_free"),
                                  "reserved_GB": round(torch.cuda.memory_reserved() / 1e9, 2)}), flush=True)
            return r
        return w
    setattr(torch, name, mk(orig, name))
for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 15):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    bb = P.TensorBasis2D(P.Basis1D(P.KnotVector(knots.copy(), 4)), P.Basis1D(P.KnotVector(knots.copy(), 4)))
    cf = P.classify_elements(bb, [P.trimming.PeriodicBSplineTrim(ctrl.copy())])
    M = P.assemble_mass(bb, cf, None, strategy="dwq")
    del M
    torch.cuda.synchronize()
    ms = torch.cuda.memory_stats()
    print("step", k, round(time.perf_counter() - t0, 4), "mallocs", ms.get("num_device_alloc"), "frees", ms.get("num_device_free"), flush=True)
