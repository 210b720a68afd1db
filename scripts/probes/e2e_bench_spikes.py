"""The bench's own e2e loop with per-call clocks on form / to_host and the
device allocator's counters (dev aid: where do the e2e step spikes come from)."""
import sys, time, json; sys.path.insert(0, ".")
import torch
import bench
from paper_2101_08053_b200 import assembly as A
log = []
def wrap(obj, name):
    fn = getattr(obj, name)
    def w(*a, **k):
        if torch.cuda.is_current_stream_capturing() or k.get("capture") is not None:
            return fn(*a, **k)
        torch.cuda.synchronize(); t = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        ms = torch.cuda.memory_stats()
        log.append((name, round(time.perf_counter() - t, 4), ms.get("num_alloc_retries"), ms.get("segment.all.allocated"),
                    round(torch.cuda.memory_reserved() / 1e9, 2)))
        print(json.dumps(log[-1]), file=sys.stderr, flush=True)
        return r
    setattr(obj, name, w)
wrap(A.DeviceCSR, "to_host")
wrap(A, "form")
sys.argv = ["bench.py", "--no-cpu", "--no-config4", "--e2e-steps", "12", "--steps", "20"]
bench.main()
