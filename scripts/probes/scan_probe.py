"""Time tq_scan_indptr alone on 3.08M row counts (dev aid)."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2101_08053_b200 import _lib as L
n = 3_078_139
counts = torch.from_numpy(np.random.default_rng(0).integers(0, 100, n).astype(np.int32)).cuda()
out = torch.empty(n + 1, dtype=torch.int32, device="cuda")
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
g = torch.cuda.CUDAGraph()
for _ in range(3):
    L.call("tq_scan_indptr", L.ptr(counts), n, L.ptr(out), None, L.stream())
torch.cuda.synchronize()
s = torch.cuda.Stream()
ws = torch.empty(L.lib().tq_scan_workspace_bytes(n), dtype=torch.uint8, device="cuda")
REP = 10    # scans per graph: the graph launch latency is amortised
with torch.cuda.graph(g, stream=s):
    for _ in range(REP):
        if "ws" in sys.argv:
            L.call("tq_scan_indptr_ws", L.ptr(counts), n, L.ptr(out), L.ptr(ws), None, L.stream())
        else:
            L.call("tq_scan_indptr", L.ptr(counts), n, L.ptr(out), None, L.stream())
for fl in (False, True):
    ts = []
    for _ in range(20):
        if fl:
            flush.fill_(1)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / REP)
    print(f"per scan (L2 warm after the first), flush={fl}: median {np.median(ts):.1f} us  min {min(ts):.1f} us")
ref = np.concatenate([[0], np.cumsum(counts.cpu().numpy())])
assert np.array_equal(out.cpu().numpy(), ref)
