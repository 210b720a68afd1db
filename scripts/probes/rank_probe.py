"""Per-rank step time of the row-sharded formation (one rank's row block on
one GPU; an estimate for N-GPU strong scaling, dev aid)."""
import sys; sys.path.insert(0, ".")
import torch
from paper_2101_08053_b200 import cases as C
from paper_2101_08053_b200.assembly import GraphFormation
c5 = C.baseline_config(5)
b2d, cfg = C.build_space(None, 2048, 4, curves=c5["curves"])
cfg.cut_cell_rule(4)
K = cfg.active_index()[0]["K"]
flush = torch.empty(256 * 2**20 // 8, dtype=torch.float64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for world in (1, 2, 4, 8):
    worst = 0.0
    per = []
    for rank in range(world):
        from paper_2101_08053_b200.distributed import row_block, window_counts
        rb, re_ = row_block(K, world, rank, window_counts(cfg) if world > 1 else None)
        gf = GraphFormation(b2d, cfg, None, "dwq", row_range=(rb, re_))
        ts = []
        for k in range(13):
            flush.fill_(1.0)
            e0.record(); gf.run(); e1.record(); torch.cuda.synchronize()
            if k >= 3:
                ts.append(e0.elapsed_time(e1))
        ts.sort()
        worst = max(worst, ts[len(ts) // 2])
        per.append(round(ts[len(ts) // 2], 3))
        del gf
    print(f"world {world}: per-rank step {worst:.3f} ms  ranks {per}", flush=True)
