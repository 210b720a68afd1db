"""Aggregate an ncu report's SASS source page by opcode: instructions
executed and warp-stall samples.  Usage: python scripts/ncu_sass.py rep [top]"""
import csv, io, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
kfilt = ["-k", sys.argv[3]] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, *kfilt, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
k = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
r = list(csv.reader(io.StringIO("\n".join(lines[k:]))))
h = r[0]
ie = h.index("Instructions Executed")
iw = h.index("Warp Stall Sampling (All Samples)")
isrc = h.index("Source")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
agg = defaultdict(lambda: [0.0, 0.0])
stalls = defaultdict(float)
for x in r[1:]:
    op = x[isrc].strip().split()[0] if x[isrc].strip() else "?"
    if op.startswith("@"):
        op = x[isrc].strip().split()[1]
    op = op.split(".")[0]
    agg[op][0] += float(x[ie] or 0)
    agg[op][1] += float(x[iw] or 0)
    for i in stall_cols:
        stalls[h[i]] += float(x[i] or 0)
ti = sum(v[0] for v in agg.values())
tw = sum(v[1] for v in agg.values())
print(f"total instructions {ti:.3e} stall samples {tw:.0f}")
for op, (a, b) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{op:12s} inst {a / ti:6.1%} stall {b / tw:6.1%}")
print("stall reasons:", ", ".join(f"{k[6:]} {v / tw:.0%}" for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]))
