"""Aggregate an ncu report's source page by CUDA source line: instructions
executed and warp-stall samples (needs -lineinfo).  Usage:
  python scripts/ncu_source.py report.ncu-rep [top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
k = next(i for i, l in enumerate(lines) if l.startswith('"#",') or l.startswith('"Line"') or '"Source"' in l)
r = list(csv.reader(io.StringIO("\n".join(lines[k:]))))
h = r[0]
ie = next(i for i, c in enumerate(h) if c.startswith("Instructions Executed"))
iw = next(i for i, c in enumerate(h) if c.startswith("Warp Stall Sampling (All"))
isrc = h.index("Source")
il = 0
rows = r[1:]
tot_i = sum(float(x[ie] or 0) for x in rows)
tot_w = sum(float(x[iw] or 0) for x in rows)
print(f"total instructions {tot_i:.3e}, stall samples {tot_w:.0f}")
rows.sort(key=lambda x: -float(x[iw] or 0))
for x in rows[:top]:
    print(f"{x[il]:>5} inst {float(x[ie] or 0) / tot_i:6.1%} stall {float(x[iw] or 0) / tot_w:6.1%}  {x[isrc].strip()[:100]}")
