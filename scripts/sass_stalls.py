"""Top SASS instructions by warp-stall samples of one kernel in an ncu report
(dev aid): python scripts/sass_stalls.py rep.ncu-rep kernel_regex [top]"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass", "-k",
                      "regex:" + sys.argv[2]], capture_output=True, text=True).stdout
lines = out.splitlines()
k = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
r = list(csv.reader(io.StringIO("\n".join(lines[k:]))))
h = r[0]
iw, ie, isrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
rows = [x for x in r[1:] if len(x) > iw and x[0].startswith("0x")]
tw = sum(float(x[iw] or 0) for x in rows)
print("instructions", len(rows), "samples", tw)
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
idx = sorted(range(len(rows)), key=lambda i: -float(rows[i][iw] or 0))[:top]
for i in sorted(idx):
    x = rows[i]
    print(f"{i:5d} {float(x[iw] or 0) / tw:6.1%} {x[isrc].strip()[:90]}")
