"""Top SASS lines by warp-stall samples from `ncu --page source --csv
--print-source sass` output on stdin -- development aid."""
import csv
import sys

r = list(csv.reader(sys.stdin))
h = next(x for x in r if "Source" in x and "Address" in x)
rows = [x for x in r if x and x[0].startswith("0x")]
i_s, i_src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
i_ex = h.index("Instructions Executed")
tot = sum(int(x[i_s] or 0) for x in rows)
print("total samples", tot, "sass lines", len(rows))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
for x in sorted(rows, key=lambda x: -int(x[i_s] or 0))[:n]:
    print(x[i_s].rjust(6), x[i_ex].rjust(9), x[0][-5:], x[i_src][:100])
