"""Opcode mix (executed warp instructions) from `ncu --page source --csv
--print-source sass` on stdin -- development aid."""
import collections
import csv
import sys

r = list(csv.reader(sys.stdin))
h = next(x for x in r if "Source" in x and "Address" in x)
rows = [x for x in r if x and x[0].startswith("0x")]
i_src, i_ex = h.index("Source"), h.index("Instructions Executed")
c = collections.Counter()
for x in rows:
    ops = [o for o in x[i_src].split() if not o.startswith("@")]
    c[ops[0].split(".")[0] if ops else "?"] += int(x[i_ex] or 0)
tot = sum(c.values())
print("total", tot, " ".join(f"{k}:{100 * v / tot:.0f}%" for k, v in c.most_common(14)))
