"""Per-kernel totals of an ncu --csv launch list (gpu__time_duration.sum)."""
import csv, sys
from collections import defaultdict
lines = open(sys.argv[1]).read().splitlines()
k = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[k:]))
h = rows[0]
ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = {}
for r in rows[1:]:
    if len(r) > iv:
        d.setdefault((r[iid], r[ik]), {})[r[im]] = r[iv]
agg = defaultdict(lambda: [0, 0.0])
tot = 0.0
for (i, kname), m in d.items():
    t = float(m.get("gpu__time_duration.sum", "0").replace(",", ""))
    unit_ns = True
    name = kname.split("(")[0].replace("void ", "")[:64]
    agg[name][0] += 1
    agg[name][1] += t
    tot += t
for kname, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{kname:64s} {n:3d} {t / 1e3:9.1f} us {t / tot:6.1%}")
print(f"total {tot / 1e3:.1f} us over {len(d)} launches")
