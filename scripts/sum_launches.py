"""Sum an ncu launch-list CSV by kernel name -- development aid."""
import csv, sys, collections
rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[1:]:
    v = float(r[vi].replace(",", "")); v = {"ns": v / 1e3, "nsecond": v / 1e3, "ms": v * 1e3, "msecond": v * 1e3}.get(r[ui], v)
    name = r[ki].split("(")[0].split("<")[0]
    tot[name] += v; cnt[name] += 1
T = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:10.1f} us {100*v/T:5.1f}%  x{cnt[k]:<4d} {k}")
print(f"{T:10.1f} us total, {sum(cnt.values())} launches")
