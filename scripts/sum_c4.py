"""Per-kernel totals of an ncu launch list (dev aid)."""
import csv, collections, sys
rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
h = rows[0]; k = h.index("Kernel Name"); v = h.index("Metric Value"); u = h.index("Metric Unit")
sc = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[1:]:
    n = r[k].split("(")[0].replace("void ", "")
    tot[n] += float(r[v].replace(",", "")) * sc[r[u]]; cnt[n] += 1
print("total us", round(sum(tot.values()), 1))
for n, t in sorted(tot.items(), key=lambda x: -x[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 10]:
    print(f"  {n[:45]:45s} {cnt[n]:3d} {t:8.1f}")
