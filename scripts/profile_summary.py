"""Regenerate the committed profile summaries under profiles/ from the ncu
outputs of a gpurun session (dev aid).

  python scripts/profile_summary.py <pass_launches.csv> <bench_launches.csv> <fill.ncu-rep> <tag>

pass_launches: one formation pass (scripts/step_launches.py 2048 eager under
  ncu --profile-from-start off --metrics gpu__time_duration.sum)
bench_launches: the launch list of bench.py --profile-eager under ncu
fill.ncu-rep: ncu --set full of k_fill_tiles and k_fill_irregular
"""
import collections, csv, json, os, shutil, subprocess, sys

pass_csv, bench_csv, rep, tag = sys.argv[1:5]
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
shutil.copy(pass_csv, os.path.join(out, f"{tag}_pass_launches_config5.csv"))
shutil.copy(bench_csv, os.path.join(out, f"{tag}_bench_launches_config5.csv"))

def launches(path):
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    h = rows[0]
    k, v, u = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    return [(r[k].split("(")[0].replace("void ", "").split("<")[0], float(r[v].replace(",", "")) * scale[r[u]])
            for r in rows[1:] if r[v]]

tot = collections.defaultdict(float)
cnt = collections.Counter()
for name, us in launches(pass_csv):
    tot[name] += us
    cnt[name] += 1
T = sum(tot.values())
print("| kernel | launches | µs (cold, serialised) | share |")
print("|---|---|---|---|")
for name, us in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"| `{name}` | {cnt[name]} | {us:.1f} | {100 * us / T:.1f}% |")
print(f"| **total** | {sum(cnt.values())} | {T:.1f} | |")

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units = rows[0], rows[1]
keep = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum"]
cols = [h.index(c) for c in keep if c in h]
with open(os.path.join(out, f"{tag}_ncu_full_fill.csv"), "w", newline="") as fh:
    w = csv.writer(fh)
    w.writerow([h[c] for c in cols])
    w.writerow([units[c] for c in cols])
    for r in rows[2:]:
        w.writerow([r[c] for c in cols])

def to_bytes(val, unit):
    return float(val.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]

dram = 0.0
per = {}
for r in rows[2:]:
    b = sum(to_bytes(r[h.index(m)], units[h.index(m)]) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    per[r[h.index("Kernel Name")].split("(")[0]] = b
    dram += b
summary = {"dram_bytes_per_launch": dram, "per_kernel_dram_bytes": per,
           "source": f"ncu --set full of k_fill_tiles + k_fill_irregular (one fill), {os.path.basename(rep)}"}
json.dump(summary, open(os.path.join(out, "fill_ncu_summary.json"), "w"), indent=1)
print(json.dumps(summary))
