for i in 1 2; do timeout 300 python scripts/config4_probe.py 8 256 2>&1 | tail -1 | cut -c60-110; timeout 300 python scripts/config4_probe.py 6 256 2>&1 | tail -1 | cut -c60-110; done
ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__registers_per_thread,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,launch__block_size --clock-control none --csv python scripts/config4_probe.py 8 256 prof 2>/dev/null > gpurun_out/regs.csv; python - <<'PY'
import csv
rows = list(csv.reader(l for l in open("gpurun_out/regs.csv") if l.startswith('"')))
h = rows[0]; k = h.index("Kernel Name"); m = h.index("Metric Name"); v = h.index("Metric Value")
d = {}
for r in rows[1:]:
    n = r[k].split("(")[0][-40:]
    d.setdefault(n, {})[r[m]] = r[v]
for n, x in d.items():
    print(f"{n:40s} {x.get('gpu__time_duration.sum'):>10s} regs {x.get('launch__registers_per_thread'):>4s} blk {x.get('launch__block_size'):>4s} lim_reg {x.get('launch__occupancy_limit_registers'):>3s} lim_smem {x.get('launch__occupancy_limit_shared_mem'):>3s}")
PY
