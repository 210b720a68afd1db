TQ_STAMPS=1 timeout 300 python scripts/step_launches.py 2048 stamps 2>&1 | tail -45
timeout 300 python scripts/probes/gc_census.py 2>&1 | tail -8
timeout 600 python scripts/probes/rank_probe.py 2>&1 | tail -4
