timeout 300 python scripts/probes/c5_hash.py 256; timeout 300 python scripts/probes/c5_hash.py 1024
for g in 0 1; do TQ_GEOMETRIC_NEAR=$g timeout 600 python bench.py --no-cpu --no-config4 --e2e-steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('near=$g', d['ms_per_step'], d['parity']['pattern_sha256'], d['e2e']['median_seconds'])"; done
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:k_row_counts_list python scripts/step_launches.py 2048 eager 2>&1 | grep -E "duration"
TQ_STAMPS=1 timeout 300 python scripts/step_launches.py 2048 stamps 2>&1 | grep -E "side:|join|counts|scan|fill"
timeout 1700 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -2
