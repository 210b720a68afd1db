for v in 0 1; do TQ_CUTCELL_LISTS=$v timeout 300 python scripts/probes/c5_hash.py 256; done
for v in 0 1 0 1; do TQ_CUTCELL_LISTS=$v timeout 600 python bench.py --no-config4 --e2e-steps 0 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lists=$v c5', d['ms_per_step'], d['parity']['pattern_sha256'])"; done
for v in 0 1; do TQ_CUTCELL_LISTS=$v ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:"k_raw_cutcells" python scripts/step_launches.py 2048 eager 2>&1 | grep -E "duration"; done
