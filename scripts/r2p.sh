timeout 300 python scripts/probes/c5_hash.py 256; timeout 300 python scripts/probes/c5_hash.py 1024
for i in 1 2; do timeout 600 python bench.py --no-config4 --e2e-steps 0 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', d['ms_per_step'], d['parity']['pattern_sha256'])"; done
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:"k_row_counts_list|k_list_geometry" python scripts/step_launches.py 2048 eager 2>&1 | grep -E "duration|k_row|k_list"
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_rowblocks.py tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_scan.py -q -x 2>&1 | tail -2
