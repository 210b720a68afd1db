for p in 8 6 4; do timeout 300 python scripts/probes/c4_hash.py $p 64; done
for i in 1 2; do timeout 300 python scripts/config4_probe.py 8 256 2>&1 | tail -1 | cut -c60-110; timeout 300 python scripts/config4_probe.py 6 256 2>&1 | tail -1 | cut -c60-110; done
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:"k_gauss_pairs" python scripts/config4_probe.py 8 256 prof 2>&1 | grep -E "duration"
timeout 900 python -m pytest tests/test_gpu_planes.py tests/test_gpu_trimmed.py -q -x 2>&1 | tail -2
