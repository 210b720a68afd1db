for i in 1 2; do timeout 300 python scripts/config4_probe.py 8 256 2>&1 | tail -1 | cut -c60-110; timeout 300 python scripts/config4_probe.py 6 256 2>&1 | tail -1 | cut -c60-110; done
ncu --profile-from-start off --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.sum --clock-control none -k regex:"k_cut_pairs" python scripts/config4_probe.py 8 256 prof 2>&1 | grep -E "duration|fp64"
timeout 900 python -m pytest tests/test_gpu_planes.py tests/test_gpu_trimmed.py tests/test_gpu_rowblocks.py -q -x 2>&1 | tail -3
