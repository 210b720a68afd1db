timeout 900 python -m pytest tests/test_gpu_planes.py tests/test_gpu_trimmed.py -q -x 2>&1 | tail -2
TQ_STAMPS=1 timeout 300 python scripts/probes/c4_timeline.py 8 256 2>&1 | tail -20
timeout 300 python scripts/config4_probe.py 8 256 2>&1 | tail -1 | cut -c1-110
