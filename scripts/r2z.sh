for p in 8 6 4; do timeout 300 python scripts/probes/c4_hash.py $p 64; done
timeout 900 python -m pytest tests/test_gpu_planes.py tests/test_gpu_trimmed.py tests/test_gpu_kernel_variants.py -q -x 2>&1 | tail -2
for i in 1 2; do timeout 300 python scripts/config4_probe.py 8 256 2>&1 | tail -1 | cut -c1-110; timeout 300 python scripts/config4_probe.py 6 256 2>&1 | tail -1 | cut -c1-110; done
TQ_STAMPS=1 timeout 300 python scripts/probes/c4_timeline.py 8 256 2>&1 | tail -19
