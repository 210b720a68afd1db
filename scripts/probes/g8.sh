timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/r2b_tests.log 2>&1; tail -3 gpurun_out/r2b_tests.log
timeout 600 python scripts/probes/rank_probe.py 2>&1 | tail -4
