set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/r2a_tests.log 2>&1; tail -3 gpurun_out/r2a_tests.log
timeout 900 python bench.py > gpurun_out/r2a_bench.log 2>&1; tail -2 gpurun_out/r2a_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2a_ref.log 2>&1; tail -1 gpurun_out/r2a_ref.log
