set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/r2b_tests.log 2>&1; tail -3 gpurun_out/r2b_tests.log
timeout 900 python bench.py > gpurun_out/r2b_bench.log 2>&1; tail -3 gpurun_out/r2b_bench.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1; tail -1 gpurun_out/r2b_smoke.log
python scripts/config4_probe.py 8 256 > gpurun_out/c4p8.log 2>&1; tail -1 gpurun_out/c4p8.log
python scripts/config4_probe.py 6 256 > gpurun_out/c4p6.log 2>&1; tail -1 gpurun_out/c4p6.log
