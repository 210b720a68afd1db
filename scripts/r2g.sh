# re-entry validation: GPU suite, smoke, bench line, reference arm
set -x
timeout 1700 python -m pytest tests/ -q -m gpu > gpurun_out/r2g_tests.log 2>&1; tail -2 gpurun_out/r2g_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r2g_bench.log 2>&1; tail -1 gpurun_out/r2g_bench.log > gpurun_out/r2g_bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2g_ref.log 2>&1; tail -1 gpurun_out/r2g_ref.log > gpurun_out/r2g_ref.json
