python -m pytest tests/ -q -m gpu -x > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
python bench.py --e2e-steps 0 --no-cpu > gpurun_out/b.log 2>&1
grep -o "\"value\": [0-9.]*\|ms_per_step\": [0-9.]*\|\"fill\": [0-9.]*\|frac\": [0-9.]*\|Error.*" gpurun_out/b.log | head -5
