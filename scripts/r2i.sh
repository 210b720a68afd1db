# last validation of round 2: GPU suite, smoke, bench + reference arm, launch lists, fill ncu
set -x
timeout 1700 python -m pytest tests/ -q -m gpu > gpurun_out/r2i_tests.log 2>&1; tail -2 gpurun_out/r2i_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r2i_bench.log 2>&1; tail -1 gpurun_out/r2i_bench.log > gpurun_out/r2i_bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2i_ref.log 2>&1; tail -1 gpurun_out/r2i_ref.log > gpurun_out/r2i_ref.json
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2i_pass_c5.csv python scripts/step_launches.py 2048 eager > /dev/null 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2i_pass_c4p8.csv python scripts/config4_probe.py 8 256 prof > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r2i_bench_launches.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu --no-config4 --profile-eager > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_fill_tiles|k_fill_irregular" -c 2 -f -o gpurun_out/r2i_fill python scripts/step_launches.py 2048 eager > /dev/null 2>&1
python scripts/ncu_brief.py gpurun_out/r2i_fill.ncu-rep > gpurun_out/r2i_fill.txt 2>&1
