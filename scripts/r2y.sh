# round-2 late measurement: default bench line, reference arm, config-4 timelines, launch lists
timeout 900 python bench.py > gpurun_out/r2y_bench.log 2>&1; tail -1 gpurun_out/r2y_bench.log > gpurun_out/r2y_bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2y_ref.log 2>&1; tail -1 gpurun_out/r2y_ref.log
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2y_pass_c4p8.csv python scripts/config4_probe.py 8 256 prof > /dev/null 2>&1
python scripts/sum_c4.py gpurun_out/r2y_pass_c4p8.csv 14
TQ_STAMPS=1 timeout 300 python scripts/probes/c4_timeline.py 8 256 > gpurun_out/r2y_timeline_c4p8.txt 2>&1
TQ_STAMPS=1 timeout 300 python scripts/step_launches.py 2048 stamps > gpurun_out/r2y_timeline_c5.txt 2>&1
timeout 600 python scripts/probes/rank_probe.py 2>&1 | tail -4
