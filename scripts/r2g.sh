timeout 900 python bench.py > gpurun_out/r2g_bench.log 2>&1; tail -1 gpurun_out/r2g_bench.log > gpurun_out/r2g_bench.json
TQ_STAMPS=1 timeout 300 python scripts/probes/c4_timeline.py 8 256 > gpurun_out/r2g_timeline_c4p8.txt 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2g_pass_c4p8.csv python scripts/config4_probe.py 8 256 prof > /dev/null 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2g_pass_c4p6.csv python scripts/config4_probe.py 6 256 prof > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_sf_strips|k_cut_pairs<|k_planes_csr|k_gauss_pairs|k_cut_rows_gather" -c 6 -f -o gpurun_out/r2g_c4p8_full python scripts/config4_probe.py 8 256 prof > /dev/null 2>&1
python scripts/ncu_brief.py gpurun_out/r2g_c4p8_full.ncu-rep > gpurun_out/r2g_c4p8_full.txt 2>&1
