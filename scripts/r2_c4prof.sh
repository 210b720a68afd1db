# config-4 p=8 profiles (round 2): pass launch list + ncu --set full of the three c != 1 row kernels
python scripts/config4_probe.py 8 256 > gpurun_out/c4p8.log 2>&1; tail -1 gpurun_out/c4p8.log
python scripts/config4_probe.py 6 256 > gpurun_out/c4p6.log 2>&1; tail -1 gpurun_out/c4p6.log
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4p8_launches.csv python scripts/config4_probe.py 8 256 prof > /dev/null 2>&1
python scripts/sum_c4.py gpurun_out/c4p8_launches.csv 20
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_raw_sf_coef|k_raw_gauss_coef|k_cut_blocks_wide|k_row_counts_list|k_fill_rows" -c 6 -f -o gpurun_out/c4p8_full python scripts/config4_probe.py 8 256 prof > gpurun_out/c4p8_full.log 2>&1; tail -3 gpurun_out/c4p8_full.log
