# round-2 profiles: pass launch lists (config 5, config 4 p=8/p=6), bench launch list,
# ncu --set full of the fill (config 5) and of the config-4 p=8 row kernels
set -x
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_pass_c5.csv python scripts/step_launches.py 2048 eager > /dev/null 2>&1
python scripts/sum_c4.py gpurun_out/r2_pass_c5.csv 25
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_pass_c4p8.csv python scripts/config4_probe.py 8 256 prof > /dev/null 2>&1
python scripts/sum_c4.py gpurun_out/r2_pass_c4p8.csv 25
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_pass_c4p6.csv python scripts/config4_probe.py 6 256 prof > /dev/null 2>&1
python scripts/sum_c4.py gpurun_out/r2_pass_c4p6.csv 12
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_sf_strips|k_planes_csr|k_raw_gauss|k_cut_blocks_wide|k_cut_pairs|k_gauss_pairs|k_coeff_grid" -c 12 -f -o gpurun_out/r2_c4p8_full python scripts/config4_probe.py 8 256 prof > gpurun_out/r2_c4p8_full.log 2>&1; tail -2 gpurun_out/r2_c4p8_full.log
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_fill_tiles|k_fill_irregular" -c 2 -f -o gpurun_out/r2_c5_fill python scripts/step_launches.py 2048 eager > gpurun_out/r2_c5_fill.log 2>&1; tail -2 gpurun_out/r2_c5_fill.log
