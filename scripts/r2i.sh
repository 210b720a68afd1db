ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_row_counts_list" -c 1 -f -o gpurun_out/r2_cntlist python scripts/step_launches.py 2048 eager > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_planes_csr" -c 1 -f -o gpurun_out/r2_planes python scripts/config4_probe.py 8 256 prof > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_cut_rows_gather" -c 1 -f -o gpurun_out/r2_gather python scripts/config4_probe.py 8 256 prof > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
