ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4p8_planes.csv python scripts/config4_probe.py 8 256 prof > /dev/null 2>&1
python scripts/sum_c4.py gpurun_out/c4p8_planes.csv 10
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_sf_strips|k_planes_csr" -c 3 -f -o gpurun_out/c4p8_planes_full python scripts/config4_probe.py 8 256 prof > gpurun_out/c4p8_planes_full.log 2>&1; tail -1 gpurun_out/c4p8_planes_full.log
