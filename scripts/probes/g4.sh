timeout 300 python scripts/probes/planes_check.py 2>&1 | grep -v "^frame" | tail -10
python scripts/config4_probe.py 8 256 | cut -c1-140; python scripts/config4_probe.py 6 256 | cut -c1-140
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4p8_planes.csv python scripts/config4_probe.py 8 256 prof > /dev/null 2>&1
python scripts/sum_c4.py gpurun_out/c4p8_planes.csv 10
