ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_wq_fit|k_basis_eval_multi" -c 4 -f -o gpurun_out/r2_fit python scripts/step_launches.py 2048 eager > /dev/null 2>&1
python scripts/ncu_brief.py gpurun_out/r2_fit.ncu-rep | grep -v "lg_thr\|compute_mem"
