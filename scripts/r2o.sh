for old in 1 0; do TQ_CUTCELLS_OLD=$old bash -c 'echo OLD=$TQ_CUTCELLS_OLD; timeout 300 python scripts/probes/c5_hash.py 256; timeout 300 python scripts/probes/c5_hash.py 1024'; done
for em in 0 1; do for p in 8 6 4; do TQ_GATHER_EM=$em timeout 300 python scripts/probes/c4_hash.py $p 64; done; done
TQ_GATHER_EM=1 timeout 300 python scripts/config4_probe.py 8 256 2>&1 | tail -1 | cut -c1-110; TQ_GATHER_EM=1 timeout 300 python scripts/config4_probe.py 6 256 2>&1 | tail -1 | cut -c1-110
TQ_GATHER_EM=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:k_cut_rows_gather python scripts/config4_probe.py 8 256 prof 2>&1 | grep -E "duration|inst_exec"
for old in 1 0; do TQ_CUTCELLS_OLD=$old timeout 600 python bench.py --no-config4 --e2e-steps 0 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('old=$old ms', d['ms_per_step'], d['kernels_ms_per_step']['fill'])"; done
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:k_raw_cutcells python scripts/step_launches.py 2048 eager 2>&1 | grep -E "k_raw|duration"
TQ_STAMPS=1 timeout 300 python scripts/step_launches.py 2048 stamps 2>&1 | grep -E "side:|join|counts|scan|fill"
