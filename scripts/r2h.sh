# planes CSR rows-per-tile A/B (config 4): correctness under both, then timings
set -x
for t in 16 8; do
  TQ_PL_TILE=$t timeout 600 python -m pytest tests/test_gpu_planes.py tests/test_gpu_trimmed.py -q -x 2>&1 | tail -1
  for p in 8 6; do
    for i in 1 2; do TQ_PL_TILE=$t python scripts/config4_probe.py $p 256 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tile $t p $p step_ms', d['step_ms'])"; done
  done
  TQ_PL_TILE=$t ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2h_c4p8_tile$t.csv python scripts/config4_probe.py 8 256 prof > /dev/null 2>&1
  grep planes_csr gpurun_out/r2h_c4p8_tile$t.csv | tail -1
done
