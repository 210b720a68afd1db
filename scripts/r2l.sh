for conf in "" "expandable_segments:True" "backend:cudaMallocAsync"; do
  PYTORCH_CUDA_ALLOC_CONF="$conf" timeout 600 python bench.py --no-config4 --no-cpu --e2e-steps 16 --steps 5 > gpurun_out/al.log 2>&1
  python -c "
import json,sys
l=[x for x in open('gpurun_out/al.log') if x.startswith('{')]
d=json.loads(l[-1]); e=d['e2e']; print(repr('$conf'), 'ms', round(d['ms_per_step'],4), 'e2e mean', round(e['seconds_per_step'],4), 'median', round(e['median_seconds'],4), e['step_seconds'])" || tail -5 gpurun_out/al.log
done
