timeout 1700 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -2
for v in 1 0; do TQ_PAGEABLE_UPLOADS=0 timeout 300 python scripts/probes/e2e_spikes.py plain 2>&1 | tail -6 | python -c "
import sys, json
ts=[json.loads(l)['total'] for l in sys.stdin if l.startswith('{')]
print('e2e steps', ts)"; done
timeout 600 python scripts/e2e_phases.py 2>&1 | tail -14
