timeout 300 python scripts/probes/graph_prio.py 2>&1 | tail -3
for v in 0 1 0 1; do echo "prio=$v"; TQ_GRAPH_PRIO=$v timeout 300 python scripts/config4_probe.py 8 256 2>&1 | tail -1 | cut -c60-110; TQ_GRAPH_PRIO=$v timeout 300 python scripts/config4_probe.py 6 256 2>&1 | tail -1 | cut -c60-110
 TQ_GRAPH_PRIO=$v timeout 600 python bench.py --no-config4 --e2e-steps 0 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', d['ms_per_step'], d['roofline']['frac'])"; done
