#!/bin/bash
# A/B sweep of the early (head/tail) fill knobs on the config-5 step (development aid)
run() { echo -n "$* : "; env "$@" python bench.py --steps 20 --warmup 3 --no-cpu --no-config4 --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['parity']['pattern_sha256'])"; }
run X=0
run TQ_HEAD_FILL=1 TQ_HEAD_BPS=1
run TQ_HEAD_FILL=1 TQ_HEAD_BPS=2
run TQ_HEAD_FILL=1 TQ_HEAD_BPS=3
run TQ_HEAD_FILL=1 TQ_HEAD_BPS=2 TQ_EARLY_TAIL=1
run TQ_HEAD_FILL=1 TQ_HEAD_BPS=3 TQ_EARLY_TAIL=1
run X=0
