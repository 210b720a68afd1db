#!/bin/bash
# A/B sweep of stream priorities on the config-5 step (development aid)
run() { echo -n "$* : "; env "$@" python bench.py --steps 20 --warmup 3 --no-cpu --no-config4 --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4))"; }
run X=0
run TQ_PRIO_CUT_BLOCKS=-1 TQ_PRIO_CUT_BLOCKS2=-1
run TQ_PRIO_CUT_BLOCKS=0 TQ_PRIO_CUT_BLOCKS2=0
run TQ_PRIO_CUT_BLOCKS=-1 TQ_PRIO_CUT_BLOCKS2=-1 TQ_PRIO_FITS=-2
run TQ_PRIO_CUT_BLOCKS=0 TQ_PRIO_CUT_BLOCKS2=0 TQ_PRIO_FITS=-1
run TQ_PRIO_FITS=-2
run TQ_PRIO_CAPTURE=-3
run X=0
