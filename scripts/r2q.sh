for combo in "-2 -2" "-2 -4" "-4 -4" "-2 -5" "-4 -5" "-5 -5"; do set -- $combo
  r8=$(TQ_PRIO_CUT_BLOCKS=$1 TQ_PRIO_CUT_BLOCKS2=$2 timeout 300 python scripts/config4_probe.py 8 256 2>&1 | tail -1 | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['step_ms'],4))")
  r6=$(TQ_PRIO_CUT_BLOCKS=$1 TQ_PRIO_CUT_BLOCKS2=$2 timeout 300 python scripts/config4_probe.py 6 256 2>&1 | tail -1 | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['step_ms'],4))")
  r5=$(TQ_PRIO_CUT_BLOCKS=$1 TQ_PRIO_CUT_BLOCKS2=$2 timeout 600 python bench.py --no-config4 --e2e-steps 0 --no-cpu 2>/dev/null | python -c "import json,sys; print(round(json.loads(sys.stdin.readlines()[-1])['ms_per_step'],4))")
  echo "cut_blocks=$1 cut_blocks2=$2  c4p8 $r8  c4p6 $r6  c5 $r5"
done
