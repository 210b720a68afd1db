# captured-pass timelines under tuning knobs (timeline stamps) -- development aid
for v in "TQ_HEAD_FILL=0" "TQ_HEAD_BPS=1" "TQ_HEAD_BPS=2" "TQ_HEAD_BPS=3" "TQ_HEAD_BPS=2 TQ_PRIO_CAPTURE=-3"; do
  echo "== $v"
  env $v python scripts/step_launches.py 2048 stamps 2>&1 | grep -E "^(head_fill|fits_joined|side:cutcells|counts_deep|join|counts_rest|scan|fill) "
done
