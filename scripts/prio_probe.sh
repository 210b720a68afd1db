# stream-priority layouts of the captured pass (timeline stamps) -- development aid
for v in "" "TQ_PRIO_CAPTURE=-3" "TQ_PRIO_CAPTURE=-3 TQ_PRIO_CUT_BLOCKS=-3 TQ_PRIO_CUT_BLOCKS2=-3" "TQ_PRIO_CAPTURE=-3 TQ_PRIO_CUT_BLOCKS=-3" "TQ_PRIO_CAPTURE=-3 TQ_PRIO_CUT_BLOCKS=-3 TQ_PRIO_FITS=-2" "TQ_PRIO_CAPTURE=-2 TQ_PRIO_CUT_BLOCKS=-3 TQ_PRIO_CUT_BLOCKS2=-3 TQ_PRIO_FITS=-3"; do
  echo "== $v"
  env $v python scripts/step_launches.py 2048 stamps 2>&1 | grep -E "^(preA:|preB:|cutpre|fits_joined|weights|raw_interior|side:|counts_deep|join|counts_rest|scan|fill)"
done
