# A/B the bench step of this tree against another checkout (dev aid): bash scripts/ab_tree.sh _prev
for i in 1 2 3; do
  for t in . "$@"; do
    echo -n "[$t] "; (cd $t && python bench.py --e2e-steps 0 --no-cpu 2>&1 | grep -o "ms_per_step\": [0-9.]*" | tr "\n" " "); echo
  done
done
