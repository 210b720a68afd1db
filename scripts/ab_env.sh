# A/B environment settings on the bench step (dev aid): bash scripts/ab_env.sh "A=1" "A=2 B=3" ...
for i in 1 2 3; do
  for v in "$@"; do
    echo -n "[$v] "; env $v python bench.py --e2e-steps 0 --no-cpu 2>&1 | grep -o "ms_per_step\": [0-9.]*" | tr "\n" " "; echo
  done
done
