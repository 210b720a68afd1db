# A/B two builds of the library on the bench step (dev aid): bash scripts/ab.sh a.so b.so
for i in 1 2 3; do
  for lib in "$@"; do
    echo -n "$lib "; TQ_LIB=$lib python bench.py --e2e-steps 0 --no-cpu 2>&1 | grep -o "ms_per_step\": [0-9.]*\|\"fill\": [0-9.]*" | tr "\n" " "; echo
  done
done
