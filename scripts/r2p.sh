for v in "" ef "" ef; do lib=paper_2101_08053_b200/libtq_b200${v:+_$v}.so
 TQ_LIB=$PWD/$lib timeout 600 python bench.py --no-config4 --e2e-steps 0 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v c5', d['ms_per_step'], d['kernels_ms_per_step'], d['roofline']['frac'])"; done
