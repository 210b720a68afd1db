timeout 300 python scripts/probes/c5_hash.py 256
for v in ns "" ns ""; do lib=paper_2101_08053_b200/libtq_b200${v:+_$v}.so
 TQ_LIB=$PWD/$lib timeout 600 python bench.py --no-config4 --e2e-steps 0 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v c5', d['ms_per_step'], d['kernels_ms_per_step']['fill'], d['parity']['pattern_sha256'])"; done
for v in ns ""; do lib=paper_2101_08053_b200/libtq_b200${v:+_$v}.so; echo "== $v"; TQ_LIB=$PWD/$lib timeout 600 python scripts/probes/rank_probe.py 2>&1 | tail -4; done
