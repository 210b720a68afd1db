for m in plain collect; do echo "== $m"; timeout 600 python scripts/probes/e2e_spikes.py $m 2>&1 | tail -12; done
