timeout 900 python scripts/probes/e2e_bench_spikes.py > gpurun_out/spk.out 2> gpurun_out/spk.err; grep -v '"form"' gpurun_out/spk.err | tail -40; grep -o '"step_seconds": \[[^]]*\]' gpurun_out/spk.out
bash scripts/r2d.sh
