TQ_STAMPS=1 timeout 300 python scripts/probes/c4_timeline.py 8 256 2>&1 | tail -40
timeout 900 python scripts/probes/e2e_bench_spikes.py > gpurun_out/spk.out 2> gpurun_out/spk.err; grep -v '"form"' gpurun_out/spk.err | tail -40; grep -o '"step_seconds": \[[^]]*\]' gpurun_out/spk.out
