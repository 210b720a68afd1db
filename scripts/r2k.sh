timeout 600 python scripts/e2e_cprofile.py > gpurun_out/cprof.txt 2>&1; grep -n "call \|function calls" gpurun_out/cprof.txt
