timeout 600 python scripts/e2e_phases.py 2>&1 | tail -30
timeout 600 python scripts/e2e_cprofile.py 2>&1 | tail -45
