python tools/e2e_probe2.py 2>&1 | tail -5
