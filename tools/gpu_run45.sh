python tools/e2e_probe2.py 2>&1 | tail -3
MWCG_L2PIN=0 python tools/e2e_probe2.py 2>&1 | tail -3
