python bench.py --no-per-arith --cpu-seconds 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pin', d['value'], d['e2e']['ms_per_step'])"
MWCG_L2PIN=0 python bench.py --no-per-arith --cpu-seconds 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nopin', d['value'], d['e2e']['ms_per_step'])"
E2E_STEPS=14 python tools/e2e_probe2.py 2>&1 | tail -4
