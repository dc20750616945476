for i in 1 2; do
python bench.py --cpu-seconds 1 --no-per-arith 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('noper', d['value'], d['e2e']['ms_per_step'])"
python bench.py --cpu-seconds 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('per', d['value'], d['e2e']['ms_per_step'])"
done
MWCG_L2PIN=0 python bench.py --cpu-seconds 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('per-nopin', d['value'], d['e2e']['ms_per_step'])"
