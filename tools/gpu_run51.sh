python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --cpu-seconds 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('full', d['value'], d['e2e']['value'], d['gpu_launches'])
for m,v in d['per_arithmetic'].items(): print(m, round(v['us_per_iter'],1), round(v['roofline_frac'],3))"
