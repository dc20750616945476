python bench.py --cpu-seconds 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('full', d['value'], d['e2e']['ms_per_step'])
for m,v in d['per_arithmetic'].items(): print(m, round(v['us_per_iter'],1), round(v['roofline_frac'],3))"
python tools/sweep.py run default default:MWCG_L2PIN_K3=1 --cfg C2 --modes dw,qdw,tw,qtw --iters 60 2>&1
