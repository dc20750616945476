python -m pytest tests/test_gpu_parity.py -x -q -k "c1 or acceptance" 2>&1 | tail -2
python tools/sweep.py run default default:MWCG_TMA2=0 default:MWCG_TMA=0 --cfg C2 --modes qtw,qdw --iters 60 2>&1
python bench.py --cpu-seconds 1 --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('full', d['value'])
for m,v in d['per_arithmetic'].items(): print(m, round(v['us_per_iter'],1), round(v['roofline_frac'],3))"
