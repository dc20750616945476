python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py 2> gpurun_out/b60.err > gpurun_out/bench60.json; python -c "
import json; d=json.load(open('gpurun_out/bench60.json'))
print(d['value'], d['roofline']['frac'], d['roofline']['launch_us'], d['roofline']['stage_us'], d['roofline']['iteration']['frac'], d['e2e']['value'], d['e2e']['ms_per_step_median'])
for m,v in d['per_arithmetic'].items(): print(m, round(v['us_per_iter'],1), round(v['roofline_frac'],3))"
