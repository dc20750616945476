python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/bench11.json 2> gpurun_out/bench11.err; tail -2 gpurun_out/bench11.err; python -c "
import json; d=json.load(open('gpurun_out/bench11.json'))
print(d['value'], d['roofline']['frac'], d['roofline']['iteration']['frac'], d['e2e']['value'])
for m,v in d['per_arithmetic'].items(): print(m, round(v['us_per_iter'],1), round(v['roofline_frac'],3), v['bound'])"
