python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py > gpurun_out/bench9.json 2> gpurun_out/bench9.err; tail -2 gpurun_out/bench9.err; python -c "
import json; d=json.load(open('gpurun_out/bench9.json'))
print(d['value'], d['roofline']['frac'], d['roofline']['iteration']['frac'], d['e2e']['value'])
for m,v in d['per_arithmetic'].items(): print(m, round(v['us_per_iter'],1), round(v['roofline_frac'],3), v['bound'])"
for m in tw qtw fp64 qdw; do timeout 600 ncu --set full --clock-control none -k regex:"cg_spmv_pq|cg_update|cg_xpay" --launch-skip 6 -c 3 -o gpurun_out/ncu_full_${m}_r1c -f python tools/prof_c2.py --modes $m --iters 5 > /dev/null 2>&1; done
ls gpurun_out/*r1c*
