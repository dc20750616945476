python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in C2 C4; do python tools/sweep.py run default --cfg $c --modes fp64,dw,qdw,tw,qtw --iters 60 --out gpurun_out/sweep23_$c.json 2>&1; done
python bench.py > gpurun_out/bench10.json 2> gpurun_out/bench10.err; tail -2 gpurun_out/bench10.err; python -c "
import json; d=json.load(open('gpurun_out/bench10.json'))
print(d['value'], d['roofline']['frac'], d['roofline']['iteration']['frac'], d['e2e']['value'])
for m,v in d['per_arithmetic'].items(): print(m, round(v['us_per_iter'],1), round(v['roofline_frac'],3), v['bound'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cg_spmv_pq" --launch-skip 3 -c 1 -o gpurun_out/ncu_k1_dw_r1d -f python tools/prof_c2.py --modes dw --iters 5 > /dev/null 2>&1
du -sh gpurun_out
