python bench.py > gpurun_out/bench12.json 2> gpurun_out/bench12.err; tail -2 gpurun_out/bench12.err; python -c "
import json; d=json.load(open('gpurun_out/bench12.json'))
print(d['value'], d['roofline']['frac'], d['roofline']['iteration']['frac'], d['e2e']['value'], d['clocks'])
for m,v in d['per_arithmetic'].items(): print(m, round(v['us_per_iter'],1), round(v['roofline_frac'],3), v['bound'])"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref12.json 2>/dev/null; cut -c1-300 gpurun_out/ref12.json
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
ncu --metrics $M --cache-control none --clock-control none -k regex:"cg_spmv_pq|cg_update|cg_xpay" --csv --log-file gpurun_out/k123_launches_c2e.csv python tools/prof_c2.py --modes fp64,dw,qdw,tw,qtw --iters 6 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r1e.csv python bench.py --steps 2 --warmup 3 --no-per-arith --no-e2e --cpu-seconds 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cg_spmv_pq" --launch-skip 3 -c 1 -o gpurun_out/ncu_k1_dw_r1e -f python tools/prof_c2.py --modes dw --iters 5 > /dev/null 2>&1
du -sh gpurun_out
