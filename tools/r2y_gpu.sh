set -x
python tools/tail_probe.py C2 > gpurun_out/r2y_tail_c2.log 2>&1; cat gpurun_out/r2y_tail_c2.log | tail -5
python tools/tail_probe.py C4 dw,qtw > gpurun_out/r2y_tail_c4.log 2>&1; tail -2 gpurun_out/r2y_tail_c4.log
python tools/tail_probe.py C1 dw,tw > gpurun_out/r2y_tail_c1.log 2>&1; tail -2 gpurun_out/r2y_tail_c1.log
python tools/k1w_sweep.py --config C2 --modes tw,qtw --variants 'MWCG_X=twcompact' --out gpurun_out/r2y_sweep_c2.json > gpurun_out/r2y_sweep.log 2>&1
python tools/k1w_sweep.py --config C4 --modes qtw --variants 'MWCG_X=twcompact' --out gpurun_out/r2y_sweep_c4.json >> gpurun_out/r2y_sweep.log 2>&1
grep -h '"k1_us"' gpurun_out/r2y_sweep.log | cut -c1-180
