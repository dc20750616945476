set -x
python tools/k1w_sweep.py --config C2 --modes dw,qdw,qtw,tw --variants 'MWCG_L2PIN=0;MWCG_L2PIN=16;MWCG_UNROLL=16;MWCG_X=default' --out gpurun_out/r3f_sweep_c2.json > gpurun_out/r3f_sweep.log 2>&1
python tools/k1w_sweep.py --config C4 --modes dw,qtw --variants 'MWCG_L2PIN=0;MWCG_X=default' --out gpurun_out/r3f_sweep_c4.json >> gpurun_out/r3f_sweep.log 2>&1
grep -h '"k1_us"' gpurun_out/r3f_sweep.log | cut -c1-150
