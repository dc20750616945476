set -x
python tools/k1w_sweep.py --config C2 --variants 'MWCG_X=k2minb' --out gpurun_out/r3j_sweep_c2.json > gpurun_out/r3j_sweep.log 2>&1
python tools/k1w_sweep.py --config C4 --modes fp64,dw,qdw,qtw --variants 'MWCG_X=k2minb' --out gpurun_out/r3j_sweep_c4.json >> gpurun_out/r3j_sweep.log 2>&1
python tools/k1w_sweep.py --config C3 --modes dw,qtw --variants 'MWCG_X=k2minb' --out gpurun_out/r3j_sweep_c3.json >> gpurun_out/r3j_sweep.log 2>&1
grep -h '"k1_us"' gpurun_out/r3j_sweep.log | cut -c1-260
