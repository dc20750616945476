set -x
python -m pytest tests/test_gpu_k1w.py -x -q -k "default or every" > gpurun_out/r2e_k1w.log 2>&1; tail -3 gpurun_out/r2e_k1w.log
python tools/k1w_sweep.py --config C2 --variants 'MWCG_K1W=0;MWCG_K1W=1;MWCG_K1W=1,MWCG_K1W_R=256' --out gpurun_out/r2e_sweep_c2.json > gpurun_out/r2e_sweep.log 2>&1
python tools/k1w_sweep.py --config C4 --modes dw,qtw --variants 'MWCG_K1W=0;MWCG_K1W=1;MWCG_K1W=1,MWCG_K1W_R=256' --out gpurun_out/r2e_sweep_c4.json >> gpurun_out/r2e_sweep.log 2>&1
tail -2 gpurun_out/r2e_sweep.log
