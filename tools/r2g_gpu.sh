set -x
python tools/k1w_sweep.py --config C2 --variants 'MWCG_K1P=0;MWCG_K1P=1' --out gpurun_out/r2g_sweep_c2.json > gpurun_out/r2g_sweep.log 2>&1
python tools/k1w_sweep.py --config C4 --modes fp64,dw,qtw --variants 'MWCG_K1P=0;MWCG_K1P=1' --out gpurun_out/r2g_sweep_c4.json >> gpurun_out/r2g_sweep.log 2>&1
python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2g_parity.log 2>&1; tail -3 gpurun_out/r2g_parity.log
