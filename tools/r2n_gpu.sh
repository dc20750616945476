set -x
timeout 900 python -m pytest tests/test_gpu_uniform_slices.py tests/test_gpu_parity.py -x -q > gpurun_out/r2n_parity.log 2>&1; tail -3 gpurun_out/r2n_parity.log
python tools/k1w_sweep.py --config C2 --variants 'MWCG_GRID_FULL=0;MWCG_GRID_FULL=1' --modes fp64,dw,qdw,qtw --out gpurun_out/r2n_sweep_c2.json > gpurun_out/r2n_sweep.log 2>&1
python tools/k1w_sweep.py --config C2 --variants 'MWCG_X=1' --modes tw --out gpurun_out/r2n_sweep_c2_tw.json >> gpurun_out/r2n_sweep.log 2>&1
for v in uu6 uu7 uu8; do MWCG_LIB=build_var/$v.so python tools/k1w_sweep.py --config C2 --modes dw,qdw,qtw --variants "MWCG_V=$v" --out gpurun_out/r2n_sweep_c2_$v.json >> gpurun_out/r2n_sweep.log 2>&1; done
python tools/k1w_sweep.py --config C4 --modes fp64,dw,qdw,qtw --variants 'MWCG_GRID_FULL=0;MWCG_GRID_FULL=1' --out gpurun_out/r2n_sweep_c4.json >> gpurun_out/r2n_sweep.log 2>&1
python tools/k1w_sweep.py --config C3 --modes fp64,dw,qtw --variants 'MWCG_GRID_FULL=0;MWCG_GRID_FULL=1' --out gpurun_out/r2n_sweep_c3.json >> gpurun_out/r2n_sweep.log 2>&1
grep -h '"k1_us"' gpurun_out/r2n_sweep.log | cut -c1-200
