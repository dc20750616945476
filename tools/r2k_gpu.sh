set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_uniform_slices.py -x -q > gpurun_out/r2k_uniform.log 2>&1; tail -5 gpurun_out/r2k_uniform.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sell_sigma.py tests/test_gpu_dist.py tests/test_gpu_api_edges.py -x -q > gpurun_out/r2k_parity.log 2>&1; tail -3 gpurun_out/r2k_parity.log
python tools/k1w_sweep.py --config C2 --variants 'MWCG_DIA_UNIFORM=0;MWCG_DIA_UNIFORM=1' --out gpurun_out/r2k_sweep_c2.json > gpurun_out/r2k_sweep.log 2>&1
MWCG_LIB=build_var/uu7.so python tools/k1w_sweep.py --config C2 --modes dw,qdw,tw,qtw --variants 'MWCG_DIA_UNIFORM=1' --out gpurun_out/r2k_sweep_c2_uu7.json >> gpurun_out/r2k_sweep.log 2>&1
MWCG_LIB=build_var/uu8.so python tools/k1w_sweep.py --config C2 --modes dw,qdw,tw,qtw --variants 'MWCG_DIA_UNIFORM=1' --out gpurun_out/r2k_sweep_c2_uu8.json >> gpurun_out/r2k_sweep.log 2>&1
python tools/k1w_sweep.py --config C1 --modes fp64,dw,qtw --variants 'MWCG_DIA_UNIFORM=0;MWCG_DIA_UNIFORM=1' --out gpurun_out/r2k_sweep_c1.json >> gpurun_out/r2k_sweep.log 2>&1
grep -h '"k1_us"' gpurun_out/r2k_sweep.log | cut -c1-230
