set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_uniform_slices.py tests/test_gpu_bounds.py -x -q > gpurun_out/r3e_tests.log 2>&1; tail -3 gpurun_out/r3e_tests.log
python tools/k1w_sweep.py --config C2 --variants 'MWCG_X=full64' --out gpurun_out/r3e_sweep_c2.json > gpurun_out/r3e_sweep.log 2>&1
python tools/k1w_sweep.py --config C4 --modes fp64,dw,qtw --variants 'MWCG_X=full64' --out gpurun_out/r3e_sweep_c4.json >> gpurun_out/r3e_sweep.log 2>&1
python tools/k1w_sweep.py --config C3 --modes fp64,dw --variants 'MWCG_X=full64' --out gpurun_out/r3e_sweep_c3.json >> gpurun_out/r3e_sweep.log 2>&1
grep -h '"k1_us"' gpurun_out/r3e_sweep.log | cut -c1-150
