set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api_edges.py tests/test_gpu_dist.py -x -q > gpurun_out/r3h_tests.log 2>&1; tail -3 gpurun_out/r3h_tests.log
python tools/tail_probe.py C2 > gpurun_out/r3h_tail_c2.log 2>&1; cat gpurun_out/r3h_tail_c2.log | tail -5
python tools/k1w_sweep.py --config C2 --variants 'MWCG_X=prefetch' --out gpurun_out/r3h_sweep_c2.json > gpurun_out/r3h_sweep.log 2>&1
python tools/k1w_sweep.py --config C1 --modes dw,qtw --variants 'MWCG_X=prefetch' --out gpurun_out/r3h_sweep_c1.json >> gpurun_out/r3h_sweep.log 2>&1
grep -h '"k1_us"' gpurun_out/r3h_sweep.log | cut -c1-150
