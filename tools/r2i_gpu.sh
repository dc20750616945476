set -x
python -m pytest tests/test_gpu_sell_sigma.py -x -q > gpurun_out/r2i_sigma.log 2>&1; tail -3 gpurun_out/r2i_sigma.log
python -m pytest tests/test_gpu_k1w.py tests/test_gpu_api_edges.py tests/test_gpu_nccl.py tests/test_gpu_dist.py -x -q > gpurun_out/r2i_misc.log 2>&1; tail -3 gpurun_out/r2i_misc.log
python -m pytest tests/test_gpu_scale.py -x -q -k "C2 or C3 or C5s or first" > gpurun_out/r2i_scale.log 2>&1; tail -3 gpurun_out/r2i_scale.log
