set -x
timeout 1200 python -m pytest tests/test_gpu_colblocks.py -x -q > gpurun_out/r2o_colblocks.log 2>&1; tail -15 gpurun_out/r2o_colblocks.log
timeout 900 python -m pytest tests/test_gpu_sell_sigma.py tests/test_gpu_dist.py tests/test_gpu_nccl.py -x -q > gpurun_out/r2o_misc.log 2>&1; tail -3 gpurun_out/r2o_misc.log
for cb in 0 2097152 4194304 1048576; do MWCG_COLBLOCK=$cb timeout 900 python tools/c5_probe.py 16000000 dw,qtw > gpurun_out/r2o_c5_cb$cb.log 2>&1; tail -4 gpurun_out/r2o_c5_cb$cb.log; done
