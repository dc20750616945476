set -x
timeout 600 python -m pytest tests/test_gpu_colblocks.py tests/test_gpu_sell_sigma.py -x -q > gpurun_out/r2r_tests.log 2>&1; tail -3 gpurun_out/r2r_tests.log
timeout 900 python tools/c5_probe.py 16000000 dw,qtw,fp64 > gpurun_out/r2r_c5_default.log 2>&1; tail -3 gpurun_out/r2r_c5_default.log
MWCG_COLBLOCK=0 timeout 900 python tools/c5_probe.py 16000000 dw > gpurun_out/r2r_c5_noblock.log 2>&1; tail -1 gpurun_out/r2r_c5_noblock.log
MWCG_COLBLOCK=1048576 timeout 900 python tools/c5_probe.py 16000000 dw > gpurun_out/r2r_c5_1m.log 2>&1; tail -1 gpurun_out/r2r_c5_1m.log
MWCG_COLBLOCK=3145728 timeout 900 python tools/c5_probe.py 16000000 dw > gpurun_out/r2r_c5_3m.log 2>&1; tail -1 gpurun_out/r2r_c5_3m.log
