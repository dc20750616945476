set -x
timeout 900 python -m pytest tests/test_gpu_colblocks.py tests/test_gpu_sell_sigma.py tests/test_gpu_dist.py -x -q > gpurun_out/r2u_tests.log 2>&1; tail -3 gpurun_out/r2u_tests.log
timeout 900 python tools/c5_probe.py 16000000 dw,qtw,fp64 > gpurun_out/r2u_c5_tg.log 2>&1; tail -3 gpurun_out/r2u_c5_tg.log
MWCG_TGROUP=0 timeout 900 python tools/c5_probe.py 16000000 dw,qtw,fp64 > gpurun_out/r2u_c5_notg.log 2>&1; tail -3 gpurun_out/r2u_c5_notg.log
MWCG_COLBLOCK=0 timeout 900 python tools/c5_probe.py 16000000 dw > gpurun_out/r2u_c5_noblock_tg.log 2>&1; tail -1 gpurun_out/r2u_c5_noblock_tg.log
E2E_STEPS=4 timeout 600 python tools/e2e_probe2.py > gpurun_out/r2u_e2e.log 2>&1; tail -4 gpurun_out/r2u_e2e.log
