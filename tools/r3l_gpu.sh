set -x
python tools/e2e_outlier_probe.py > gpurun_out/r3l_e2e_gc1.log 2>&1; cat gpurun_out/r3l_e2e_gc1.log | tail -12
E2E_GC=0 python tools/e2e_outlier_probe.py > gpurun_out/r3l_e2e_gc0.log 2>&1; cat gpurun_out/r3l_e2e_gc0.log | tail -12
timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -k "C4s" > gpurun_out/r3l_scale.log 2>&1; tail -2 gpurun_out/r3l_scale.log
