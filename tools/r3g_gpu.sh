set -x
timeout 1800 python -m pytest tests/test_gpu_scale.py -x -q > gpurun_out/r3g_scale.log 2>&1; tail -5 gpurun_out/r3g_scale.log
