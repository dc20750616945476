set -x
timeout 1500 python -m pytest tests/test_gpu_colblocks.py tests/test_gpu_parity.py -x -q > gpurun_out/r3i_tests.log 2>&1; tail -3 gpurun_out/r3i_tests.log
python tools/tail_probe.py C2 dw,qtw > gpurun_out/r3i_tail_c2.log 2>&1; tail -2 gpurun_out/r3i_tail_c2.log
timeout 900 python tools/c5_probe.py 16000000 dw > gpurun_out/r3i_c5.log 2>&1; tail -2 gpurun_out/r3i_c5.log
