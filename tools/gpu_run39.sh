python -m pytest tests/test_gpu_parity.py -x -q -k "tw" 2>&1 | tail -2
python tools/sweep.py run noskip default --cfg C2 --modes tw --iters 60 --out gpurun_out/sweep27_c2.json 2>&1
python tools/sweep.py run noskip default --cfg C4 --modes tw --iters 60 --out gpurun_out/sweep27_c4.json 2>&1
