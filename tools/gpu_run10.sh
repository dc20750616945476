./tools/spmv_probe > gpurun_out/probe1.txt 2>&1; cat gpurun_out/probe1.txt
python tools/sweep.py run default --cfg C2 --modes fp64,dw,qdw,tw,qtw --iters 100 --out gpurun_out/sweep5_c2.json 2>&1
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
