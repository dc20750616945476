python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
python tools/sweep.py run prev default m6 --cfg C2 --modes fp64,dw,qdw,tw,qtw --iters 60 --out gpurun_out/sweep24_c2.json 2>&1
python tools/sweep.py run prev default --cfg C4 --modes fp64,dw,qdw,tw,qtw --iters 60 --out gpurun_out/sweep24_c4.json 2>&1
