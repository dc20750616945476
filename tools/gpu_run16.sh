python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/sweep.py run head default --cfg C2 --modes fp64,dw,qdw,tw,qtw --iters 100 --out gpurun_out/sweep11_c2.json 2>&1
python tools/sweep.py run head default --cfg C4 --modes fp64,dw,qtw --iters 100 --out gpurun_out/sweep11_c4.json 2>&1
