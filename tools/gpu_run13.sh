python tools/sweep.py run head default novf --cfg C2 --modes fp64,dw,qdw,tw,qtw --iters 100 --out gpurun_out/sweep8_c2.json 2>&1
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
