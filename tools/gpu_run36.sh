python tools/sweep.py run default u2m5 u3 m3 --cfg C2 --modes dw,qdw,tw,qtw --iters 60 --out gpurun_out/sweep25_c2.json 2>&1
