python tools/sweep.py run head default m3 m2 u2_m4 --cfg C2 --modes fp64,dw,qdw,tw,qtw --iters 100 --out gpurun_out/sweep7_c2.json 2>&1
