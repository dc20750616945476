python tools/sweep.py run default xtw_m2 xtw_m4 --cfg C2 --modes tw,qtw --iters 60 --out gpurun_out/sweep14_c2.json 2>&1
