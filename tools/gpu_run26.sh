python tools/sweep.py run default u6 u7 u8 u8m4 --cfg C2 --modes fp64,dw,qdw,qtw --iters 60 --out gpurun_out/sweep19_c2.json 2>&1
python tools/sweep.py run default u6 u8 --cfg C4 --modes fp64,dw,qdw,qtw --iters 60 --out gpurun_out/sweep19_c4.json 2>&1
