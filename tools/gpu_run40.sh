for c in C2 C4; do python tools/sweep.py run default sel --cfg $c --modes fp64,dw,qdw,qtw --iters 60 --out gpurun_out/sweep28_$c.json 2>&1; done
