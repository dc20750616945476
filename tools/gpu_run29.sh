python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q 2>&1 | tail -2
for c in C2 C4; do python tools/sweep.py run prev default --cfg $c --modes fp64,dw,qdw,tw,qtw --iters 60 --out gpurun_out/sweep21_$c.json 2>&1; done
