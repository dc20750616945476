python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for c in C2 C4 C3; do python tools/sweep.py run head dia1 default --cfg $c --modes fp64,dw,qdw,qtw --iters 60 --out gpurun_out/sweep12_$c.json 2>&1; done
