python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for c in C2 C4; do python tools/sweep.py run prev default --cfg $c --modes fp64,dw,qdw,tw,qtw --iters 60 --out gpurun_out/sweep20_$c.json 2>&1; done
for m in tw qtw; do timeout 600 ncu --set full --clock-control none -k regex:"cg_spmv_pq" --launch-skip 2 -c 1 -o gpurun_out/ncu_k1_${m}_r1c -f python tools/prof_c2.py --modes $m --iters 4 > /dev/null 2>&1; done
du -sh gpurun_out
