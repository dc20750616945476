set -x
python tools/prof_c2.py --modes tw --iters 5 > gpurun_out/r3o_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cg_update|cg_spmv_pq" --launch-skip 4 -c 2 -o gpurun_out/r3o_ncu_k12_tw -f python tools/prof_c2.py --modes tw --iters 5 > gpurun_out/r3o_ncu.log 2>&1
tail -2 gpurun_out/r3o_ncu.log
