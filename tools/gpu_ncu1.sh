timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cg_spmv_pq|cg_update|cg_xpay" --launch-skip 3 -c 3 -o gpurun_out/ncu_dw_c2 -f python tools/prof_c2.py --modes dw --iters 3 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cg_spmv_pq" --launch-skip 1 -c 1 -o gpurun_out/ncu_fp64_c2 -f python tools/prof_c2.py --modes fp64 --iters 3 >> gpurun_out/ncu1.log 2>&1
tail -3 gpurun_out/ncu1.log
