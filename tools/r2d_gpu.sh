set -x
python tools/prof_c2.py --modes dw --iters 4 > gpurun_out/r2d_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cg_spmv_pq" --launch-skip 2 -c 1 \
    -o gpurun_out/r2d_k1w_dw -f python tools/prof_c2.py --modes dw --iters 4 > gpurun_out/r2d_ncu.log 2>&1
MWCG_K1W=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cg_spmv_pq" --launch-skip 2 -c 1 \
    -o gpurun_out/r2d_k1_dw -f python tools/prof_c2.py --modes dw --iters 4 >> gpurun_out/r2d_ncu.log 2>&1
tail -3 gpurun_out/r2d_ncu.log
