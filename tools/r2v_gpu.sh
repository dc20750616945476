set -x
python tools/prof_c2.py --modes tw --iters 5 > gpurun_out/r2v_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cg_update|cg_xpay" --launch-skip 4 -c 2 -o gpurun_out/r2v_ncu_k23_tw -f python tools/prof_c2.py --modes tw --iters 5 > gpurun_out/r2v_ncu.log 2>&1
tail -2 gpurun_out/r2v_ncu.log
python tools/prof_c2.py --modes qtw --iters 5 > gpurun_out/r2v_plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cg_update|cg_spmv" --launch-skip 4 -c 2 -o gpurun_out/r2v_ncu_k12_qtw -f python tools/prof_c2.py --modes qtw --iters 5 > gpurun_out/r2v_ncu2.log 2>&1
tail -2 gpurun_out/r2v_ncu2.log
