set -x
export C5_KERNELS=1
timeout 600 python tools/c5_probe.py 16000000 dw > gpurun_out/r2p_plain.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on -k regex:cg_spmv_pq -s 16 -c 8 -o gpurun_out/r2p_c5_k1_dw -f python tools/c5_probe.py 16000000 dw > gpurun_out/r2p_ncu.log 2>&1
tail -3 gpurun_out/r2p_plain.log; tail -5 gpurun_out/r2p_ncu.log
ls -la gpurun_out/*.ncu-rep
