M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
ncu --metrics $M --cache-control none --clock-control none -k regex:"cg_spmv_pq|cg_update|cg_xpay" --csv --log-file gpurun_out/k123_launches_c2.csv python tools/prof_c2.py --modes fp64,dw,qdw,tw,qtw --iters 6 > /dev/null 2>&1
ls -la gpurun_out/k123_launches_c2.csv
