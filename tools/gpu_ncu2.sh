M=gpu__time_duration.sum,dram__bytes_read.sum,sm__warps_active.avg.per_cycle_active,launch__registers_per_thread,launch__grid_size
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/k1_launches_part.csv python tools/prof_c2.py --modes fp64,dw --iters 4 --red partitions > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/k1_launches_tile.csv python tools/prof_c2.py --modes fp64,dw --iters 4 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cg_spmv_pq_tma" --launch-skip 2 -c 1 -o gpurun_out/ncu_k1t_dw -f python tools/prof_c2.py --modes dw --iters 4 > /dev/null 2>&1
ls gpurun_out
