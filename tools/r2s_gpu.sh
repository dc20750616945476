# full GPU round on the current tree: tests, smoke, bench, launch lists, K1 capture
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/r2s_cpu.txt
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2s_gputests.log 2>&1; tail -3 gpurun_out/r2s_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err; tail -2 gpurun_out/r2s_bench.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
python tools/prof_c2.py --modes fp64,dw,qdw,tw,qtw --iters 6 > /dev/null 2>&1 && ncu --metrics $M --cache-control none --clock-control none -k regex:"cg_spmv_pq|cg_update|cg_xpay" --csv \
    --log-file gpurun_out/r2s_k123_launches.csv python tools/prof_c2.py --modes fp64,dw,qdw,tw,qtw --iters 6 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s_launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-per-arith --no-e2e --cpu-seconds 1 --extra-configs "" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cg_spmv_pq" --launch-skip 3 -c 1 \
    -o gpurun_out/r2s_ncu_k1_dw -f python tools/prof_c2.py --modes dw --iters 5 > /dev/null 2>&1
ls -la gpurun_out/r2s_*
