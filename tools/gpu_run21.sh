python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/bench8.json 2> gpurun_out/bench8.err; tail -2 gpurun_out/bench8.err; cat gpurun_out/bench8.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv python bench.py --steps 2 --warmup 3 --no-per-arith --no-e2e --cpu-seconds 1 > gpurun_out/ncu_bench_r1b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cg_spmv_pq" --launch-skip 3 -c 1 -o gpurun_out/ncu_full_k1_dw_r1b -f python tools/prof_c2.py --modes dw --iters 5 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cg_update|cg_xpay" --launch-skip 6 -c 2 -o gpurun_out/ncu_full_k23_dw_r1b -f python tools/prof_c2.py --modes dw --iters 5 > /dev/null 2>&1
ls -la gpurun_out | tail -5
