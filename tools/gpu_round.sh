# The standard GPU check of a change (run through gpurun from the repo root):
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh'
# parity tests, smoke, the bench line, the launch list and one full capture of
# the dominant kernel (each profiler pass only after its command ran clean).
set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
ncu --metrics $M --cache-control none --clock-control none -k regex:"cg_spmv_pq|cg_update|cg_xpay" --csv \
    --log-file gpurun_out/k123_launches.csv python tools/prof_c2.py --modes fp64,dw,qdw,tw,qtw --iters 6 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-per-arith --no-e2e --cpu-seconds 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cg_spmv_pq" --launch-skip 3 -c 1 \
    -o gpurun_out/ncu_k1_dw -f python tools/prof_c2.py --modes dw --iters 5 > /dev/null 2>&1
