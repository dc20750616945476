python bench.py --partitioned --steps 3 --warmup 3 > gpurun_out/part1.json 2> gpurun_out/part1.err; tail -2 gpurun_out/part1.err; cat gpurun_out/part1.json
python bench.py > gpurun_out/bench6.json 2> gpurun_out/bench6.err; tail -2 gpurun_out/bench6.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-per-arith --no-e2e --cpu-seconds 1 > gpurun_out/ncu_bench.log 2>&1
tail -2 gpurun_out/ncu_bench.log; wc -l gpurun_out/launches_bench.csv
