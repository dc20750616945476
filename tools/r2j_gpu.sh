set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/r2j_cpu.txt
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2j_gputests.log 2>&1; tail -3 gpurun_out/r2j_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err; tail -2 gpurun_out/r2j_bench.err
