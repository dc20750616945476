set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests/test_gpu_nccl.py tests/test_gpu_api_edges.py -x -q > gpurun_out/r2a_newtests.log 2>&1; tail -3 gpurun_out/r2a_newtests.log
python -m pytest tests -m gpu -q -x > gpurun_out/r2a_gputests.log 2>&1; tail -3 gpurun_out/r2a_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; tail -2 gpurun_out/r2a_bench.err
