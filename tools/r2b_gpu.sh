set -x
python -m pytest tests/test_gpu_k1w.py -x -q > gpurun_out/r2b_k1w.log 2>&1; tail -3 gpurun_out/r2b_k1w.log
python -m pytest tests -m gpu -q -x > gpurun_out/r2b_gputests.log 2>&1; tail -3 gpurun_out/r2b_gputests.log
python bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; tail -2 gpurun_out/r2b_bench.err
MWCG_K1W=0 python bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/r2b_bench_k1w0.json 2> gpurun_out/r2b_bench_k1w0.err; tail -2 gpurun_out/r2b_bench_k1w0.err
