set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/bench7.json 2> gpurun_out/bench7.err; tail -3 gpurun_out/bench7.err; cat gpurun_out/bench7.json
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref7.json 2>gpurun_out/ref7.err; tail -2 gpurun_out/ref7.err; cat gpurun_out/ref7.json
