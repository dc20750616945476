set -x
python -m pytest tests -m gpu -x -q -k "dist" 2>&1 | tail -3
python bench.py --partitioned --steps 3 --warmup 3 > gpurun_out/part1.json 2> gpurun_out/part1.err; tail -2 gpurun_out/part1.err
cat gpurun_out/part1.json
