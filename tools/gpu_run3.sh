python -m pytest tests -m gpu -x -q -k "dist" 2>&1 | tail -2
python bench.py --partitioned --steps 3 --warmup 3 2> gpurun_out/part2.err | tee gpurun_out/part2.json; tail -2 gpurun_out/part2.err
python tools/e2e_probe.py 2>&1 | tail -5
