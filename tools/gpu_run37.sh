timeout 900 python tools/c5_probe.py 2>&1 | tail -5
timeout 600 python bench.py --partitioned --steps 3 --warmup 3 > gpurun_out/part3.json 2> gpurun_out/part3.err; tail -2 gpurun_out/part3.err; cut -c1-600 gpurun_out/part3.json
