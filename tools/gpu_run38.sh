python -m pytest tests/test_gpu_parity.py -x -q -k "slice_shared" 2>&1 | tail -2
python tools/sweep.py run default ns1m3 ns1m4 ns2m2 --cfg C2 --modes dw,qdw,qtw --iters 60 --out gpurun_out/sweep26_c2.json 2>&1
