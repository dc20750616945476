set -x
MWCG_LIB=build_var/pair3.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_uniform_slices.py -x -q > gpurun_out/r3c_tests.log 2>&1; tail -3 gpurun_out/r3c_tests.log
for v in pair2 pair3 pair4 pair3m3 pair4m3; do MWCG_LIB=build_var/$v.so python tools/k1w_sweep.py --config C2 --modes dw,qdw,qtw,tw --variants "MWCG_V=$v" --out gpurun_out/r3c_sweep_c2_$v.json >> gpurun_out/r3c_sweep.log 2>&1; done
python tools/k1w_sweep.py --config C2 --modes dw,qdw,qtw,tw --variants "MWCG_V=default" --out gpurun_out/r3c_sweep_c2_default.json >> gpurun_out/r3c_sweep.log 2>&1
grep -h '"k1_us"' gpurun_out/r3c_sweep.log | cut -c1-150
