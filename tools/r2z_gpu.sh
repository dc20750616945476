set -x
timeout 600 python -m pytest tests/test_gpu_uniform_slices.py tests/test_gpu_parity.py -x -q -k "slice or layout or int16 or uniform" > gpurun_out/r2z_tests.log 2>&1; tail -2 gpurun_out/r2z_tests.log
E2E_STEPS=4 timeout 600 python tools/e2e_probe2.py > gpurun_out/r2z_e2e.log 2>&1; tail -2 gpurun_out/r2z_e2e.log
for v in u2m4 u2m5 u3m3 u2m3 u4m4; do MWCG_LIB=build_var/$v.so python tools/k1w_sweep.py --config C2 --modes tw,qtw --variants "MWCG_V=$v" --out gpurun_out/r2z_sweep_c2_$v.json >> gpurun_out/r2z_sweep.log 2>&1; done
python tools/k1w_sweep.py --config C2 --modes tw,qtw --variants "MWCG_V=default" --out gpurun_out/r2z_sweep_c2_default.json >> gpurun_out/r2z_sweep.log 2>&1
grep -h '"k1_us"' gpurun_out/r2z_sweep.log | cut -c1-170
