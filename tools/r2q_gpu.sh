set -x
timeout 600 python -m pytest tests/test_gpu_colblocks.py tests/test_gpu_uniform_slices.py -x -q > gpurun_out/r2q_tests.log 2>&1; tail -3 gpurun_out/r2q_tests.log
timeout 900 python tools/c5_probe.py 16000000 dw,qtw,fp64 > gpurun_out/r2q_c5_default.log 2>&1; tail -3 gpurun_out/r2q_c5_default.log
for v in ef u6 u8; do MWCG_LIB=build_var/$v.so timeout 900 python tools/c5_probe.py 16000000 dw,qtw > gpurun_out/r2q_c5_$v.log 2>&1; tail -2 gpurun_out/r2q_c5_$v.log; done
MWCG_COLBLOCK=0 timeout 900 python tools/c5_probe.py 16000000 dw > gpurun_out/r2q_c5_noblock.log 2>&1; tail -1 gpurun_out/r2q_c5_noblock.log
python tools/k1w_sweep.py --config C2 --variants 'MWCG_X=na' --modes fp64,dw,qtw --out gpurun_out/r2q_sweep_c2.json > gpurun_out/r2q_sweep.log 2>&1
python tools/k1w_sweep.py --config C4 --variants 'MWCG_X=na' --modes fp64,dw,qtw --out gpurun_out/r2q_sweep_c4.json >> gpurun_out/r2q_sweep.log 2>&1
python tools/k1w_sweep.py --config C3 --variants 'MWCG_X=na' --modes fp64,dw,qtw --out gpurun_out/r2q_sweep_c3.json >> gpurun_out/r2q_sweep.log 2>&1
MWCG_LIB=build_var/ef.so python tools/k1w_sweep.py --config C4 --variants 'MWCG_X=ef' --modes fp64,dw,qtw --out gpurun_out/r2q_sweep_c4_ef.json >> gpurun_out/r2q_sweep.log 2>&1
MWCG_LIB=build_var/ef.so python tools/k1w_sweep.py --config C3 --variants 'MWCG_X=ef' --modes fp64,dw,qtw --out gpurun_out/r2q_sweep_c3_ef.json >> gpurun_out/r2q_sweep.log 2>&1
grep -h '"k1_us"' gpurun_out/r2q_sweep.log | cut -c1-200
