set -x
timeout 900 python -m pytest tests/test_gpu_uniform_slices.py tests/test_gpu_parity.py -x -q > gpurun_out/r2m_parity.log 2>&1; tail -3 gpurun_out/r2m_parity.log
python tools/k1w_sweep.py --config C2 --variants 'MWCG_DIA_UNIFORM=1;MWCG_DIA_UNIFORM=0' --out gpurun_out/r2m_sweep_c2.json > gpurun_out/r2m_sweep.log 2>&1
MWCG_LIB=build_var/minb4.so python tools/k1w_sweep.py --config C2 --modes dw,qdw,tw,qtw --variants 'MWCG_DIA_UNIFORM=1;MWCG_DIA_UNIFORM=0' --out gpurun_out/r2m_sweep_c2_minb4.json >> gpurun_out/r2m_sweep.log 2>&1
MWCG_LIB=build_var/minb3.so python tools/k1w_sweep.py --config C2 --modes dw,tw,qtw --variants 'MWCG_DIA_UNIFORM=1' --out gpurun_out/r2m_sweep_c2_minb3.json >> gpurun_out/r2m_sweep.log 2>&1
python tools/k1w_sweep.py --config C4 --modes fp64,dw,qtw --variants 'MWCG_DIA_UNIFORM=1' --out gpurun_out/r2m_sweep_c4.json >> gpurun_out/r2m_sweep.log 2>&1
MWCG_LIB=build_var/minb4.so python tools/k1w_sweep.py --config C4 --modes dw,qtw --variants 'MWCG_DIA_UNIFORM=1' --out gpurun_out/r2m_sweep_c4_minb4.json >> gpurun_out/r2m_sweep.log 2>&1
grep -h '"k1_us"' gpurun_out/r2m_sweep.log | cut -c1-200
