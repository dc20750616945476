set -x
for v in m3 m5 m6; do MWCG_LIB=build_var/$v.so timeout 900 python tools/c5_probe.py 16000000 dw,qtw > gpurun_out/r3a_c5_$v.log 2>&1; tail -2 gpurun_out/r3a_c5_$v.log; done
timeout 900 python tools/c5_probe.py 16000000 dw,qtw > gpurun_out/r3a_c5_default.log 2>&1; tail -2 gpurun_out/r3a_c5_default.log
