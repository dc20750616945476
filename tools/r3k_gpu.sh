set -x
for v in nok1pre oldpidx both; do
MWCG_LIB=build_var/$v.so python tools/k1w_sweep.py --config C4 --modes dw,qtw --variants "MWCG_V=$v" --out gpurun_out/r3k_c4_$v.json >> gpurun_out/r3k_sweep.log 2>&1
MWCG_LIB=build_var/$v.so python tools/k1w_sweep.py --config C2 --modes dw,tw,qtw --variants "MWCG_V=$v" --out gpurun_out/r3k_c2_$v.json >> gpurun_out/r3k_sweep.log 2>&1
done
python tools/k1w_sweep.py --config C4 --modes dw,qtw --variants "MWCG_V=current" --out gpurun_out/r3k_c4_cur.json >> gpurun_out/r3k_sweep.log 2>&1
python tools/k1w_sweep.py --config C2 --modes dw,tw,qtw --variants "MWCG_V=current" --out gpurun_out/r3k_c2_cur.json >> gpurun_out/r3k_sweep.log 2>&1
grep -h '"k1_us"' gpurun_out/r3k_sweep.log | cut -c1-150
