set -x
python tools/sweep.py run default:MWCG_K1P=0 m4u4:MWCG_K1P=0 m4u6:MWCG_K1P=0 m4u8:MWCG_K1P=0 m3u8:MWCG_K1P=0 --cfg C2 --modes fp64,dw,qdw,qtw --iters 200 --out gpurun_out/r2h_sweep_c2.json > gpurun_out/r2h_sweep.log 2>&1
python tools/sweep.py run default:MWCG_K1P=0 m4u4:MWCG_K1P=0 m4u6:MWCG_K1P=0 m4u8:MWCG_K1P=0 m3u8:MWCG_K1P=0 --cfg C4 --modes dw,qtw --iters 200 --out gpurun_out/r2h_sweep_c4.json >> gpurun_out/r2h_sweep.log 2>&1
tail -3 gpurun_out/r2h_sweep.log
