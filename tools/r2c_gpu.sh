set -x
python -m pytest tests/test_gpu_k1w.py -x -q > gpurun_out/r2c_k1w.log 2>&1; tail -3 gpurun_out/r2c_k1w.log
python tools/k1w_sweep.py --config C2 --variants 'MWCG_K1W=0;MWCG_K1W=1,MWCG_K1W_NC=512;MWCG_K1W=1,MWCG_K1W_NC=512,MWCG_K1W_R=1024;MWCG_K1W=1,MWCG_K1W_NC=256;MWCG_K1W=1,MWCG_K1W_NC=256,MWCG_K1W_R=512' --out gpurun_out/r2c_sweep_c2.json > gpurun_out/r2c_sweep.log 2>&1
python tools/k1w_sweep.py --config C4 --modes dw,qtw --variants 'MWCG_K1W=0;MWCG_K1W=1,MWCG_K1W_NC=512;MWCG_K1W=1,MWCG_K1W_NC=256' --out gpurun_out/r2c_sweep_c4.json >> gpurun_out/r2c_sweep.log 2>&1
python -m pytest tests -m gpu -q -x > gpurun_out/r2c_gputests.log 2>&1; tail -3 gpurun_out/r2c_gputests.log
