python -m pytest tests/test_gpu_parity.py -x -q -k "c1 or small or int16" 2>&1 | tail -2
python tools/sweep.py run default default:MWCG_L2PIN=0 default:MWCG_L2PIN=40 --cfg C2 --modes fp64,dw,qdw,tw,qtw --iters 60 --out gpurun_out/sweep29_c2.json 2>&1
MWCG_L2PIN=0 timeout 600 python tools/c5_probe.py 2>&1 | tail -2
timeout 600 python tools/c5_probe.py 2>&1 | tail -2
