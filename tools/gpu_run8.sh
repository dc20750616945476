python tools/sweep.py run default default:MWCG_TMA=0 default:MWCG_TMA1=0 default:MWCG_TMA=0,MWCG_TMA1=0 --cfg C2 --modes fp64,dw,qtw --iters 100 --out gpurun_out/sweep3_c2.json 2>&1
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
