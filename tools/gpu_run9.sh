python tools/sweep.py run default:MWCG_TMA1=0 selacc:MWCG_TMA1=0 u8b:MWCG_TMA1=0 selacc_u8:MWCG_TMA1=0 --cfg C2 --modes fp64,dw,qdw,tw,qtw --iters 100 --out gpurun_out/sweep4_c2.json 2>&1
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
