python tools/sweep.py run default default:MWCG_TMA=0 --cfg C2 --modes fp64,dw,qdw,tw,qtw --iters 100 --out gpurun_out/sweep2_c2.json 2>&1
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
