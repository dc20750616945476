python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/sweep.py run head default default:MWCG_TMA=1 default:MWCG_TMA=0 --cfg C2 --modes fp64,dw,qdw,tw,qtw --iters 100 --out gpurun_out/sweep9_c2.json 2>&1
