python tools/sweep.py run default default:MWCG_PDL=0 --cfg C2 --modes fp64,dw,qdw,tw,qtw --iters 60 --out gpurun_out/sweep17_c2.json 2>&1
python tools/sweep.py run default default:MWCG_PDL=0 --cfg C4 --modes fp64,dw,qtw --iters 60 --out gpurun_out/sweep17_c4.json 2>&1
