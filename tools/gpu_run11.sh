python tools/sweep.py run default default:MWCG_TMA=0 pf1 pf2 pf1_m4 pf1:MWCG_TMA=0 --cfg C2 --modes fp64,dw,qdw,tw,qtw --iters 100 --out gpurun_out/sweep6_c2.json 2>&1
