python tools/sweep.py run default up2 up2xp1 up1xp1 default:MWCG_TMA=1 up2xp1:MWCG_TMA=1 --cfg C2 --modes dw,qdw,qtw --iters 60 --out gpurun_out/sweep22_c2.json 2>&1
