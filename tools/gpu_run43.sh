python tools/sweep.py run default:MWCG_L2PIN=20 default:MWCG_L2PIN=32 default:MWCG_L2PIN=48 default:MWCG_L2PIN=64 --cfg C2 --modes fp64,dw,qdw,tw,qtw --iters 60 --out gpurun_out/sweep30_c2.json 2>&1
python tools/sweep.py run default:MWCG_L2PIN=0 default:MWCG_L2PIN=32 default:MWCG_L2PIN=48 --cfg C4 --modes fp64,dw,qdw,qtw --iters 60 --out gpurun_out/sweep30_c4.json 2>&1
MWCG_L2PIN=40 timeout 600 python tools/c5_probe.py 2>&1 | tail -2
