python tools/sweep.py run default default:MWCG_PDL=0 --cfg C2 --modes fp64,dw,qdw,tw,qtw --iters 60 --out gpurun_out/sweep16_c2.json 2>&1
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
