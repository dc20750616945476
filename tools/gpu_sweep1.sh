python tools/sweep.py run default pipe_m3 u8 pipe_u8_m2 t512_m2 pipe_t512_m1 --cfg C2 --modes dw,qtw,fp64 --iters 100 --out gpurun_out/sweep1_c2.json 2>&1
