set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_uniform_slices.py tests/test_gpu_colblocks.py tests/test_gpu_bounds.py tests/test_gpu_dist.py tests/test_gpu_nccl.py tests/test_cli.py -m gpu -x -q > gpurun_out/r2t_tests.log 2>&1; tail -5 gpurun_out/r2t_tests.log
python tools/k1w_sweep.py --config C2 --variants 'MWCG_X=dense' --out gpurun_out/r2t_sweep_c2.json > gpurun_out/r2t_sweep.log 2>&1
MWCG_LIB=build_var/shuf.so python tools/k1w_sweep.py --config C2 --variants 'MWCG_X=shuf' --out gpurun_out/r2t_sweep_c2_shuf.json >> gpurun_out/r2t_sweep.log 2>&1
python tools/k1w_sweep.py --config C4 --modes dw,qtw --variants 'MWCG_X=dense' --out gpurun_out/r2t_sweep_c4.json >> gpurun_out/r2t_sweep.log 2>&1
MWCG_LIB=build_var/shuf.so python tools/k1w_sweep.py --config C4 --modes dw,qtw --variants 'MWCG_X=shuf' --out gpurun_out/r2t_sweep_c4_shuf.json >> gpurun_out/r2t_sweep.log 2>&1
python tools/k1w_sweep.py --config C1 --modes dw,tw --variants 'MWCG_X=dense' --out gpurun_out/r2t_sweep_c1.json >> gpurun_out/r2t_sweep.log 2>&1
MWCG_LIB=build_var/shuf.so python tools/k1w_sweep.py --config C1 --modes dw,tw --variants 'MWCG_X=shuf' --out gpurun_out/r2t_sweep_c1_shuf.json >> gpurun_out/r2t_sweep.log 2>&1
grep -h '"k1_us"' gpurun_out/r2t_sweep.log | cut -c1-180
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --partitioned --steps 2 --warmup 1 > gpurun_out/r2t_partitioned.json 2> gpurun_out/r2t_partitioned.err; tail -c 1500 gpurun_out/r2t_partitioned.json; tail -3 gpurun_out/r2t_partitioned.err
