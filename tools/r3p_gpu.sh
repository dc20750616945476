set -x
# the whole GPU suite through the -DMWCG_BOUNDS library (device-side index checks on every matrix walk)
MWCG_LIB=$PWD/paper_2510_13536_b200/libmwcg_cuda_bounds.so timeout 3000 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_bounds.py > gpurun_out/r3p_gputests_bounds.log 2>&1; tail -4 gpurun_out/r3p_gputests_bounds.log
grep -c MWCG_BOUNDS gpurun_out/r3p_gputests_bounds.log
