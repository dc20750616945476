python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for u in 1 2 4 8; do echo "UNROLL=$u"; MWCG_UNROLL=$u MODES=fp64,dw,qtw python quick_c2.py 2>&1 | grep -v stages | grep -v gen; done
