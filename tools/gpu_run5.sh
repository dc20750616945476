python -m pytest tests -m gpu -x -q 2>&1 | tail -3
MWCG_UNROLL=8 MODES=fp64,dw,qdw,tw,qtw python quick_c2.py 2>&1 | grep -v gen
