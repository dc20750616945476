for i in 1 2 3; do
MWCG_L2PIN=0 python bench.py --cpu-seconds 1 2> gpurun_out/b54_$i.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nopin', d['value'], d['e2e']['ms_per_step'])"
grep "e2e step" gpurun_out/b54_$i.err
done
