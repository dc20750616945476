for i in 1 2 3; do
python bench.py --cpu-seconds 1 2> gpurun_out/b53_$i.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('per', d['value'], d['e2e']['ms_per_step'])"
grep "e2e step" gpurun_out/b53_$i.err
done
