"""Pretty-print a sweep log (tools/sweep.py run output)."""
import json
import sys

for l in open(sys.argv[1]):
    if l.startswith('['):
        continue
    nm, _, js = l.partition(' ')
    try:
        d = json.loads(js)
    except Exception:
        print(l[:300].rstrip())
        continue
    if 'error' in d:
        print(nm, 'ERROR', d['error'][-300:])
        continue
    print(nm.ljust(24), '  '.join(
        f"{m}:{v['stages_us'].get('spmv', 0):.1f}/{v['stages_us'].get('axpy', 0):.1f}/"
        f"{v['stages_us'].get('scal_add', 0):.1f}|{v['graph_us_per_iter']:.1f}"
        for m, v in d.items() if m != 'gen_s'))
