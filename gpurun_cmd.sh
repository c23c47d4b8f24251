timeout 1200 python tools/bench_configs.py --configs c1,c2,c3,c5 --c5-N 1e6 --var-targets 256 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['N'], 'mean cg', d['cg_iters'], 'var', d.get('variance'))
"
