"""Time the type-1 spreading of config c5 for several SORTED geometries (env overrides).

    python tools/spread_sweep.py --N 2e8 [--runs 3]
Each variant runs in a fresh subprocess (the geometry is fixed at efgp_setup).
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, os, sys, torch
sys.path.insert(0, %r)
from efgp_data import CONFIGS
from efgp_data import gpu as G
from paper_2210_10210_b200 import EFGP
c = CONFIGS['c5']
N = int(float(%r)); runs = int(%r); method = %r; weights = %r
x, y = G.generate_points(c, 0, N)
torch.cuda.synchronize()
g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, max_iter=1, spread=method, weights=weights)
ts = []
for r in range(runs + 1):
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter('ignore')
        g.fit(x, y)
    ts.append(g.info()['t_spread_ms'])
inf = g.info()
print(json.dumps({'method': method, 'weights': weights, 'T1': inf['sorted_t1'], 'T2': inf['sorted_t2'],
                  'R': inf['sorted_round'], 'chunk': inf['sorted_chunk'],
                  'spread_ms': min(ts[1:]), 'pts_per_s': N / (min(ts[1:]) / 1e3)}))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", default="2e8")
    ap.add_argument("--runs", default="3")
    ap.add_argument("--variants", default="default")
    a = ap.parse_args()
    variants = [{}]
    if a.variants != "default":
        variants = json.loads(a.variants)
    for v in variants:
        env = dict(os.environ)
        method = v.pop("method", "sorted")
        weights = v.pop("weights", "fp64")
        env.update({k: str(val) for k, val in v.items()})
        code = CHILD % (ROOT, a.N, a.runs, method, weights)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-500:]
        print(json.dumps(v), line, flush=True)


if __name__ == "__main__":
    main()
