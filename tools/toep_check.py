"""Debug: one CG iteration with the direct vs the FFT Toeplitz product (EFGP_TOEP_DIRECT)."""
import os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CHILD = r"""
import sys, warnings, numpy as np, torch
sys.path.insert(0, %r)
from efgp_data import CONFIGS
from efgp_data import gpu as G
from paper_2210_10210_b200 import EFGP
c = CONFIGS[%r]
x, y = G.generate_points(c, 0, 100000)
g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, max_iter=%d)
with warnings.catch_warnings():
    warnings.simplefilter('ignore')
    g.fit(x, y)
b = g.vector('beta')
np.save(%r, b)
print(g.info()['iters'], g.info()['m'])
"""
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for name in ("c5", "c3"):
    for it in (1, 2):
        res = {}
        for dflag in ("0", "1"):
            out = f"/tmp/beta_{name}_{it}_{dflag}.npy"
            env = dict(os.environ, EFGP_TOEP_DIRECT=dflag)
            r = subprocess.run([sys.executable, "-c", CHILD % (root, name, it, out)], env=env, capture_output=True, text=True)
            import numpy as np
            res[dflag] = np.load(out)
            print(name, it, dflag, r.stdout.strip(), r.stderr[-300:])
        a, b = res["0"], res["1"]
        print(name, it, "rel diff", float(np.linalg.norm(a - b) / np.linalg.norm(a)))
