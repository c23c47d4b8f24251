import sys, os, warnings, numpy as np
sys.path.insert(0, "/root/repo")
from efgp_data import CONFIGS
from efgp_data import gpu as G
from paper_2210_10210_b200 import EFGP
c = CONFIGS["c3"]
for N in (100_000, 1_000_000, 10_000_000):
    x, y = G.generate_points(c, 0, N)
    hs = {}
    for d in ("0", "1"):
        os.environ["EFGP_TOEP_DIRECT"] = d
        g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, max_iter=400)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            g.fit(x, y)
        hs[d] = g.residual_history()
        g.close()
    h0, h1 = hs["0"], hs["1"]
    k = min(len(h0), len(h1))
    idx = [1, 5, 20, 50, 100, 200, k - 1]
    print(N, [(i, "%.3e" % h0[i], "%.3e" % h1[i]) for i in idx if i < k], flush=True)
