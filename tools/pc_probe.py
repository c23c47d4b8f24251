import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
from _util import CONFIGS, rel, dev, model
from efgp_data import gpu as G
for name, N in [("c3", 1_000_000), ("c3", 10_000_000), ("c5", 10_000_000), ("c2", 1_000_000)]:
    c = CONFIGS[name]
    x, y = G.generate_points(c, 0, N)
    xt = dev(np.random.default_rng(3).uniform(0, 1, (500, 2)))
    gc = model(c, cg_tol=c.eps / 1e5, precond="kron"); gc.fit(x, y); conv = gc.predict(xt).cpu().numpy()
    for pc in [None, "kron"]:
        for f in [1, 10, 100]:
            g = model(c, cg_tol=c.eps / f, precond=pc); g.fit(x, y)
            inf = g.info()
            print(name, N, pc, f, inf["iters"], round(inf["t_solve_ms"], 2), "%.2e" % rel(g.predict(xt).cpu().numpy(), conv), flush=True)
            g.close()
    gc.close()
