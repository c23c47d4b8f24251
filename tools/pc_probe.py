"""CG vs Kronecker-PCG (NEXT-4) at several tolerances: iterations, solve time and distance of the
predicted mean to a tightly converged mean (device generator inputs).

    python tools/pc_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def rel(a, b):
    import numpy as np
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    import numpy as np
    import torch
    from efgp_data import CONFIGS
    from efgp_data import gpu as G
    from paper_2210_10210_b200 import EFGP
    for name, N in [("c3", 1_000_000), ("c3", 10_000_000), ("c5", 10_000_000), ("c2", 1_000_000)]:
        c = CONFIGS[name]
        x, y = G.generate_points(c, 0, N)
        xt = torch.from_numpy(np.random.default_rng(3).uniform(0, 1, (500, 2))).cuda()
        gc = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, cg_tol=c.eps / 1e5, precond="kron")
        gc.fit(x, y)
        conv = gc.predict(xt).cpu().numpy()
        for pc in [None, "kron"]:
            for f in [1, 10, 100]:
                g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, cg_tol=c.eps / f, precond=pc)
                g.fit(x, y)
                inf = g.info()
                print(name, N, pc, f, inf["iters"], round(inf["t_solve_ms"], 2),
                      "%.2e" % rel(g.predict(xt).cpu().numpy(), conv), flush=True)
                g.close()
        gc.close()


if __name__ == "__main__":
    main()
