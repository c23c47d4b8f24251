import sys, os, warnings
sys.path.insert(0, os.getcwd())
from efgp_data import CONFIGS
from efgp_data import gpu as G
from paper_2210_10210_b200 import EFGP
c = CONFIGS["c4"]
x, y = G.generate_points(c, 0, c.N)
for tol in (c.eps, c.eps / 1000):
    g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, cg_tol=tol)
    warnings.simplefilter("ignore")
    g.fit(x, y)
    inf = g.info()
    h = g.residual_history()
    print("tol", tol, "iters", inf["iters"], "solve ms", inf["t_solve_ms"], "hist tail", h[-3:], flush=True)
    g.close()
