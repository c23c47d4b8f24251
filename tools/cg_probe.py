import sys, os, warnings
sys.path.insert(0, os.getcwd())
import torch
from efgp_data import CONFIGS
from efgp_data import gpu as G
from paper_2210_10210_b200 import EFGP
c = CONFIGS["c5"]
x, y = G.generate_points(c, 0, 1_000_000)
g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu)
for _ in range(3):
    g.fit(x, y)
inf = g.info()
print("iters", inf["iters"], "solve ms", inf["t_solve_ms"], "us/it", 1e3 * inf["t_solve_ms"] / inf["iters"])
