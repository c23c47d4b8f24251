"""One c3 fit with the NEXT-4 preconditioner (for launch lists): python tools/pcg_once.py --N 1e6"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", default="1e6")
    ap.add_argument("--config", default="c3")
    ap.add_argument("--precond", default="kron")
    a = ap.parse_args()
    from efgp_data import CONFIGS
    from efgp_data import gpu as G
    from paper_2210_10210_b200 import EFGP
    c = CONFIGS[a.config]
    x, y = G.generate_points(c, 0, int(float(a.N)))
    g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, precond=None if a.precond == "none" else a.precond)
    g.fit(x, y)  # first fit: cuSOLVER handle creation, graph capture
    g.fit(x, y)
    inf = g.info()
    print(f"iters {inf['iters']} solve {inf['t_solve_ms']:.2f} ms  {inf['t_solve_ms'] / max(inf['iters'], 1) * 1e3:.1f} us/iter")


if __name__ == "__main__":
    main()
