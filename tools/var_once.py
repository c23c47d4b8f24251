"""Posterior variance at q targets for one config (launch lists / timing).

    python tools/var_once.py [--config c5] [--N 1e6] [--q 64]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--N", default="1e6")
    ap.add_argument("--q", type=int, default=64)
    a = ap.parse_args()
    from efgp_data import CONFIGS
    from efgp_data import gpu as G
    from paper_2210_10210_b200 import EFGP
    c = CONFIGS[a.config]
    x, y = G.generate_points(c, 0, int(float(a.N)))
    xt = G.generate_targets(c, 0, a.q)
    g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu)
    g.fit(x, y)
    g.predict_var(xt)
    inf = g.info()
    print(f"{a.config} N={a.N} q={a.q}: {inf['t_var_ms']:.2f} ms, {inf['var_iters_max']} iterations, "
          f"batch {inf['var_batch']}, {inf['t_var_ms'] / max(inf['var_iters_max'], 1) * 1e3:.1f} us/iteration")


if __name__ == "__main__":
    main()
