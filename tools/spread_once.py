"""Run the c5 type-1 spreading (efgp_fit with max_iter=1) a few times; for ncu captures.

    python tools/spread_once.py --N 2e7 [--weights fp32] [--spread sorted] [--fits 2]
"""
import argparse
import os
import sys
import warnings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", default="2e7")
    ap.add_argument("--weights", default="fp64")
    ap.add_argument("--spread", default="sorted")
    ap.add_argument("--fits", type=int, default=2)
    ap.add_argument("--config", default="c5")
    a = ap.parse_args()
    import torch
    from efgp_data import CONFIGS
    from efgp_data import gpu as G
    from paper_2210_10210_b200 import EFGP
    c = CONFIGS[a.config]
    N = int(float(a.N))
    x, y = G.generate_points(c, 0, N)
    torch.cuda.synchronize()
    g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, max_iter=1, spread=a.spread, weights=a.weights)
    for _ in range(a.fits):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            g.fit(x, y)
        inf = g.info()
        print(f"spread {inf['t_spread_ms']:.3f} ms  {N / inf['t_spread_ms'] * 1e3:.3e} pts/s", flush=True)
    g.close()


if __name__ == "__main__":
    main()
