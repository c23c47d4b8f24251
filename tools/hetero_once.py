"""Time the NEXT-3 heteroskedastic fit's per-iteration product (fixed CG iteration count).

    python tools/hetero_once.py --N 2e8 [--iters 10] [--config c5] [--fits 2]
Prints the one-time sort time and ms per CG iteration (each = one type-2 + type-1 pass over N).
"""
import argparse
import os
import sys
import warnings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", default="2e8")
    ap.add_argument("--iters", type=int, default=10)
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
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)
    sd = c.sigma * (0.5 + torch.rand(N, dtype=torch.float64, device="cuda", generator=gen))
    torch.cuda.synchronize()
    g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, max_iter=a.iters, cg_tol=1e-15)
    for _ in range(a.fits):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            g.fit_hetero(x, y, sd)
        inf = g.info()
        it = max(inf["iters"], 1)
        print(f"sorted={inf['hetero_sorted']} rhs {inf['t_spread_ms']:.2f} ms  sort {inf['t_modes_ms']:.2f} ms  "
              f"{inf['t_solve_ms'] / it:.3f} ms/iter  {N / (inf['t_solve_ms'] / it) * 1e3:.3e} pts/s/iter", flush=True)


if __name__ == "__main__":
    main()
