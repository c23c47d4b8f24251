"""Posterior-variance CG iterations and time with and without the NEXT-4 preconditioner (SE configs).

    python tools/var_probe.py [--config c3] [--Ns 3e3,1e5,1e6,1e7] [--q 64]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--Ns", default="3e3,1e5,1e6,1e7")
    ap.add_argument("--q", type=int, default=64)
    a = ap.parse_args()
    import torch
    from efgp_data import CONFIGS
    from efgp_data import gpu as G
    from paper_2210_10210_b200 import EFGP
    c = CONFIGS[a.config]
    for Ns in a.Ns.split(","):
        N = int(float(Ns))
        x, y = G.generate_points(c, 0, N)
        xt = G.generate_targets(c, 0, a.q)
        for pc in (None, "kron"):
            g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, precond=pc)
            g.fit(x, y)
            v = g.predict_var(xt)
            v = g.predict_var(xt)
            inf = g.info()
            print(f"{a.config} N={N} precond={pc} var_iters_max={inf['var_iters_max']} t_var={inf['t_var_ms']:.2f} ms "
                  f"mean={float(v.mean()):.6e}", flush=True)
            g.close()
        del x, y
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
