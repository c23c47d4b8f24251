"""Dump the GPU's type-1 outputs (Toeplitz vector v on J_2m, right-hand side b on J_m, full layout) of
one config at its BASELINE size, for host-side CG experiments against the oracle.

    python tools/dump_type1.py --config c3 --out gpurun_out/c3_vb.npz [--runs 2]
"""
import argparse
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--out", required=True)
    ap.add_argument("--runs", type=int, default=2)
    a = ap.parse_args()
    import numpy as np
    from efgp_data import CONFIGS
    from efgp_data import gpu as G
    from paper_2210_10210_b200 import EFGP, half_to_full
    c = CONFIGS[a.config]
    x, y = G.generate_points(c, 0, c.N)
    out = {}
    for r in range(a.runs):
        g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, max_iter=1)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            g.fit(x, y)
        inf = g.info()
        m, d = inf["m"], inf["d"]
        out[f"v{r}"] = half_to_full(g.vector("v"), m, d, K=2 * m)
        out[f"b{r}"] = half_to_full(g.vector("rhs"), m, d)
        g.close()
    np.savez(a.out, **out)
    print("saved", a.out, {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
