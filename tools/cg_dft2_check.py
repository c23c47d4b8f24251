"""Persistent DFT CG (2D, m beyond the direct product: c2) against the padded real-FFT CG
(EFGP_TOEP_DFT2=0) on the SAME v and F^*y (one spread, two solves): iterations, beta, time per
iteration.  python tools/cg_dft2_check.py [--parity]"""
import argparse
import json
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--parity", action="store_true")
    ap.add_argument("--config", default="c2")
    a = ap.parse_args()
    import torch
    from efgp_data import CONFIGS
    from efgp_data import gpu as G
    from paper_2210_10210_b200 import EFGP
    c = CONFIGS[a.config]
    x, y = G.generate_points(c, 0, c.N)
    g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, cg_tol=c.eps / 1000 if a.parity else None)
    modes = g.fit_local(x, y)
    out = {}
    for name, env in (("fft", "0"), ("dft2", "1"), ("dft2_again", "1")):
        os.environ["EFGP_TOEP_DFT2"] = env
        ts = []
        for _ in range(3):
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                g.fit_solve(modes, c.N)
            ts.append(g.info()["t_solve_ms"])
        inf = g.info()
        out[name] = (g.weights(), inf)
        b0 = out["fft"][0]
        d = float(abs(out[name][0] - b0).max() / abs(b0).max())
        print(json.dumps({"config": a.config, "path": name, "parity": a.parity, "cg_dft2": inf["cg_dft2"], "iters": inf["iters"],
                          "solve_ms": min(ts), "us_per_it": 1e3 * min(ts) / max(1, inf["iters"]),
                          "beta_maxrel_vs_fft": d}), flush=True)
    os.environ.pop("EFGP_TOEP_DFT2")


if __name__ == "__main__":
    main()
