"""Partial-transform Toeplitz product (cg.cu, toeplitz_pt) against the padded real-FFT product on
the same fit: beta after a fixed number of CG iterations, and the per-iteration solve time of both.

    python tools/pt_check.py [--configs c2,c4] [--iters 40]
"""
import argparse
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2,c4")
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--N", type=float, default=2e5)
    ap.add_argument("--G", default="")
    a = ap.parse_args()
    import numpy as np
    from efgp_data import CONFIGS
    from efgp_data import gpu as G
    from paper_2210_10210_b200 import EFGP
    warnings.simplefilter("ignore")
    for name in a.configs.split(","):
        c = CONFIGS[name]
        x, y = G.generate_points(c, 0, int(a.N))
        out = {}
        for mode, env in (("fft", {"EFGP_TOEP_PT": "0"}), ("pt", {"EFGP_TOEP_PT": "1"})) + tuple(
                (f"pt_G{g}", {"EFGP_TOEP_PT": "1", "EFGP_PT_G": g}) for g in a.G.split(",") if g):
            os.environ.update(env)
            g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, max_iter=a.iters, cg_tol=1e-30)
            ts = []
            try:
                for _ in range(3):
                    g.fit(x, y)
                    ts.append(g.info()["t_solve_ms"])
            except Exception as ex:  # report and go on with the other variants
                print(f"{name} {mode}: {ex}", flush=True)
                g.close()
                os.environ.pop("EFGP_PT_G", None)
                os.environ.pop("EFGP_PT_CONV", None)
                continue
            inf = g.info()
            out[mode] = (g.weights(), inf["iters"], min(ts))
            g.close()
            os.environ.pop("EFGP_PT_G", None)
            os.environ.pop("EFGP_PT_CONV", None)
        ref = out["fft"][0]
        for mode, (w, it, t) in out.items():
            err = float(np.linalg.norm(w - ref) / np.linalg.norm(ref))
            print(f"{name} {mode:8s} iters {it} solve {t:.3f} ms = {1e3 * t / it:.1f} us/it  rel diff vs fft {err:.2e}")


if __name__ == "__main__":
    main()
