"""K9 A/B in one process (for one ncu capture of both variants): the plain and the bank-aware
2D interpolation kernels on the same q targets.  python tools/interp_ab.py --q 2e8"""
import argparse
import os
import sys
import warnings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--q", default="2e8")
    a = ap.parse_args()
    import torch
    from efgp_data import CONFIGS
    from efgp_data import gpu as G
    from paper_2210_10210_b200 import EFGP
    c = CONFIGS["c5"]
    q = int(float(a.q))
    x, y = G.generate_points(c, 0, q)
    g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        g.fit(x[:1_000_000], y[:1_000_000])
    mu = torch.empty(q, dtype=torch.float64, device=x.device)
    g.predict(x, out=mu)  # warm-up (type-2 grid)
    for plain in (1, 0, 1, 0):
        if plain:
            os.environ["EFGP_INTERP_PLAIN"] = "1"
        else:
            os.environ.pop("EFGP_INTERP_PLAIN", None)
        g.predict(x, out=mu)
        t = g.info()["t_predict_ms"]
        print(f"{'plain' if plain else 'banked'}: {t:.3f} ms  {q / t * 1e3:.3e} targets/s", flush=True)
    g.close()


if __name__ == "__main__":
    main()
