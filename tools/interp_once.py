"""Time the type-2 interpolation (K9) at many targets: mu at the N training points (NEXT-1).

    python tools/interp_once.py --q 1e9 [--config c5] [--reps 3]
"""
import argparse
import os
import sys
import warnings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--q", default="1e9")
    ap.add_argument("--config", default="c5")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch
    from efgp_data import CONFIGS
    from efgp_data import gpu as G
    from paper_2210_10210_b200 import EFGP
    c = CONFIGS[a.config]
    q = int(float(a.q))
    x, y = G.generate_points(c, 0, q)
    g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        g.fit(x[:1_000_000], y[:1_000_000])
    mu = torch.empty(q, dtype=torch.float64, device=x.device)
    for r in range(a.reps + 1):
        g.predict(x, out=mu)
        t = g.info()["t_predict_ms"]
        if r:
            print(f"predict q={q:.0e}: {t:.3f} ms  {q / t * 1e3:.3e} targets/s  {24 * q / t / 1e6:.1f} GB/s alg", flush=True)
    g.close()


if __name__ == "__main__":
    main()
