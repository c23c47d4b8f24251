"""K9 A/B in one process (for one ncu capture of every variant): the plain, bank-aware and
shifted-copy (C = 2, C = 4) 2D interpolation kernels on the same q targets, checked bitwise
against the plain kernel.  python tools/interp_ab.py --q 2e8 [--reps 2]"""
import argparse
import os
import sys
import warnings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

VARIANTS = ("plain", "banked", "c2", "c4", "c4r")


def set_variant(v):
    os.environ.pop("EFGP_INTERP_PLAIN", None)
    os.environ.pop("EFGP_K9", None)
    if v == "plain":
        os.environ["EFGP_INTERP_PLAIN"] = "1"
    else:
        os.environ["EFGP_K9"] = v


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--q", default="2e8")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--variants", default=",".join(VARIANTS))
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
    ref = torch.empty_like(mu)
    set_variant("plain")
    g.predict(x, out=ref)  # warm-up (type-2 grid) and the bitwise reference
    vs = a.variants.split(",")
    for _ in range(a.reps):
        for v in vs:
            set_variant(v)
            mu.fill_(0.0)
            g.predict(x, out=mu)
            t = g.info()["t_predict_ms"]
            same = bool(torch.equal(mu, ref))
            print(f"{v}: {t:.3f} ms  {q / t * 1e3:.3e} targets/s  bitwise={same}", flush=True)
    g.close()


if __name__ == "__main__":
    main()
