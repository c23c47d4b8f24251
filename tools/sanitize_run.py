"""Small-shape run of every kernel family of the library, for compute-sanitizer (memcheck, racecheck,
synccheck; one tool per process).  SURVEY §4.2-8 / §5: the SORTED spreader relies on cross-CTA
spin-waits and acquire/release counters, CELLSORT on shared-memory counting sorts, CG/PCG and the
variance on CUDA graphs.  Sizes are small so the sanitizers finish in minutes.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys
import warnings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from efgp_data import CONFIGS, generate
    from paper_2210_10210_b200 import EFGP
    warnings.simplefilter("ignore")
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    for name, N, kw in (("c5", 60_000, {}), ("c2", 20_000, dict(m=20)), ("c3", 30_000, {}), ("c4", 8_000, dict(m=6)),
                        ("c1", 5_000, {})):
        c = CONFIGS[name]
        x, y, xt = generate(c, N=N, q=1000)
        if "m" in kw:  # the library's own h with a smaller m (keeps the CG short)
            g0 = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu)
            kw = dict(h=g0.info()["h"], m=kw["m"])
            g0.close()
        for precond in (None, "auto"):
            g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, precond=precond, **kw)
            g.fit(t(x), t(y))
            mu = g.predict(t(xt))
            var = g.predict_var(t(xt[:16]))
            inf = g.info()
            print(f"{name} precond={precond}: spread={inf['spread_method']} iters={inf['iters']} "
                  f"mu[0]={float(mu[0]):.4f} var[0]={float(var[0]):.3e}", flush=True)
            g.close()
        if c.d <= 2:
            sd = c.sigma * (0.5 + np.random.default_rng(1).uniform(size=N))
            for meth in ("toeplitz", "nufft"):
                g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, hetero=meth, **kw)
                g.fit_hetero(t(x), t(y), t(sd))
                print(f"{name} hetero={meth}: iters={g.info()['iters']} mu[0]={float(g.predict(t(xt))[0]):.4f}",
                      flush=True)
                g.close()
    # SORTED with several chunks and a list overflow (concentrated cloud), K9 bank-aware order
    os.environ["EFGP_SORTED_CHUNK"] = "16384"
    c = CONFIGS["c5"]
    rng = np.random.default_rng(7)
    x = np.concatenate([0.3 + 0.004 * rng.uniform(size=(30_000, 2)), rng.uniform(size=(20_000, 2))])
    y = rng.normal(size=len(x))
    g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, max_iter=2, spread="sorted")
    g.fit(t(x), t(y))
    xq = rng.uniform(size=(148 * 512 + 333, 2))
    mu = g.predict(t(xq))
    print(f"sorted chunks+overflow: spread={g.info()['spread_method']} mu finite={bool(torch.isfinite(mu).all())}")
    g.close()
    torch.cuda.synchronize()
    print("sanitize_run: done")


if __name__ == "__main__":
    main()
