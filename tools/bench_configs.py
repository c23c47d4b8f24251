"""Per-config measurement of the whole path on one GPU (every BASELINE config, production options):
fit (spread + FFT/deconvolution + Toeplitz/CG) and predict device times, CG iterations, spread
throughput and its HBM fraction.  One JSON line per config.

    python tools/bench_configs.py [--configs c1,c2,c3,c4,c5] [--reps 3] [--c5-N 1e9]
Inputs are device-generated (efgp_data); c5 at its full N = 1e9 unless --c5-N is given.
"""
import argparse
import json
import os
import statistics
import sys
import warnings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--c5-N", type=float, default=None)
    ap.add_argument("--var-targets", type=int, default=0, help="also time the posterior variance (NEXT-2)")
    ap.add_argument("--precond", default="none", choices=["none", "kron", "auto", "jacobi"], help="NEXT-4 preconditioner")
    ap.add_argument("--hetero", action="store_true", help="also time NEXT-3 (fit_hetero, sigma_n = sigma (0.5 + U))")
    a = ap.parse_args()
    import torch
    from efgp_data import CONFIGS
    from efgp_data import gpu as G
    from paper_2210_10210_b200 import EFGP
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f)["hbm_gbs"])
    for name in a.configs.split(","):
        c = CONFIGS[name]
        N = int(a.c5_N) if (name == "c5" and a.c5_N) else c.N
        x, y = G.generate_points(c, 0, N)
        xt = G.generate_targets(c, 0, c.q)
        mu = torch.empty(c.q, dtype=torch.float64, device=x.device)
        g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, precond=None if a.precond == "none" else a.precond)
        rows = []
        for r in range(a.reps + 1):
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                g.fit(x, y)
            g.predict(xt, out=mu)
            inf = g.info()
            if r:
                rows.append(inf)
        med = lambda k: statistics.median(float(i[k]) for i in rows)
        sp = med("t_spread_ms")
        fit_ms = sp + med("t_modes_ms") + med("t_solve_ms")
        out = {"config": name, "precond": a.precond, "N": N, "q": c.q, "d": c.d, "m": rows[0]["m"], "M": rows[0]["M"], "w": rows[0]["w"],
               "spread": rows[0]["spread_method"], "cg_iters": med("iters"),
               "ms": {"spread": sp, "fft_deconv": med("t_modes_ms"), "toeplitz_cg": med("t_solve_ms"),
                      "predict": med("t_predict_ms")},
               "fit_predict_points_per_s": N / ((fit_ms + med("t_predict_ms")) / 1e3),
               "cg_us_per_iteration": 1e3 * med("t_solve_ms") / max(1.0, med("iters")),
               "spread_points_per_s": N / (sp / 1e3),
               "spread_hbm_frac": N * 8 * (c.d + 1) / (sp / 1e3) / 1e9 / peak}
        if a.var_targets:
            qv = min(a.var_targets, c.q)
            var = torch.empty(qv, dtype=torch.float64, device=x.device)
            g.predict_var(xt[:qv], out=var)
            g.predict_var(xt[:qv], out=var)
            iv = g.info()
            out["variance"] = {"q": qv, "ms": iv["t_var_ms"], "targets_per_s": qv / (iv["t_var_ms"] / 1e3),
                               "cg_iters_max": iv["var_iters_max"]}
        if a.hetero:
            gen = torch.Generator(device=x.device)
            gen.manual_seed(99)
            sd = c.sigma * (0.5 + torch.rand(N, dtype=torch.float64, device=x.device, generator=gen))
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                g.fit_hetero(x, y, sd)
                g.fit_hetero(x, y, sd)
            ih = g.info()
            out["hetero"] = {"solver": {0: "nufft-unfused", 1: "nufft-sorted", 2: "toeplitz"}[ih["hetero_sorted"]],
                             "iters": ih["iters"], "ms": ih["t_spread_ms"] + ih["t_modes_ms"] + ih["t_solve_ms"],
                             "type1_ms": ih["t_spread_ms"], "solve_ms": ih["t_solve_ms"]}
            del sd
        print(json.dumps(out), flush=True)
        g.close()
        del x, y, xt, mu
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
