"""Persistent direct CG (k_cg_toep2_persist) against the launched fused path (EFGP_CG_PERSIST=0):
same iteration count, weights equal to roundoff, time per iteration; split sweep (EFGP_CG_PSPLIT).

    python tools/cg_persist_check.py [--configs c5,c3]
"""
import argparse
import json
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c5,c3")
    ap.add_argument("--splits", default="1,2,3,4,5,6,8")
    ap.add_argument("--parity", action="store_true", help="cg_tol = eps / 1000 (parity mode, reading G9)")
    a = ap.parse_args()
    import torch
    from efgp_data import CONFIGS
    from efgp_data import gpu as G
    from paper_2210_10210_b200 import EFGP
    for name in a.configs.split(","):
        c = CONFIGS[name]
        N = min(c.N, 10_000_000)
        x, y = G.generate_points(c, 0, N)
        g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, cg_tol=c.eps / 1000 if a.parity else None)

        modes = g.fit_local(x, y)  # one spread: every solve below sees the same v and F^*y

        def run(env):
            for k in ("EFGP_CG_PERSIST", "EFGP_CG_PSPLIT"):
                os.environ.pop(k, None)
            os.environ.update(env)
            rows = []
            for _ in range(3):
                with warnings.catch_warnings():
                    warnings.simplefilter("ignore")
                    g.fit_solve(modes, N)
                rows.append(g.info())
            inf = min(rows, key=lambda i: i["t_solve_ms"])
            return inf, torch.from_numpy(g.weights().copy())

        base, b0 = run({"EFGP_CG_PERSIST": "0"})
        # sensitivity of the launched path itself: modes perturbed at 1e-13 relative
        m0 = modes.clone()
        gen = torch.Generator(device=modes.device)
        gen.manual_seed(5)
        modes.mul_(1 + 1e-13 * torch.randn(modes.shape, dtype=modes.dtype, device=modes.device, generator=gen))
        pert, bp = run({"EFGP_CG_PERSIST": "0"})
        modes.copy_(m0)
        print(json.dumps({"config": name, "path": "launched, modes x (1 + 1e-13 n)", "iters": pert["iters"],
                          "beta_maxrel_vs_launched": float((bp - b0).abs().max() / b0.abs().max())}), flush=True)
        print(json.dumps({"config": name, "N": N, "path": "launched", "iters": base["iters"],
                          "solve_ms": base["t_solve_ms"], "us_per_it": 1e3 * base["t_solve_ms"] / base["iters"]}), flush=True)
        for sp in a.splits.split(",") + a.splits.split(",")[-1:]:
            inf, b = run({"EFGP_CG_PSPLIT": sp})
            d = float((b - b0).abs().max() / b0.abs().max())
            print(json.dumps({"config": name, "N": N, "path": "persistent", "split_req": int(sp),
                              "split": inf.get("cg_persist_split"), "iters": inf["iters"], "solve_ms": inf["t_solve_ms"],
                              "us_per_it": 1e3 * inf["t_solve_ms"] / inf["iters"], "beta_maxrel_vs_launched": d}), flush=True)
        g.close()


if __name__ == "__main__":
    main()
