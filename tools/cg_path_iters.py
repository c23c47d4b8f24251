"""CG iteration counts of one config at its BASELINE size on each CG product path (the persistent
direct kernel, the launched fused direct kernels, the FFT product), production and parity mode.

    python tools/cg_path_iters.py --config c3
"""
import argparse
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--paths", default="persist,launched,fft")
    a = ap.parse_args()
    from efgp_data import CONFIGS
    from efgp_data import gpu as G
    from paper_2210_10210_b200 import EFGP
    c = CONFIGS[a.config]
    x, y = G.generate_points(c, 0, c.N)
    env = {"persist": {}, "launched": {"EFGP_CG_PERSIST": "0"},
           "fft": {"EFGP_CG_PERSIST": "0", "EFGP_CG_FUSED": "0"}}
    for path in a.paths.split(","):
        for k in ("EFGP_CG_PERSIST", "EFGP_CG_FUSED"):
            os.environ.pop(k, None)
        os.environ.update(env[path])
        for tol in (c.eps, c.eps / 1000):
            g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, cg_tol=tol, max_iter=20000)
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                g.fit(x, y)
            inf = g.info()
            print(f"{a.config} {path:9s} tol {tol:.0e} iters {inf['iters']} solve {inf['t_solve_ms']:.2f} ms "
                  f"persist_split {inf.get('cg_persist_split')} dft2 {inf.get('cg_dft2')}", flush=True)
            g.close()


if __name__ == "__main__":
    main()
