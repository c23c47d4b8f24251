"""c4 (3D, m = 37, 150^3 Toeplitz box) fit at a small N with a few CG iterations, for a launch list
of one FFT-Toeplitz CG iteration.  python tools/c4_cg_probe.py [--iters 6]"""
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from efgp_data import CONFIGS
    from efgp_data import gpu as G
    from paper_2210_10210_b200 import EFGP
    it = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else 6
    c = CONFIGS["c4"]
    x, y = G.generate_points(c, 0, 200_000)
    g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, max_iter=it, graph_iters=2)
    warnings.simplefilter("ignore")
    for _ in range(2):
        g.fit(x, y)
    inf = g.info()
    print(f"c4: iters {inf['iters']} solve {inf['t_solve_ms']:.3f} ms = {1e3 * inf['t_solve_ms'] / inf['iters']:.1f} us/it")


if __name__ == "__main__":
    main()
