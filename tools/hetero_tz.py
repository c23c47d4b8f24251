"""Time the NEXT-3 TOEPLITZ heteroskedastic fit (reading G11b) on c5-shaped data:
sigma_n = sigma (0.5 + U[0,1)).   python tools/hetero_tz.py [--N 1e9]"""
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from efgp_data import CONFIGS
    from efgp_data import gpu as G
    from paper_2210_10210_b200 import EFGP
    N = int(float(sys.argv[sys.argv.index("--N") + 1])) if "--N" in sys.argv else int(1e9)
    c = CONFIGS["c5"]
    x, y = G.generate_points(c, 0, N)
    gen = torch.Generator(device=x.device)
    gen.manual_seed(1234)
    sd = c.sigma * (0.5 + torch.rand(N, dtype=torch.float64, device=x.device, generator=gen))
    g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, hetero="toeplitz")
    warnings.simplefilter("ignore")
    for _ in range(3):
        g.fit_hetero(x, y, sd)
        inf = g.info()
        print(f"hetero toeplitz N={N:.0e}: type-1 {inf['t_spread_ms']:.2f} ms  setup {inf['t_modes_ms']:.2f} ms  "
              f"solve {inf['t_solve_ms']:.2f} ms ({inf['iters']} it)  fit {inf['t_spread_ms'] + inf['t_modes_ms'] + inf['t_solve_ms']:.2f} ms",
              flush=True)
    g.close()


if __name__ == "__main__":
    main()
