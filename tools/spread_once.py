"""Run the c5 type-1 spreading (efgp_fit with max_iter=1) a few times; for ncu captures.

    python tools/spread_once.py --N 2e7 [--weights fp32] [--spread sorted] [--fits 2]
"""
import argparse
import os
import sys
import warnings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", default="2e7")
    ap.add_argument("--weights", default="fp64")
    ap.add_argument("--spread", default="sorted")
    ap.add_argument("--fits", type=int, default=2)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--hetero", action="store_true",
                    help="the NEXT-3 one-pass weighted spread (fit_hetero, sigma_n = sigma (0.5 + U))")
    a = ap.parse_args()
    import torch
    from efgp_data import CONFIGS
    from efgp_data import gpu as G
    from paper_2210_10210_b200 import EFGP
    c = CONFIGS[a.config]
    N = int(float(a.N))
    x, y = G.generate_points(c, 0, N)
    torch.cuda.synchronize()
    g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, max_iter=1, spread=a.spread, weights=a.weights)
    sd = None
    if a.hetero:
        gen = torch.Generator(device=x.device)
        gen.manual_seed(1234)
        sd = c.sigma * (0.5 + torch.rand(N, dtype=torch.float64, device=x.device, generator=gen))
    for _ in range(a.fits):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            if sd is None:
                g.fit(x, y)
            else:
                g.fit_hetero(x, y, sd)
        inf = g.info()
        print(f"spread {inf['t_spread_ms']:.3f} ms  {N / inf['t_spread_ms'] * 1e3:.3e} pts/s", flush=True)
    if os.environ.get("EFGP_SORTED_TRACE"):
        import ctypes as C
        import numpy as np
        n = g._lib.efgp_debug_trace(g._h, None, 0)
        buf = np.zeros(n, dtype=np.uint64)
        g._lib.efgp_debug_trace(g._h, buf.ctypes.data_as(C.c_void_p), n)
        G = 148
        nch = (n - G * 2 * 8 - G * 4 * 8) // (G * 4)
        ph = buf[nch * G * 4:nch * G * 4 + G * 2 * 8].reshape(G * 2, 8).astype(np.float64)[:, :7]
        bph = buf[nch * G * 4 + G * 2 * 8:].reshape(G * 4, 8).astype(np.float64)
        bnames = ["chunk hand-off", "TMA wait", "load+classify+rank", "tile scan+reserve", "permutation", "copy-out"]
        nb = bph[:, 6].sum()
        if nb > 0:  # (a build with -DEFGP_SORTED_BTRACE=1, e.g. tools/build_variant.sh)
            print("binner phases (lane 0 of each binner warp, cycles per batch of 256 points, mean over warps):",
                  ", ".join(f"{nm} {bph[:, q].sum() / nb:.0f}" for q, nm in enumerate(bnames)))
        names = ["wait/chunk", "tma wait", "pass1+scan", "pass2", "phaseC", "fold", "flush"]
        tot = ph.sum(axis=1, keepdims=True)
        frac = (ph / tot).mean(axis=0)
        print("accumulator phase shares (thread 0 of each group, clock64):",
              ", ".join(f"{nm} {100 * f:.1f}%" for nm, f in zip(names, frac)))
        buf = buf[:nch * G * 4]
        tr = buf.reshape(-1, G, 4).astype(np.float64)
        t0 = tr[tr > 0].min()
        tr = (tr - t0) / 1e3  # us
        nch = tr.shape[0]
        for k in list(range(min(nch, 6))) + [nch - 1]:
            b, w0, w1, d = tr[k, :, 0], tr[k, :, 1], tr[k, :, 2], tr[k, :, 3]
            print(f"chunk {k:3d}: binned [{b.min():8.1f} .. {b.max():8.1f}]  acc wait from [{w0.min():8.1f} .. {w0.max():8.1f}] "
                  f"start [{w1.min():8.1f} .. {w1.max():8.1f}]  done [{d.min():8.1f} .. {d.max():8.1f}] us")
        waits = (tr[:, :, 2] - tr[:, :, 1]).sum(axis=0)
        work = (tr[:, :, 3] - tr[:, :, 2]).sum(axis=0)
        print(f"acc total wait per CTA: mean {waits.mean():.1f} us, acc work per CTA mean {work.mean():.1f} us (max {work.max():.1f})")
    g.close()


if __name__ == "__main__":
    main()
