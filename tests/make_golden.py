#!/usr/bin/env python
"""Golden dumps of the oracle at the BASELINE configs' own sizes.

Test infrastructure (lives in tests/, the only place besides smoke() and bench.py's cpu_baseline that
may run the oracle): imports only ``oracle`` and ``efgp_data`` (never the product package).  For one
config it runs Algorithm a1 exactly as the oracle states it:

  * the type-1 sums v (eq 88) and F^*y (eq rhs) over ALL N points, split into index shards that
    worker processes sum independently (the sum over n is linear; only the order of additions
    changes), each shard regenerated from the seeded Philox recipe (efgp_data);
  * CG twice: parity mode (cg_tol = eps/1000, reading G9) and production mode
    (cg_tol = eps), both with the default cap, recording ||r_k||/||b||;
    the Toeplitz product is the direct one (dense T when M <= 10^4) or, for c4 only, the host FFT
    of reading G11;
  * mu at the config's targets (eq muws) for both solutions.

Output: tests/golden/full_<cfg>.npz (arrays) + full_<cfg>.json (metadata: sizes, (h, m), reading,
iteration counts, per-stage oracle seconds, host cores/model, sha256 of oracle/efgp_oracle.py and of
the data recipe).  The GPU test tests/test_gpu_golden.py regenerates the same inputs on the device
and gates on these.

  python tests/make_golden.py c2 [--N 1e6] [--workers 8]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import math
import multiprocessing as mp
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))  # tests/ -> repo root
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from efgp_data import CONFIGS, observations, points, targets  # noqa: E402

DEFAULT_N = {"c5": 100_000_000}  # c5's 1e9 would take ~4 h of host time; 1e8 keeps the same path


def sha256(path):
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def oracle_hash():
    return sha256(os.path.join(ROOT, "oracle", "efgp_oracle.py"))


def data_hash():
    return hashlib.sha256(b"".join(open(os.path.join(ROOT, "efgp_data", f), "rb").read()
                                   for f in ("configs.py", "philox.py"))).hexdigest()


def host_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def _shard(args):
    """Partial sums of v and F^*y over records [a, b) (eq 88, eq rhs), single-threaded BLAS."""
    name, a, b, h, m = args
    from threadpoolctl import threadpool_limits
    cfg = CONFIGS[name]
    with threadpool_limits(1):
        x = points(cfg, a, b)
        y = observations(cfg, x, a)
        v = O.toeplitz_vector(x, h, m)
        fy = O.rhs_Fy(x, y, h, m)
    return v, fy


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--N", type=float, default=None)
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    ap.add_argument("--shard", type=int, default=None)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden"))
    ap.add_argument("--perturb", type=int, default=6,
                    help="CG reruns on v, b perturbed at the NUFFT tolerance (reading G10b), per mode")
    ap.add_argument("--cache", default=os.path.join(ROOT, ".golden_cache"),
                    help="full v and F^*y of each run (not tracked), reused with --reuse")
    ap.add_argument("--reuse", action="store_true", help="take v and F^*y (and finished CG runs) from the cache")
    ap.add_argument("--perturb-modes", default=None,
                    help="CG modes rerun under perturbation (default: parity,production; c4: production only, "
                         "its parity-mode CG alone takes ~30 min of host FFTs, and parity-mode counts are reported, "
                         "not gated)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    N = int(args.N) if args.N else DEFAULT_N.get(cfg.name, cfg.N)
    q = cfg.q
    h, m = O.choose_params(cfg.kernel, cfg.ell, cfg.d, cfg.eps, cfg.nu)
    M = (2 * m + 1) ** cfg.d
    shard = args.shard or (50_000 if cfg.d == 3 else 500_000)
    t = {}
    log = lambda s: print(f"[{cfg.name} {time.strftime('%H:%M:%S')}] {s}", flush=True)
    log(f"N={N} q={q} h={h} m={m} M={M} workers={args.workers} shard={shard}")

    t0 = time.perf_counter()
    cache = os.path.join(args.cache, f"{cfg.name}_N{N}_{oracle_hash()[:12]}.npz")
    if args.reuse and os.path.exists(cache):
        z = np.load(cache)
        v, fy = z["v"], z["fy"]
        log(f"type-1 sums from {cache}")
    else:
        jobs = [(cfg.name, a, min(N, a + shard), h, m) for a in range(0, N, shard)]
        v = np.zeros((4 * m + 1,) * cfg.d, dtype=np.complex128)
        fy = np.zeros((2 * m + 1,) * cfg.d, dtype=np.complex128)
        with mp.get_context("fork").Pool(args.workers) as pool:
            for k, (vp, fp) in enumerate(pool.imap_unordered(_shard, jobs)):
                v += vp
                fy += fp
                if (k + 1) % max(1, len(jobs) // 20) == 0:
                    log(f"type-1 sums {k + 1}/{len(jobs)} shards")
        os.makedirs(args.cache, exist_ok=True)
        np.savez(cache, v=v, fy=fy)
    t["type1_sums_s"] = time.perf_counter() - t0
    D = O.spectral_weights(cfg.kernel, cfg.ell, cfg.d, h, m, cfg.nu)
    b = D * fy
    log(f"type-1 sums {t['type1_sums_s']:.1f} s, v0={v[(2 * m,) * cfg.d].real:.1f}")

    use_fft = cfg.name == "c4"          # reading G11: the one exception to the direct product
    T = None
    if not use_fft:
        t0 = time.perf_counter()
        T = O.toeplitz_matrix(v, m)      # dense T_pq = v_{j_p - j_q} (eq 223), M <= 9801
        t["dense_T_s"] = time.perf_counter() - t0
    A = lambda p: O.system_apply(v, D, cfg.sigma ** 2, p, T, fft=use_fft)

    res = {}
    for mode, tol in (("parity", cfg.eps / 1000), ("production", cfg.eps)):
        cap = O.default_max_iter(N, cfg.sigma, tol)
        cg_cache = os.path.join(args.cache, f"{cfg.name}_N{N}_{oracle_hash()[:12]}_cg_{mode}.npz")
        t0 = time.perf_counter()
        if args.reuse and os.path.exists(cg_cache):
            z = np.load(cg_cache)
            beta, iters, hist = z["beta"], int(z["iters"]), list(z["hist"])
            t[f"cg_{mode}_s"] = float(z["seconds"])
            log(f"CG {mode} from {cg_cache}")
        else:
            beta, iters, hist = O.cg(A, b, tol, cap)
            t[f"cg_{mode}_s"] = time.perf_counter() - t0
            np.savez(cg_cache, beta=beta, iters=iters, hist=np.asarray(hist), seconds=t[f"cg_{mode}_s"])
        true_rel = float(np.linalg.norm(A(beta) - b) / np.linalg.norm(b))
        log(f"CG {mode}: tol {tol:g} iters {iters} (cap {cap}) true rel resid {true_rel:.2e} "
            f"{t[f'cg_{mode}_s']:.1f} s")
        res[mode] = (beta, iters, np.asarray(hist), true_rel, cap)

    # Reading G10b: the oracle's own first crossings when v and F^*y carry an error of the size the
    # NUFFT contract allows (relative l2 = nufft_tol = eps/10), seeds 1..K.  v is perturbed
    # by 64 phantom points of equal positive mass (eq 88's sum over extra points, so T stays positive
    # semidefinite: white noise of that size makes the c2 system indefinite), F^*y by Hermitian white
    # noise.  The GPU's count passes if it lies within these counts +-2 (or in G10's window): the
    # crossing of a plateaued residual moves by more than +-2 under any such error.
    ntol = cfg.eps / 10
    perturbed = {"parity": [], "production": []}
    pmodes = (args.perturb_modes or ("production" if cfg.name == "c4" else "parity,production")).split(",")

    def herm(z):
        return 0.5 * (z + np.conj(z[(slice(None, None, -1),) * z.ndim]))

    for k in range(1, args.perturb + 1):
        rng = np.random.default_rng(k)
        dv = O.toeplitz_vector(rng.uniform(size=(64, cfg.d)), h, m)
        db = herm(rng.normal(size=b.shape) + 1j * rng.normal(size=b.shape))
        vk = v + dv * (ntol * np.linalg.norm(v) / np.linalg.norm(dv))
        bk = b + db * (ntol * np.linalg.norm(b) / np.linalg.norm(db))
        Tk = None if use_fft else O.toeplitz_matrix(vk, m)
        Ak = lambda p: O.system_apply(vk, D, cfg.sigma ** 2, p, Tk, fft=use_fft)
        for mode, tol in (("parity", cfg.eps / 1000), ("production", cfg.eps)):
            if mode not in pmodes:
                continue
            cap = min(O.default_max_iter(N, cfg.sigma, tol), 3 * res[mode][1] + 50)
            _, it_k, _ = O.cg(Ak, bk, tol, cap)
            perturbed[mode].append(int(it_k))
        log(f"perturbed CG {k}: " + " ".join(f"{md} {perturbed[md][-1]}" for md in pmodes))
        del Tk

    xt = targets(cfg, 0, q)
    mus = {}
    for mode in ("parity", "production"):
        t0 = time.perf_counter()
        mus[mode] = O.posterior_mean(res[mode][0], D, h, xt)
        t[f"mu_{mode}_s"] = time.perf_counter() - t0
    log(f"mu done; parity vs production rel {np.linalg.norm(mus['parity'] - mus['production']) / np.linalg.norm(mus['parity']):.2e}")

    os.makedirs(args.out, exist_ok=True)
    arrays = {"mu_parity": mus["parity"], "mu_production": mus["production"],
              "hist_parity": res["parity"][2], "hist_production": res["production"][2]}
    # small mode vectors in full; c4's (149^3 / 75^3) as norms + seeded samples
    if v.size * 16 <= 4 << 20:
        arrays.update(v=v, b=b, beta_parity=res["parity"][0])
    else:
        rng = np.random.default_rng(1234)
        iv = rng.integers(0, v.size, 4096)
        ib = rng.integers(0, b.size, 4096)
        arrays.update(v_idx=iv, v_sample=v.reshape(-1)[iv], b_idx=ib, b_sample=b.reshape(-1)[ib],
                      beta_parity_sample=res["parity"][0].reshape(-1)[ib])
    base = os.path.join(args.out, f"full_{cfg.name}")
    np.savez_compressed(base + ".npz", **arrays)
    meta = {"config": cfg.name, "N": N, "q": q, "seed": cfg.seed, "h": h, "m": m, "M": M,
            "reading": "A (Matern eps rescaling by ||k||_L2), G1 signs, G9 parity mode eps/1000",
            "toeplitz_product": "host FFT (reading G11)" if use_fft else "direct (dense T)",
            "v_norm": float(np.linalg.norm(v)), "b_norm": float(np.linalg.norm(b)),
            "iters_parity": int(res["parity"][1]), "iters_production": int(res["production"][1]),
            "cap_parity": int(res["parity"][4]), "cap_production": int(res["production"][4]),
            "true_rel_resid_parity": res["parity"][3], "true_rel_resid_production": res["production"][3],
            "iters_perturbed": perturbed,
            "perturbation": "relative l2 = eps/10: v + 64 phantom points (PSD), F^*y + white noise (reading G10b)",
            "oracle_sha256": oracle_hash(), "data_sha256": data_hash(),
            "oracle_seconds": t, "host": {"cores": args.workers, "model": host_model()},
            "written": time.strftime("%Y-%m-%dT%H:%M:%S")}
    with open(base + ".json", "w") as f:
        json.dump(meta, f, indent=1)
    log(f"wrote {base}.npz/.json: {json.dumps({k: meta[k] for k in ('iters_parity', 'iters_production')})}")


if __name__ == "__main__":
    main()
