"""GPU parity at the BASELINE configs' own sizes against cached oracle dumps (tests/golden).

The dumps come from tests/make_golden.py (oracle + efgp_data only): Algorithm a1 run by the oracle
over ALL N points of each config (c5: the first 1e8 of its 1e9 records), with CG to eps/1000 (parity
mode, reading G9) and to eps (production mode), the direct Toeplitz product (dense T) or, for c4, the
host FFT of reading G11.  This test regenerates the same inputs on the device (efgp_data's CUDA
Philox: uniforms bitwise equal, normals within a few ulp), runs the library through the C ABI in the
launch configuration bench.py / tools/bench_configs.py time (default options: SORTED for c2/c5,
CELLSORT for c3/c4, the FFT Toeplitz CG for c2 (m = 49) and c4 (m = 37), the direct one for c3/c5),
and gates:

  * (h, m) equal to the oracle's;
  * type-1 outputs v and Phi^*y against the oracle's exact sums: relative l2 <= 5 nufft_tol (c4:
    4096 sampled entries, error relative to the oracle's norm);
  * parity mode: mu relative l2 over the config's targets <= 10 eps (north_star);
  * iteration counts (both modes): within +-2 of the oracle's, inside its [2 eps_cg, eps_cg/2]
    crossing window (reading G10), or within +-2 of the span of first crossings the ORACLE itself
    shows from exact v and F^*y to v and F^*y carrying an error of the size the NUFFT contract allows
    (reading G10b, counts stored by tests/make_golden.py).  Gated in production mode; in parity mode (thousands of
    iterations on a plateaued residual) reported, with both residual histories, where it misses —
    there the mu gate is authoritative (reading G9).

Both histories and the counts of every config are written to $EFGP_GOLDEN_REPORT (a directory) when
set, so a GPU run leaves the evidence behind (profiles/r02_golden_*.json).
"""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

from _util import CONFIGS, O, gpu_beta_full, gpu_rhs_full, gpu_v_full, model, rel

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
# configs gated on G10 alone when a dump has no perturbed counts
G10_PRODUCTION = {"c1", "c4", "c5"}
# c3's production first crossing (eps = 1e-6 on a plateaued residual, 2800-3200
# iterations) moves by hundreds of iterations under roundoff-level changes of v and F^*y (the oracle's
# own counts under NUFFT-level perturbations span 2980-3077 against 2790 unperturbed).  There the
# survey asks for the mismatch to be REPORTED with both residual histories (written to
# $EFGP_GOLDEN_REPORT and printed), and the parity-mode mu gate (G9) is authoritative.
G10_REPORT_ONLY = {"c3"}


def _load(name):
    base = os.path.join(GOLD, f"full_{name}")
    if not os.path.exists(base + ".json"):
        pytest.skip(f"no golden dump for {name} (tests/make_golden.py {name})")
    with open(base + ".json") as f:
        meta = json.load(f)
    with open(os.path.join(ROOT, "oracle", "efgp_oracle.py"), "rb") as f:
        h = hashlib.sha256(f.read()).hexdigest()
    assert meta["oracle_sha256"] == h, f"golden {name} was written by another oracle: rerun tests/make_golden.py {name}"
    return meta, np.load(base + ".npz")


def _window(hist, tol):
    lo = next((k for k, r in enumerate(hist) if r <= 2 * tol), len(hist))
    hi = next((k for k, r in enumerate(hist) if r <= tol / 2), len(hist) + 10)
    return lo, hi


def _count_ok(k_g, k_o, hist_o, tol, perturbed):
    """Readings G10 / G10b: +-2, or the oracle's crossing window, or (G10b) the span of the oracle's own
    counts from exact inputs (k_o) to inputs carrying the NUFFT contract's error (the perturbed runs),
    +-2: the GPU's type-1 error lies between the two."""
    lo, hi = _window(hist_o, tol)
    g10 = abs(k_g - k_o) <= 2 or lo <= k_g <= hi
    span = list(perturbed) + [k_o]
    g10b = bool(perturbed) and min(span) - 2 <= k_g <= max(span) + 2
    return g10, g10b, (lo, hi)


def _report(name, rec):
    d = os.environ.get("EFGP_GOLDEN_REPORT")
    if not d:
        return
    os.makedirs(d, exist_ok=True)
    path = os.path.join(d, f"golden_{name}.json")
    old = {}
    if os.path.exists(path):
        with open(path) as f:
            old = json.load(f)
    old.update(rec)
    with open(path, "w") as f:
        json.dump(old, f)


def _inputs(c, N, q):
    from efgp_data import gpu as G
    x, y = G.generate_points(c, 0, N)
    xt = G.generate_targets(c, 0, q)
    return x, y, xt


@pytest.mark.parametrize("name", list(CONFIGS))
def test_golden_parity_mode(name):
    import torch
    meta, G = _load(name)
    c = CONFIGS[name]
    N, q = meta["N"], meta["q"]
    x, y, xt = _inputs(c, N, q)
    cg_tol = c.eps / 1000
    g = model(c, cg_tol=cg_tol)
    g.fit(x, y)
    inf = g.info()
    assert inf["m"] == meta["m"] and inf["h"] == pytest.approx(meta["h"], rel=1e-15, abs=0)
    tol = inf["nufft_tol"]
    # type-1 at full N against the oracle's exact sums
    if "v" in G.files:
        ev, eb = rel(gpu_v_full(None, g), G["v"]), rel(gpu_rhs_full(g), G["b"])
    else:
        vv = gpu_v_full(None, g).reshape(-1)[G["v_idx"]]
        bb = gpu_rhs_full(g).reshape(-1)[G["b_idx"]]
        ev = np.linalg.norm(vv - G["v_sample"]) / (meta["v_norm"] * np.sqrt(len(vv) / (4 * meta["m"] + 1) ** c.d))
        eb = np.linalg.norm(bb - G["b_sample"]) / (meta["b_norm"] * np.sqrt(len(bb) / meta["M"]))
    assert ev <= 5 * tol and eb <= 5 * tol, (ev, eb, tol)
    mu = g.predict(xt).cpu().numpy()
    err = rel(mu, G["mu_parity"])
    hist_g = g.residual_history()
    pert = meta.get("iters_perturbed", {}).get("parity", [])
    g10, g10b, (lo, hi) = _count_ok(inf["iters"], meta["iters_parity"], G["hist_parity"], cg_tol, pert)
    _report(name, {"N": N, "m": meta["m"], "spread": inf["spread_method"], "parity": {
        "mu_rel_err": err, "gate": 10 * c.eps, "type1_rel_err": [ev, eb], "iters_gpu": inf["iters"],
        "iters_oracle": meta["iters_parity"], "oracle_window": [lo, hi], "oracle_perturbed": pert,
        "g10_pass": g10, "g10b_pass": g10b,
        "hist_gpu": list(map(float, hist_g)), "hist_oracle": list(map(float, G["hist_parity"]))}})
    if not (g10 or g10b):
        print(f"{name} parity mode: iteration count {inf['iters']} vs oracle {meta['iters_parity']} "
              f"(window [{lo}, {hi}], perturbed oracle {pert}); mu gate authoritative (G9)")
    assert err <= 10 * c.eps, (err, 10 * c.eps)
    assert len(hist_g) == inf["iters"] + 1 and hist_g[-1] <= cg_tol
    # the trajectories agree to NUFFT accuracy before roundoff decorrelates them
    k = min(10, meta["iters_parity"], inf["iters"])
    np.testing.assert_allclose(hist_g[:k + 1], G["hist_parity"][:k + 1], rtol=max(1e-3, 100 * tol))
    g.close()
    del x, y
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name", list(CONFIGS))
def test_golden_production_iterations(name):
    import torch
    meta, G = _load(name)
    c = CONFIGS[name]
    N, q = meta["N"], meta["q"]
    x, y, xt = _inputs(c, N, q)
    g = model(c)
    g.fit(x, y)
    inf = g.info()
    mu = g.predict(xt).cpu().numpy()
    k_g, k_o = inf["iters"], meta["iters_production"]
    pert = meta.get("iters_perturbed", {}).get("production", [])
    g10, g10b, (lo, hi) = _count_ok(k_g, k_o, G["hist_production"], c.eps, pert)
    ok = g10 or g10b
    hist_g = np.asarray(g.residual_history())
    ho = np.asarray(G["hist_production"])
    kk = min(len(hist_g), len(ho))
    _report(name, {"production": {
        "iters_gpu": k_g, "iters_oracle": k_o, "oracle_window": [lo, hi], "oracle_perturbed": pert,
        "g10_pass": g10, "g10b_pass": g10b,
        "mu_rel_to_oracle_production": rel(mu, G["mu_production"]),
        "mu_rel_to_oracle_parity": rel(mu, G["mu_parity"]),
        "oracle_production_rel_to_parity": rel(G["mu_production"], G["mu_parity"]),
        "hist_ratio_max_first25": float(np.max(np.abs(hist_g[:min(kk, 26)] / ho[:min(kk, 26)] - 1))),
        "hist_gpu": list(map(float, hist_g)), "hist_oracle": list(map(float, ho))}})
    # the GPU's production answer is as close to the converged (parity-mode) answer as the oracle's
    # own production answer is (x2), plus 10 eps (reading G9: the first crossing is hypersensitive)
    e_o = rel(G["mu_production"], G["mu_parity"])
    assert rel(mu, G["mu_parity"]) <= 2 * e_o + 10 * c.eps, (rel(mu, G["mu_parity"]), e_o)
    if not ok:
        print(f"{name} production: iteration count {k_g} vs oracle {k_o} (window [{lo}, {hi}], perturbed oracle "
              f"{pert}); gpu history tail {hist_g[-6:]}, oracle history tail {ho[-6:]}")
    if (pert or name in G10_PRODUCTION) and name not in G10_REPORT_ONLY:
        assert ok, (f"G10/G10b: gpu {k_g} vs oracle {k_o}, window [{lo}, {hi}], perturbed oracle {pert}; "
                    f"histories: gpu {hist_g[max(0, k_o - 5):k_g + 2]} oracle {ho[max(0, k_o - 5):k_o + 2]}")
    g.close()
    del x, y
    torch.cuda.empty_cache()


@pytest.mark.parametrize("N", [1_000_000_000, (1 << 31) + 12_345])
def test_sorted_equals_global_at_full_size(N):
    # the bench's SORTED launch at N = 1e9 and past 2^31 points (int64 indexing in the chunk, segment
    # and batch arithmetic) against GLOBAL (one fp64 RED per touch) on the same points: v to
    # roundoff (a single lost or doubled point would show at ~1e-7), F^*y to the NUFFT tolerance
    # (SORTED spreads y on the n1 grid, GLOBAL on n2)
    import torch
    from efgp_data import gpu as Gd
    c = CONFIGS["c5"]
    try:
        x, y = Gd.generate_points(c, 0, N)
    except RuntimeError as exc:  # pragma: no cover
        pytest.skip(f"cannot allocate {N} points: {exc}")
    out = {}
    for method in ("sorted", "global"):
        g = model(c, max_iter=1, spread=method)
        with pytest.warns(RuntimeWarning):
            g.fit(x, y)
        inf = g.info()
        assert inf["spread_method"] == method and inf["N"] == N
        out[method] = (g.vector("v"), g.vector("rhs"), inf["nufft_tol"])
        g.close()
    assert rel(out["sorted"][0], out["global"][0]) < 1e-12
    assert rel(out["sorted"][1], out["global"][1]) < 2 * out["sorted"][2]
    del x, y
    torch.cuda.empty_cache()
