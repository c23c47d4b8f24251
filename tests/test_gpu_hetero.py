"""NEXT-3 (heteroskedastic noise, reading G11) parity: the GPU NUFFT-pair CG against the
oracle's dense-Phi CG on the same seeded inputs, plus the homoskedastic limit against the GPU
Toeplitz path, edge cases, and a large-N property check."""
import math

import numpy as np
import pytest

from _util import O, CONFIGS, generate, rel, dev, model, gpu_beta_full

pytestmark = pytest.mark.gpu

# (N, m override or None)
HET_SIZES = {"c1": (3000, None), "c2": (3000, 12), "c3": (3000, None), "c4": (1500, 5), "c5": (4000, None)}


def noise_sd(c, N, seed):
    # per-point noise: sigma * (0.5 + u), u ~ U[0,1) (DESIGN.md input recipe, NEXT-3)
    return c.sigma * (0.5 + np.random.default_rng(seed).uniform(0, 1, N))


_ORACLE_HET = {}


def _oracle_hetero(name):
    # the three solver paths of one config share inputs: the oracle fit (c5: ~2.5 min) runs once
    if name not in _ORACLE_HET:
        c = CONFIGS[name]
        N, m_over = HET_SIZES[name]
        x, y, xt = generate(c, N=N, q=min(c.q, 1000))
        sd = noise_sd(c, N, 40 + c.id)
        kw = {}
        if m_over is not None:
            kw = dict(h=O.choose_params(c.kernel, c.ell, c.d, c.eps, c.nu)[0], m=m_over)
        fit = O.efgp_fit_hetero(x, y, sd, c.kernel, c.ell, c.eps, nu=c.nu, h=kw.get("h"), m=kw.get("m"),
                                cg_tol=c.eps / 1000)
        _ORACLE_HET[name] = (fit, O.efgp_predict(fit, xt))
    return _ORACLE_HET[name]


@pytest.mark.parametrize("path", ["toeplitz", "sorted", "unfused"])
@pytest.mark.parametrize("name", list(CONFIGS))
def test_hetero_parity(name, path, monkeypatch):
    # "toeplitz": the weighted Toeplitz system of reading G11b (SORTED / CELLSORT spreading: c2-c5);
    # "sorted": NUFFT pair per iteration, points counting-sorted once by cell, one fused pass (d <= 2);
    # "unfused": K8 + C2R + K9 + K1 + R2C per iteration (the d = 3 path; forced by the env switch)
    kw_h = {"hetero": "toeplitz" if path == "toeplitz" else "nufft"}
    if path == "unfused":
        monkeypatch.setenv("EFGP_HETERO_SORTED", "0")
    c = CONFIGS[name]
    if path == "sorted" and c.d == 3:
        pytest.skip("no sorted path in 3D (W^3 register windows)")
    if path == "toeplitz" and name == "c1":
        pytest.skip("c1 spreads y on n2 (SMEM): the TOEPLITZ solver needs the v grid (falls back to NUFFT)")
    N, m_over = HET_SIZES[name]
    x, y, xt = generate(c, N=N, q=min(c.q, 1000))
    sd = noise_sd(c, N, 40 + c.id)
    cg_tol = c.eps / 1000                                          # parity mode (reading G9)
    kw = {}
    if m_over is not None:
        h0, _ = O.choose_params(c.kernel, c.ell, c.d, c.eps, c.nu)
        kw = dict(h=h0, m=m_over)
    g = model(c, cg_tol=cg_tol, **kw, **kw_h)
    g.fit_hetero(dev(x), dev(y), dev(sd))
    mu = g.predict(dev(xt)).cpu().numpy()
    inf = g.info()
    assert inf["hetero_sorted"] == {"toeplitz": 2, "sorted": 1, "unfused": 0}[path]
    fit, ref = _oracle_hetero(name)
    assert rel(mu, ref) <= 10 * c.eps, (rel(mu, ref), 10 * c.eps)
    hist = g.residual_history()
    assert len(hist) == inf["iters"] + 1 and hist[-1] <= cg_tol
    # reading G10: +-2, or inside the oracle's [2 tol, tol/2] window, or (long parity-mode runs) 10 %
    lo = next((k for k, r in enumerate(fit.history) if r <= 2 * cg_tol), len(fit.history))
    hi = next((k for k, r in enumerate(fit.history) if r <= cg_tol / 2), len(fit.history) + 10)
    assert (abs(inf["iters"] - fit.iters) <= 2 or lo <= inf["iters"] <= hi
            or abs(inf["iters"] - fit.iters) <= 0.1 * fit.iters), (inf["iters"], fit.iters, lo, hi)
    k = min(8, fit.iters, inf["iters"])
    np.testing.assert_allclose(hist[:k + 1], fit.history[:k + 1], rtol=1e-2)
    # the right-hand side Phi^* S^-1 y to NUFFT accuracy
    from paper_2210_10210_b200 import half_to_full
    b = half_to_full(g.vector("rhs"), inf["m"], c.d)
    assert rel(b, fit.b) <= 5 * inf["nufft_tol"]
    if path == "toeplitz":
        # v^w = eq 88 with strengths sigma_n^-2 (reading G11b), and the variance with sigma^2 -> 1
        vw = half_to_full(g.vector("v"), inf["m"], c.d, K=2 * inf["m"])
        vw_ref = O.toeplitz_vector_weighted(x, 1.0 / sd ** 2, fit.h, fit.m)
        assert rel(vw, vw_ref) <= 5 * inf["nufft_tol"]
        if c.d <= 2:
            xv = xt[:8]
            var = g.predict_var(dev(xv)).cpu().numpy()
            ref_v = O.posterior_variance_hetero(fit, x, sd, xv)
            assert rel(var, ref_v) <= 10 * c.eps, (rel(var, ref_v), 10 * c.eps)
    g.close()


@pytest.mark.parametrize("spread", ["sorted", "global"])
def test_hetero_constant_noise_matches_toeplitz_fit(spread):
    # sigma_n = sigma: the NUFFT-pair operator and the Toeplitz operator are the same matrix (scaled
    # by 1/sigma^2), two independent GPU paths; beta agrees to the NUFFT tolerance
    c = CONFIGS["c5"]
    x, y, xt = generate(c, N=200_000, q=500)
    g1 = model(c, cg_tol=c.eps / 1000, spread=spread)
    g1.fit(dev(x), dev(y))
    g2 = model(c, cg_tol=c.eps / 1000, spread=spread, hetero="nufft")
    g2.fit_hetero(dev(x), dev(y), dev(np.full(len(x), c.sigma)))
    i1, i2 = g1.info(), g2.info()
    assert abs(i1["iters"] - i2["iters"]) <= 0.1 * i1["iters"] + 2
    mu1 = g1.predict(dev(xt)).cpu().numpy()
    mu2 = g2.predict(dev(xt)).cpu().numpy()
    assert rel(mu2, mu1) <= 10 * c.eps
    g1.close()
    g2.close()


def test_hetero_edge_cases():
    from paper_2210_10210_b200 import EFGPError
    c = CONFIGS["c5"]
    x, y, xt = generate(c, N=3000, q=50)
    sd = noise_sd(c, 3000, 7)
    g = model(c)
    for bad in (0.0, -1.0, float("nan"), float("inf")):
        s2 = sd.copy()
        s2[123] = bad
        with pytest.raises(EFGPError, match="INVALID"):
            g.fit_hetero(dev(x), dev(y), dev(s2))
    xb = x.copy()
    xb[5, 1] = 1.5
    with pytest.raises(EFGPError, match="INVALID"):
        g.fit_hetero(dev(xb), dev(y), dev(sd))
    g.fit_hetero(dev(x), dev(y), dev(sd))
    mu_d = g.predict(dev(xt)).cpu().numpy()
    b_d = g.vector("rhs")
    g.fit_hetero(x, y, sd)                                         # host arrays
    # spreading atomics make runs agree to roundoff; CG amplifies it (as test_host_inputs_match_device_inputs)
    assert rel(g.vector("rhs"), b_d) < 1e-13
    assert rel(g.predict(dev(xt)).cpu().numpy(), mu_d) < 10 * c.eps
    g.predict_var(dev(xt))                                         # TOEPLITZ solve: variance available
    gn = model(c, hetero="nufft")
    gn.fit_hetero(dev(x), dev(y), dev(sd))
    with pytest.raises(EFGPError, match="INVALID"):
        gn.predict_var(dev(xt))                                    # NUFFT solve: no Toeplitz operator
    gn.close()
    # a single point: closed form mu(x0) = k~(0) y / (k~(0) + sd^2), to the NUFFT tolerance
    x0 = np.array([[0.3, 0.6]])
    g.fit_hetero(dev(x0), dev(np.array([2.0])), dev(np.array([0.5])))
    D = O.spectral_weights(c.kernel, c.ell, 2, g.info()["h"], g.info()["m"], c.nu)
    k0 = float(np.sum(D ** 2))
    mu0 = g.predict(dev(x0)).cpu().numpy()[0]
    assert mu0 == pytest.approx(k0 * 2.0 / (k0 + 0.25), rel=5 * g.info()["nufft_tol"])
    g.close()


def test_hetero_large_n_two_noise_levels():
    # property at size (N = 2e7, the device generator): with sigma_n = sigma on the first half and 1e6 on
    # the second, the second half drops out and the fit equals the Toeplitz fit of the first half alone
    import torch
    from efgp_data import gpu as G
    c = CONFIGS["c5"]
    N = 20_000_000
    x, y = G.generate_points(c, 0, N)
    xt = torch.rand(1000, 2, dtype=torch.float64, device="cuda")
    sd = torch.full((N,), c.sigma, dtype=torch.float64, device="cuda")
    sd[N // 2:] = 1e6
    g = model(c, cg_tol=c.eps / 1000)
    g.fit_hetero(x, y, sd)
    mu_h = g.predict(xt).cpu().numpy()
    g2 = model(c, cg_tol=c.eps / 1000)
    g2.fit(x[:N // 2].contiguous(), y[:N // 2].contiguous())
    mu_ref = g2.predict(xt).cpu().numpy()
    assert rel(mu_h, mu_ref) <= 10 * c.eps, rel(mu_h, mu_ref)
    g.close()
    g2.close()


def test_hetero_toeplitz_with_kron_preconditioner():
    # the TOEPLITZ solver accepts the NEXT-4 preconditioner (factors from the weighted v^w, sigma^2 -> 1):
    # same answer as the plain CG, fewer iterations (c3: SE, separable density)
    from efgp_data import gpu as G
    import torch
    c = CONFIGS["c3"]
    N = 200_000
    x, y = G.generate_points(c, 0, N)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(7)
    sd = c.sigma * (0.5 + torch.rand(N, dtype=torch.float64, device="cuda", generator=gen))
    xt = dev(np.random.default_rng(8).uniform(0, 1, (300, 2)))
    out = {}
    for pc in (None, "kron"):
        g = model(c, cg_tol=c.eps / 1000, precond=pc)               # parity mode (reading G9)
        g.fit_hetero(x, y, sd)
        inf = g.info()
        assert inf["hetero_sorted"] == 2 and inf["precond"] == (1 if pc else 0)
        out[pc] = (g.predict(xt).cpu().numpy(), inf["iters"])
        g.close()
    assert rel(out["kron"][0], out[None][0]) <= 10 * c.eps
    assert out["kron"][1] < out[None][1] / 2, (out["kron"][1], out[None][1])


def test_hetero_toeplitz_with_jacobi_preconditioner():
    # Jacobi (reading G12b) on the weighted system D T(v^w) D + I of reading G11b: the same mean as the
    # oracle's dense heteroskedastic solve path (efgp_fit_hetero), c5 (Matern, 1D)
    c = CONFIGS["c5"]
    rng = np.random.default_rng(17)
    x, y, xt = generate(c, N=3_000, q=300)                         # oracle: ~16 s
    sd = c.sigma * (0.5 + rng.uniform(0, 1, len(x)))
    out = {}
    for pc in (None, "jacobi"):
        g = model(c, cg_tol=c.eps / 1000, precond=pc)
        g.fit_hetero(dev(x), dev(y), dev(sd))
        inf = g.info()
        assert inf["hetero_sorted"] == 2 and inf["precond"] == (3 if pc else 0)
        out[pc] = (g.predict(dev(xt)).cpu().numpy(), inf["iters"])
        g.close()
    fit = O.efgp_fit_hetero(x, y, sd, c.kernel, c.ell, c.eps, nu=c.nu, cg_tol=c.eps / 1000)
    ref = O.efgp_predict(fit, xt)
    assert rel(out["jacobi"][0], ref) <= 10 * c.eps
    assert rel(out[None][0], ref) <= 10 * c.eps


@pytest.mark.parametrize("eps", [1e-1, 1e-2, 1e-5])
def test_hetero_solvers_agree_every_width(eps):
    # the NUFFT-pair solver (sorted fused pass, widths W = 3, 4, 7 here) and the TOEPLITZ solver solve
    # the same system: their means agree to the NUFFT tolerance (both CGs in parity mode)
    from paper_2210_10210_b200 import EFGP
    rng = np.random.default_rng(int(1 / eps))
    N = 30_000
    x = rng.uniform(0, 1, (N, 2))
    y = np.sin(5 * x[:, 0]) * np.cos(3 * x[:, 1]) + 0.1 * rng.standard_normal(N)
    sd = 0.1 * (0.5 + rng.uniform(0, 1, N))
    xt = rng.uniform(0, 1, (200, 2))
    mus, ws = {}, {}
    for meth in ("nufft", "toeplitz"):
        g = EFGP("matern", 0.2, 0.1, eps, 2, 1.5, cg_tol=eps / 1000, hetero=meth)
        g.fit_hetero(dev(x), dev(y), dev(sd))
        inf = g.info()
        assert inf["hetero_sorted"] == (1 if meth == "nufft" else 2)
        mus[meth] = g.predict(dev(xt)).cpu().numpy()
        ws[meth] = inf["w"]
        g.close()
    assert rel(mus["nufft"], mus["toeplitz"]) <= 10 * eps, rel(mus["nufft"], mus["toeplitz"])


def test_nufft_solver_reports_no_preconditioner():
    # options.precond applies to the TOEPLITZ solver only: a NUFFT-pair fit after a preconditioned
    # homoskedastic fit reports NONE
    c = CONFIGS["c5"]
    x, y, xt = generate(c, N=5_000, q=20)
    sd = noise_sd(c, len(x), 77)
    g = model(c, precond="jacobi", hetero="toeplitz")
    g.fit_hetero(dev(x), dev(y), dev(sd))
    assert g.info()["precond"] == 3
    g.close()
    g = model(c, precond="jacobi", hetero="nufft")
    g.fit(dev(x), dev(y))
    assert g.info()["precond"] == 3
    g.fit_hetero(dev(x), dev(y), dev(sd))
    assert g.info()["precond"] == 0 and g.info()["hetero_sorted"] in (0, 1)
    assert np.all(np.isfinite(g.predict(dev(xt)).cpu().numpy()))
    g.close()


def test_hetero_sorted_raw_one_pass_matches_prep_routes():
    # SORTED reads the raw (y_n, sigma_n) and forms 1/sigma_n^2, y_n/sigma_n^2 in its own pass 2 (no prep
    # pass); CELLSORT takes the prep kernel's strengths (one pass), and an unaligned sigma array makes
    # SORTED fall back to prep + two passes.  Same strengths, same grids: the right-hand sides agree to the
    # rounding of the fp64 atomics, the iteration cap (min sigma_n) exactly, mu to the parity gate.
    import torch
    c = CONFIGS["c5"]
    N = 300_001
    x, y, xt = generate(c, N=N, q=300)
    sd = noise_sd(c, N, 11)
    sd[777] = 0.25 * c.sigma                                        # a unique minimum
    gs = model(c, cg_tol=c.eps / 1000, spread="sorted")
    gs.fit_hetero(dev(x), dev(y), dev(sd))
    assert gs.info()["spread_method"] == "sorted" and gs.info()["spread_fallback"] == "none"
    gg = model(c, cg_tol=c.eps / 1000, spread="cellsort")
    gg.fit_hetero(dev(x), dev(y), dev(sd))
    assert gg.info()["spread_method"] == "cellsort"
    bs, bg = gs.vector("rhs"), gg.vector("rhs")
    assert rel(bs, bg) < 1e-12, rel(bs, bg)
    assert gs.info()["max_iter"] == gg.info()["max_iter"]
    mu_s = gs.predict(dev(xt)).cpu().numpy()
    mu_g = gg.predict(dev(xt)).cpu().numpy()
    assert rel(mu_s, mu_g) <= 10 * c.eps
    # 8-byte-aligned (not 16) sigma: the bulk copies cannot take it -> prep + two passes, same answer
    buf = torch.empty(N + 1, dtype=torch.float64, device="cuda")
    buf[1:] = torch.from_numpy(sd)
    gs.fit_hetero(dev(x), dev(y), buf[1:])
    assert rel(gs.vector("rhs"), bg) < 1e-12
    assert gs.info()["max_iter"] == gg.info()["max_iter"]
    gs.close()
    gg.close()
