"""NEXT-4 (Kronecker preconditioner, reading G12) on the GPU: PCG parity against the
oracle's PCG on all five configs, exactness cases, and the iteration reduction."""
import numpy as np
import pytest

from _util import O, CONFIGS, generate, rel, dev, model

pytestmark = pytest.mark.gpu

PC_SIZES = {"c1": (10_000, None), "c2": (20_000, 20), "c3": (5_000, None), "c4": (3_000, 6), "c5": (50_000, None)}


@pytest.mark.parametrize("name", list(CONFIGS))
def test_pcg_parity(name):
    c = CONFIGS[name]
    N, m_over = PC_SIZES[name]
    x, y, xt = generate(c, N=N, q=min(c.q, 2000))
    cg_tol = c.eps / 1000                                          # parity mode (reading G9)
    kw = {}
    if m_over is not None:
        h0, _ = O.choose_params(c.kernel, c.ell, c.d, c.eps, c.nu)
        kw = dict(h=h0, m=m_over)
    g = model(c, cg_tol=cg_tol, precond="kron", **kw)
    g.fit(dev(x), dev(y))
    mu = g.predict(dev(xt)).cpu().numpy()
    inf = g.info()
    assert inf["precond"] == 1
    fit = O.efgp_fit(x, y, c.kernel, c.ell, c.sigma, c.eps, nu=c.nu, cg_tol=cg_tol, h=kw.get("h"), m=kw.get("m"),
                     precond="kron")
    ref = O.efgp_predict(fit, xt)
    assert rel(mu, ref) <= 10 * c.eps, (rel(mu, ref), 10 * c.eps)
    hist = g.residual_history()
    assert len(hist) == inf["iters"] + 1 and hist[-1] <= cg_tol
    lo = next((k for k, r in enumerate(fit.history) if r <= 2 * cg_tol), len(fit.history))
    hi = next((k for k, r in enumerate(fit.history) if r <= cg_tol / 2), len(fit.history) + 10)
    assert (abs(inf["iters"] - fit.iters) <= 2 or lo <= inf["iters"] <= hi
            or abs(inf["iters"] - fit.iters) <= 0.1 * fit.iters), (inf["iters"], fit.iters, lo, hi)
    # the trajectories agree to NUFFT accuracy while the residuals are well above roundoff
    k = min(5, fit.iters, inf["iters"])
    big = [i for i in range(k + 1) if fit.history[i] > 1e3 * cg_tol]
    np.testing.assert_allclose(np.asarray(hist)[big], np.asarray(fit.history)[big], rtol=1e-2)
    # the same answer as plain CG (the preconditioner changes the path, not the solution)
    g2 = model(c, cg_tol=cg_tol, **kw)
    g2.fit(dev(x), dev(y))
    assert rel(mu, g2.predict(dev(xt)).cpu().numpy()) <= 10 * c.eps
    assert inf["iters"] <= g2.info()["iters"]
    g.close()
    g2.close()


def test_pcg_exact_on_tensor_grid_se():
    # tensor-product points + separable SE density: the NUFFT v is separable too, so M is the system
    # matrix and PCG stops after one iteration
    rng = np.random.default_rng(31)
    a, b = np.sort(rng.uniform(0, 1, 40)), np.sort(rng.uniform(0, 1, 50))
    x = np.array([(p, q) for p in a for q in b])
    y = np.sin(5 * x[:, 0]) * np.cos(3 * x[:, 1])
    c = CONFIGS["c3"]
    g = model(c, cg_tol=1e-10, precond="kron")
    g.fit(dev(x), dev(y))
    assert g.info()["iters"] <= 2, g.info()["iters"]
    g.close()


def test_pcg_one_dimension_exact():
    c = CONFIGS["c1"]
    x, y, _ = generate(c, N=20_000, q=1)
    g = model(c, cg_tol=1e-10, precond="kron")
    g.fit(dev(x), dev(y))
    assert g.info()["iters"] <= 2
    g.close()


def test_pcg_reduces_iterations_at_size():
    # c3 (SE, separable density: the case reading G12 targets) at N = 1e6 from the device generator.
    # PCG stopped at eps/10 needs a fraction of plain CG's iterations at eps and lands closer to the
    # converged mean (at equal residual the two errors differ: kappa ~ N / sigma^2, reading G9)
    from efgp_data import gpu as G
    c = CONFIGS["c3"]
    x, y = G.generate_points(c, 0, 1_000_000)
    xt = dev(np.random.default_rng(3).uniform(0, 1, (500, 2)))
    g2 = model(c, cg_tol=c.eps / 1e5, precond="kron")
    g2.fit(x, y)
    conv = g2.predict(xt).cpu().numpy()
    g0 = model(c)
    g0.fit(x, y)
    g1 = model(c, cg_tol=c.eps / 10, precond="kron")
    g1.fit(x, y)
    i0, i1 = g0.info()["iters"], g1.info()["iters"]
    assert i1 < i0 / 3, (i0, i1)
    e0 = rel(g0.predict(xt).cpu().numpy(), conv)
    e1 = rel(g1.predict(xt).cpu().numpy(), conv)
    assert e1 <= e0, (e1, e0)
    for g in (g0, g1, g2):
        g.close()


def test_auto_selects_kron_for_se_jacobi_otherwise():
    for name, want in (("c3", 1), ("c5", 3)):
        c = CONFIGS[name]
        x, y, _ = generate(c, N=2000, q=1)
        g = model(c, precond="auto")
        g.fit(dev(x), dev(y))
        assert g.info()["precond"] == want
        g.close()


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_variance_with_kron_preconditioner(name, monkeypatch):
    # NEXT-2 with NEXT-4: the per-target CGs preconditioned by the fit's Kronecker factors (inside each
    # target's CTA).  Same variances as the oracle's plain per-target CG (parity mode).
    c = CONFIGS[name]
    x, y, _ = generate(c, N=3000, q=1)
    xt = np.random.default_rng(40 + c.id).uniform(0, 1, (37, c.d))
    xt[0] = x[0]
    cg_tol = c.eps / 1000
    monkeypatch.setenv("EFGP_VAR_BATCH", "16")
    g = model(c, cg_tol=cg_tol, precond="kron")
    g.fit(dev(x), dev(y))
    var = g.predict_var(dev(xt)).cpu().numpy()
    fit = O.efgp_fit(x, y, c.kernel, c.ell, c.sigma, c.eps, nu=c.nu, cg_tol=cg_tol)
    ref = O.posterior_variance(fit, xt, cg_tol=cg_tol)
    assert rel(var, ref) <= 10 * c.eps, (rel(var, ref), 10 * c.eps)
    if name == "c1":
        assert g.info()["var_iters_max"] <= 2                      # d = 1: M is the system matrix
    g.close()


def test_variance_kron_reduces_iterations_at_size():
    # c3 at N = 1e5 (device generator): preconditioned vs plain batched CG, both to eps/100
    from efgp_data import gpu as G
    c = CONFIGS["c3"]
    x, y = G.generate_points(c, 0, 100_000)
    xt = G.generate_targets(c, 0, 48)
    out = {}
    for pc in (None, "kron"):
        g = model(c, cg_tol=c.eps / 100, precond=pc)
        g.fit(x, y)
        out[pc] = (g.predict_var(xt).cpu().numpy(), g.info()["var_iters_max"])
        g.close()
    assert rel(out["kron"][0], out[None][0]) <= 10 * c.eps
    assert out["kron"][1] < out[None][1] / 2, (out["kron"][1], out[None][1])


# ---- NEXT-4, Jacobi preconditioner M = diag(D_j^2 v_0 + sigma^2) (reading G12b)

@pytest.mark.parametrize("name", ["c2", "c5", "c4"])
def test_pcg_jacobi_parity(name):
    c = CONFIGS[name]
    N, m_over = PC_SIZES[name]
    x, y, xt = generate(c, N=N, q=min(c.q, 2000))
    cg_tol = c.eps / 1000                                          # parity mode (reading G9)
    kw = {}
    if m_over is not None:
        h0, _ = O.choose_params(c.kernel, c.ell, c.d, c.eps, c.nu)
        kw = dict(h=h0, m=m_over)
    g = model(c, cg_tol=cg_tol, precond="jacobi", **kw)
    g.fit(dev(x), dev(y))
    mu = g.predict(dev(xt)).cpu().numpy()
    inf = g.info()
    assert inf["precond"] == 3
    fit = O.efgp_fit(x, y, c.kernel, c.ell, c.sigma, c.eps, nu=c.nu, cg_tol=cg_tol, h=kw.get("h"), m=kw.get("m"),
                     precond="jacobi")
    ref = O.efgp_predict(fit, xt)
    assert rel(mu, ref) <= 10 * c.eps, (rel(mu, ref), 10 * c.eps)
    hist = g.residual_history()
    assert len(hist) == inf["iters"] + 1 and hist[-1] <= cg_tol
    assert abs(inf["iters"] - fit.iters) <= max(3, 0.1 * fit.iters), (inf["iters"], fit.iters)
    k = min(5, fit.iters, inf["iters"])
    big = [i for i in range(k + 1) if fit.history[i] > 1e3 * cg_tol]
    np.testing.assert_allclose(np.asarray(hist)[big], np.asarray(fit.history)[big], rtol=1e-2)
    g.close()


def test_pcg_jacobi_reduces_iterations_matern():
    # c5 (Matern-3/2, 1D heavy-tailed spectral density: D_j^2 v_0 spans many decades) at N = 1e6
    from efgp_data import gpu as G
    c = CONFIGS["c5"]
    x, y = G.generate_points(c, 0, 1_000_000)
    out = {}
    for pc in (None, "jacobi"):
        g = model(c, precond=pc)
        g.fit(x, y)
        out[pc] = g.info()["iters"]
        g.close()
    assert out["jacobi"] < out[None] / 2, out


@pytest.mark.parametrize("name", ["c2", "c5"])
def test_variance_with_jacobi_preconditioner(name, monkeypatch):
    c = CONFIGS[name]
    x, y, _ = generate(c, N=3000, q=1)
    xt = np.random.default_rng(50 + c.id).uniform(0, 1, (8, c.d))   # oracle: ~1e3 iterations per target
    xt[0] = x[0]
    cg_tol = c.eps / 1000
    kw = {}
    if name == "c2":                                               # m = 12 keeps the oracle in seconds
        kw = dict(h=O.choose_params(c.kernel, c.ell, c.d, c.eps, c.nu)[0], m=12)
    monkeypatch.setenv("EFGP_VAR_BATCH", "16")
    g = model(c, cg_tol=cg_tol, precond="jacobi", **kw)
    g.fit(dev(x), dev(y))
    var = g.predict_var(dev(xt)).cpu().numpy()
    fit = O.efgp_fit(x, y, c.kernel, c.ell, c.sigma, c.eps, nu=c.nu, cg_tol=cg_tol, **kw)
    ref = O.posterior_variance(fit, xt, cg_tol=cg_tol, precond="jacobi")
    assert rel(var, ref) <= 10 * c.eps, (rel(var, ref), 10 * c.eps)
    g.close()
