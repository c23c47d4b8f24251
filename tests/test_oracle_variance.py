"""Pins for the oracle's posterior variance (NEXT-2): eq ``eta`` / ``sws``
against the dense function-space variance with k~ (Lemma l:equiv, an exact identity), the
single-point closed form, the bounds 0 <= s <= k~(0), and the exact SE GP within the eps bound."""
import math

import numpy as np
import pytest

import oracle as O
from efgp_data import CONFIGS


@pytest.mark.parametrize("kernel,nu,ell,sigma,d", [("se", 0.0, 0.1, 0.3, 1), ("matern", 1.5, 0.1, 0.1, 2)])
def test_lemma_equiv_variance_equals_function_space_k_tilde(kernel, nu, ell, sigma, d):
    # Lemma l:equiv, eq sws: s(x*) = sum_j eta_j phi_j(x*) with (Phi^*Phi + sigma^2) eta = sigma^2
    # conj(phi(x*)) equals k~(x*,x*) - k~(x*,X)(K~ + sigma^2)^{-1} k~(X,x*)  (Woodbury).
    rng = np.random.default_rng(3)
    N = {1: 300, 2: 250}[d]
    x = rng.uniform(0, 1, (N, d))
    xt = np.concatenate([rng.uniform(0, 1, (12, d)), x[:3]])
    eps = {1: 1e-4, 2: 1e-3}[d]
    fit = O.efgp_fit(x, np.zeros(N), kernel, ell, sigma, eps, nu=nu)
    s = O.posterior_variance(fit, xt, cg_tol=1e-13, max_iter=20000)
    kt = lambda a, b: O.kernel_tilde_matrix(a, b, fit.h, fit.m, fit.D)
    s_fs = O.dense_gp_variance(x, xt, kt, sigma)
    np.testing.assert_allclose(s, s_fs, rtol=1e-8, atol=1e-10 * float(np.sum(fit.D ** 2)))


def test_variance_single_point_closed_form():
    # N = 1 at x0: s(t) = k~(0) - k~(t - x0)^2 / (k~(0) + sigma^2); at t = x0: k~(0) sigma^2/(k~(0)+sigma^2)
    x0 = np.array([[0.37]])
    sigma = 0.2
    fit = O.efgp_fit(x0, np.array([1.0]), "se", 0.1, sigma, 1e-8, cg_tol=1e-14)
    t = np.array([[0.37], [0.41], [0.9]])
    s = O.posterior_variance(fit, t, cg_tol=1e-14)
    k0 = float(np.sum(fit.D ** 2))
    kt = O.kernel_tilde_matrix(t, x0, fit.h, fit.m, fit.D)[:, 0]
    np.testing.assert_allclose(s, k0 - kt ** 2 / (k0 + sigma ** 2), rtol=1e-10)
    assert s[0] == pytest.approx(k0 * sigma ** 2 / (k0 + sigma ** 2), rel=1e-10)


def test_variance_bounds_and_monotonicity():
    # 0 <= s <= k~(0); adding data can only decrease the variance
    rng = np.random.default_rng(4)
    c = CONFIGS["c5"]
    x = rng.uniform(0, 1, (400, 2))
    xt = rng.uniform(0, 1, (20, 2))
    fa = O.efgp_fit(x[:200], np.zeros(200), c.kernel, c.ell, c.sigma, c.eps, nu=c.nu)
    fb = O.efgp_fit(x, np.zeros(400), c.kernel, c.ell, c.sigma, c.eps, nu=c.nu)
    sa = O.posterior_variance(fa, xt, cg_tol=1e-12, max_iter=20000)
    sb = O.posterior_variance(fb, xt, cg_tol=1e-12, max_iter=20000)
    k0 = float(np.sum(fb.D ** 2))
    assert np.all(sb > 0) and np.all(sa <= k0 * (1 + 1e-12))
    assert np.all(sb <= sa + 1e-12)


def test_se_variance_matches_exact_gp_within_eps():
    # SE: the (h, m) rule bounds |k~ - k| <= eps uniformly, so the tight-CG EFGP variance is within a
    # small multiple of eps of the exact GP variance (same argument as the mean)
    c = CONFIGS["c1"]
    rng = np.random.default_rng(5)
    x = rng.uniform(0, 1, (500, 1))
    xt = np.linspace(0, 1, 40)[:, None]
    fit = O.efgp_fit(x, np.zeros(500), "se", c.ell, c.sigma, c.eps)
    s = O.posterior_variance(fit, xt, cg_tol=1e-13, max_iter=50000)
    kfun = lambda a, b: O.kernel_value("se", np.abs(a[:, None, 0] - b[None, :, 0]), c.ell)
    s_ex = O.dense_gp_variance(x, xt, kfun, c.sigma)
    assert np.max(np.abs(s - s_ex)) <= 10 * c.eps
