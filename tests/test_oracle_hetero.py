"""Pins for the oracle's heteroskedastic fit (NEXT-3, reading G11).

Pinned against: the homoskedastic oracle (Toeplitz path, a different code path) when sigma_n = sigma;
the function-space mean with K~ = Phi Phi^* and S = diag(sigma_n^2) (push-through identity, exact);
the exact SE GP with per-point noise within the eps bound; and the limit of a point whose noise
grows without bound (it drops out of the fit)."""
import numpy as np
import pytest

import oracle as O
from efgp_data import CONFIGS


def test_constant_noise_reduces_to_homoskedastic():
    # S = sigma^2 I: (Phi^*Phi/sigma^2 + I) beta = Phi^*y/sigma^2 is eq "be" scaled by 1/sigma^2, so CG
    # produces the same iterates (CG is invariant under scaling A and b together)
    c = CONFIGS["c5"]
    rng = np.random.default_rng(11)
    x = rng.uniform(0, 1, (700, 2))
    y = np.sin(6 * x[:, 0]) + 0.1 * rng.standard_normal(700)
    ho = O.efgp_fit(x, y, c.kernel, c.ell, c.sigma, c.eps, nu=c.nu, cg_tol=1e-12)
    he = O.efgp_fit_hetero(x, y, np.full(700, c.sigma), c.kernel, c.ell, c.eps, nu=c.nu, cg_tol=1e-12)
    # same trajectory until roundoff decorrelates the two products (dense Phi vs Toeplitz)
    np.testing.assert_allclose(he.history[:12], ho.history[:12], rtol=1e-7)
    assert abs(he.iters - ho.iters) <= 0.02 * ho.iters + 2
    np.testing.assert_allclose(he.beta, ho.beta, rtol=0, atol=1e-9 * np.max(np.abs(ho.beta)))
    np.testing.assert_allclose(he.b * c.sigma ** 2, ho.b, rtol=1e-12, atol=1e-12 * np.max(np.abs(ho.b)))


@pytest.mark.parametrize("kernel,nu,ell,d", [("se", 0.0, 0.1, 1), ("matern", 1.5, 0.1, 2)])
def test_push_through_identity_with_per_point_noise(kernel, nu, ell, d):
    # phi(x*) (Phi^* S^-1 Phi + I)^{-1} Phi^* S^-1 y = k~(x*,X) (K~ + S)^{-1} y  (exact identity):
    # catches S vs S^-1 placement, a dropped I, or a transposed Phi
    rng = np.random.default_rng(12)
    N = 300
    x = rng.uniform(0, 1, (N, d))
    y = rng.standard_normal(N)
    sd = rng.uniform(0.05, 0.6, N)
    xt = rng.uniform(0, 1, (25, d))
    eps = 1e-4 if d == 1 else 1e-3
    fit = O.efgp_fit_hetero(x, y, sd, kernel, ell, eps, nu=nu, cg_tol=1e-13, max_iter=50000)
    mu = O.efgp_predict(fit, xt)
    kt = lambda a, b: O.kernel_tilde_matrix(a, b, fit.h, fit.m, fit.D)
    ref = O.dense_gp_mean_hetero(x, y, xt, kt, sd)
    np.testing.assert_allclose(mu, ref, rtol=0, atol=1e-8 * np.max(np.abs(ref)))


def test_se_hetero_matches_exact_gp_within_eps():
    c = CONFIGS["c1"]
    rng = np.random.default_rng(13)
    x = rng.uniform(0, 1, (400, 1))
    y = np.cos(10 * x[:, 0]) + 0.2 * rng.standard_normal(400)
    sd = np.where(x[:, 0] < 0.5, 0.1, 1.0)
    xt = np.linspace(0, 1, 50)[:, None]
    fit = O.efgp_fit_hetero(x, y, sd, "se", c.ell, c.eps, cg_tol=1e-13, max_iter=50000)
    mu = O.efgp_predict(fit, xt)
    kfun = lambda a, b: O.kernel_value("se", np.abs(a[:, None, 0] - b[None, :, 0]), c.ell)
    ref = O.dense_gp_mean_hetero(x, y, xt, kfun, sd)
    assert np.max(np.abs(mu - ref)) <= 100 * c.eps * np.max(np.abs(y))


def test_noisy_point_drops_out():
    # sigma_n -> infinity removes point n from the posterior (its weight 1/sigma_n^2 -> 0)
    rng = np.random.default_rng(14)
    x = rng.uniform(0, 1, (200, 1))
    y = rng.standard_normal(200)
    sd = rng.uniform(0.1, 0.3, 200)
    xt = rng.uniform(0, 1, (10, 1))
    sd_big = sd.copy()
    sd_big[17] = 1e7
    a = O.efgp_fit_hetero(x, y, sd_big, "se", 0.1, 1e-8, cg_tol=1e-13)
    keep = np.arange(200) != 17
    b = O.efgp_fit_hetero(x[keep], y[keep], sd[keep], "se", 0.1, 1e-8, cg_tol=1e-13)
    np.testing.assert_allclose(O.efgp_predict(a, xt), O.efgp_predict(b, xt), rtol=0, atol=1e-9)


def test_dense_and_chunked_products_agree():
    # the formed-once Phi path of efgp_fit_hetero and hetero_system_apply are the same product
    rng = np.random.default_rng(15)
    x = rng.uniform(0, 1, (500, 2))
    sd = rng.uniform(0.1, 1.0, 500)
    D = O.spectral_weights("se", 0.2, 2, 0.5, 6)
    p = rng.standard_normal(D.shape) + 1j * rng.standard_normal(D.shape)
    Phi = O.design_matrix(x, 0.5, 6, D)
    dense = p.reshape(-1) + Phi.conj().T @ np.diag(1 / sd ** 2) @ Phi @ p.reshape(-1)
    np.testing.assert_allclose(O.hetero_system_apply(x, sd, D, 0.5, 6, p, chunk=77).reshape(-1), dense,
                               rtol=1e-12, atol=1e-12 * np.max(np.abs(dense)))


@pytest.mark.parametrize("d", [1, 2])
def test_weighted_toeplitz_identity(d):
    # Phi^* S^-1 Phi = D T(v^w) D with v^w_j = sum_n sigma_n^-2 exp(-2 pi i h j.x_n) (eq "88" with
    # weights): the per-point noise keeps the Toeplitz structure (reading G11b).  Checked against the
    # dense product of the design matrix.
    rng = np.random.default_rng(16)
    N = 150
    x = rng.uniform(0, 1, (N, d))
    sd = rng.uniform(0.05, 1.0, N)
    h, m = 0.37, 4
    D = O.spectral_weights("matern", 0.3, d, h, m, 1.5)
    Phi = O.design_matrix(x, h, m, D)
    dense = Phi.conj().T @ (Phi / sd[:, None] ** 2)
    vw = O.toeplitz_vector_weighted(x, 1.0 / sd ** 2, h, m)
    T = O.toeplitz_matrix(vw, m)
    Dv = D.reshape(-1)
    np.testing.assert_allclose(Dv[:, None] * T * Dv[None, :], dense, rtol=0, atol=1e-12 * np.max(np.abs(dense)))


def test_hetero_variance_woodbury():
    # phi (Phi^* S^-1 Phi + I)^-1 phi^* = k~(x*,x*) - k~(x*,X) (K~ + S)^-1 k~(X,x*)  (Woodbury, exact)
    rng = np.random.default_rng(17)
    x = rng.uniform(0, 1, (120, 2))
    sd = rng.uniform(0.05, 0.5, 120)
    xt = rng.uniform(0, 1, (9, 2))
    fit = O.efgp_fit_hetero(x, np.zeros(120), sd, "matern", 0.2, 1e-2, nu=1.5, cg_tol=1e-12)
    s = O.posterior_variance_hetero(fit, x, sd, xt)
    kt = lambda a, b: O.kernel_tilde_matrix(a, b, fit.h, fit.m, fit.D)
    K = kt(x, x) + np.diag(sd ** 2)
    Kt = kt(xt, x)
    ref = np.array([kt(xt[i:i + 1], xt[i:i + 1])[0, 0] for i in range(9)]) - np.einsum(
        "ij,ji->i", Kt, np.linalg.solve(K, Kt.T))
    np.testing.assert_allclose(s, ref, rtol=1e-9, atol=1e-12)
    # sigma_n = sigma reduces to the homoskedastic variance
    sig = 0.1
    fit2 = O.efgp_fit_hetero(x, np.zeros(120), np.full(120, sig), "se", 0.2, 1e-6, cg_tol=1e-12)
    hom = O.efgp_fit(x, np.zeros(120), "se", 0.2, sig, 1e-6, cg_tol=1e-12)
    np.testing.assert_allclose(O.posterior_variance_hetero(fit2, x, np.full(120, sig), xt),
                               O.posterior_variance(hom, xt, cg_tol=1e-13, max_iter=50000), rtol=1e-7)
