"""Pins for the NEXT-4 Kronecker preconditioner and PCG (reading G12).

Pinned against: a dense LAPACK solve with M built by np.kron (axis order, conjugation, scaling of
the factored inverse); exactness on a tensor-product point set with the separable SE density (PCG
then converges in one iteration); d = 1, where M equals the system matrix; and the plain-CG solution
of the same system (the preconditioner must not change the answer)."""
import numpy as np
import pytest

import oracle as O
from efgp_data import CONFIGS


def _fit_parts(x, kernel, ell, d, eps, nu=0.0):
    h, m = O.choose_params(kernel, ell, d, eps, nu)
    D = O.spectral_weights(kernel, ell, d, h, m, nu)
    v = O.toeplitz_vector(x, h, m)
    return h, m, D, v


@pytest.mark.parametrize("d", [2, 3])
def test_factored_inverse_matches_dense_solve(d):
    rng = np.random.default_rng(21)
    x = rng.uniform(0, 1, (300, d))
    h, m, D, v = _fit_parts(x, "matern", 0.3, d, 1e-2, nu=1.5)
    s2 = 0.04
    P = O.kron_preconditioner(v, D, s2)
    A = O.kron_factors(v, D)
    M = A[0]
    for Ai in A[1:]:
        M = np.kron(M, Ai)
    M = M + s2 * np.eye(M.shape[0])
    r = rng.standard_normal(D.shape) + 1j * rng.standard_normal(D.shape)
    z = O.kron_apply_inverse(P, r)
    np.testing.assert_allclose(z.reshape(-1), np.linalg.solve(M, r.reshape(-1)), rtol=1e-9, atol=1e-12)
    for Ai in A:                                         # Hermitian PSD factors
        np.testing.assert_allclose(Ai, Ai.conj().T, atol=1e-12 * np.max(np.abs(Ai)))
        assert np.min(np.linalg.eigvalsh(Ai)) > -1e-10 * np.max(np.abs(Ai))


def test_exact_on_tensor_grid_with_separable_kernel():
    # points = {a_p} x {b_q}: v_{j1,j2} = V1(j1) V2(j2) exactly, the SE density is separable, so
    # M = D T D + sigma^2 I and PCG stops after one iteration at the dense solution
    rng = np.random.default_rng(22)
    a, b = np.sort(rng.uniform(0, 1, 17)), np.sort(rng.uniform(0, 1, 23))
    x = np.array([(p, q) for p in a for q in b])
    y = np.sin(5 * x[:, 0]) * np.cos(3 * x[:, 1])
    fit_p = O.efgp_fit(x, y, "se", 0.2, 0.3, 1e-6, cg_tol=1e-12, precond="kron")
    assert fit_p.iters == 1
    T = O.toeplitz_matrix(fit_p.v, fit_p.m)
    Dv = fit_p.D.reshape(-1)
    A = Dv[:, None] * T * Dv[None, :] + 0.09 * np.eye(len(Dv))
    np.testing.assert_allclose(fit_p.beta.reshape(-1), np.linalg.solve(A, fit_p.b.reshape(-1)),
                               rtol=0, atol=1e-10 * np.max(np.abs(fit_p.beta)))


def test_one_dimension_is_exact():
    rng = np.random.default_rng(23)
    x = rng.uniform(0, 1, (500, 1))
    y = rng.standard_normal(500)
    c = CONFIGS["c1"]
    fit = O.efgp_fit(x, y, "se", c.ell, c.sigma, c.eps, cg_tol=1e-12, precond="kron")
    assert fit.iters == 1


@pytest.mark.parametrize("name", ["c3", "c5"])
def test_pcg_matches_cg_and_needs_fewer_iterations(name):
    c = CONFIGS[name]
    rng = np.random.default_rng(24)
    x = rng.uniform(0, 1, (3000, 2))
    y = np.sin(6 * x[:, 0]) * np.cos(4 * x[:, 1]) + c.sigma * rng.standard_normal(3000)
    ref = O.efgp_fit(x, y, c.kernel, c.ell, c.sigma, c.eps, nu=c.nu, cg_tol=1e-11)
    pre = O.efgp_fit(x, y, c.kernel, c.ell, c.sigma, c.eps, nu=c.nu, cg_tol=1e-11, precond="kron")
    np.testing.assert_allclose(pre.beta, ref.beta, rtol=0, atol=1e-8 * np.max(np.abs(ref.beta)))
    assert pre.iters < ref.iters / 2, (pre.iters, ref.iters)


@pytest.mark.parametrize("d", [1, 2])
def test_jacobi_diagonal_is_the_dense_diagonal(d):
    # reading G12b: diag(D T D + sigma^2 I) = D^2 v_0 + sigma^2 (T_jj = v_0 = N)
    rng = np.random.default_rng(40 + d)
    x = rng.uniform(0, 1, (400, d))
    h, m, D, v = _fit_parts(x, "matern", 0.2, d, 1e-3, nu=1.5)
    T = O.toeplitz_matrix(v, m)
    Dv = D.reshape(-1)
    A = Dv[:, None] * T * Dv[None, :] + 0.01 * np.eye(len(Dv))
    np.testing.assert_allclose(O.jacobi_diagonal(v, D, 0.01).reshape(-1), np.diag(A).real, rtol=1e-12)
    assert abs(v[(2 * m,) * d] - 400) < 1e-9


@pytest.mark.parametrize("name", ["c2", "c5"])
def test_jacobi_pcg_matches_cg_with_fewer_iterations(name):
    # at the practical tolerance eps/10 the Jacobi PCG needs fewer iterations than CG and lands at least as
    # close to the converged mean; converged (1e-11) both give the same mean and the same variances
    c = CONFIGS[name]
    rng = np.random.default_rng(41)
    x = rng.uniform(0, 1, (4000, 2))
    y = np.sin(6 * x[:, 0]) * np.cos(4 * x[:, 1]) + c.sigma * rng.standard_normal(4000)
    kw = dict(h=O.choose_params(c.kernel, c.ell, 2, c.eps, c.nu)[0], m=15) if name == "c2" else {}
    xs = rng.uniform(0, 1, (50, 2))
    conv_fit = O.efgp_fit(x, y, c.kernel, c.ell, c.sigma, c.eps, nu=c.nu, cg_tol=1e-11, max_iter=100000, **kw)
    conv = O.efgp_predict(conv_fit, xs)
    ref = O.efgp_fit(x, y, c.kernel, c.ell, c.sigma, c.eps, nu=c.nu, cg_tol=c.eps / 10, **kw)
    pre = O.efgp_fit(x, y, c.kernel, c.ell, c.sigma, c.eps, nu=c.nu, cg_tol=c.eps / 10, precond="jacobi", **kw)
    assert pre.iters < ref.iters, (pre.iters, ref.iters)
    e_ref = np.linalg.norm(O.efgp_predict(ref, xs) - conv) / np.linalg.norm(conv)
    e_pre = np.linalg.norm(O.efgp_predict(pre, xs) - conv) / np.linalg.norm(conv)
    assert e_pre <= 2 * e_ref + 10 * c.eps, (e_pre, e_ref)
    pre_c = O.efgp_fit(x, y, c.kernel, c.ell, c.sigma, c.eps, nu=c.nu, cg_tol=1e-11, max_iter=100000,
                       precond="jacobi", **kw)
    assert np.linalg.norm(O.efgp_predict(pre_c, xs) - conv) <= 1e-6 * np.linalg.norm(conv)
    xt = rng.uniform(0, 1, (3, 2))
    s0 = O.posterior_variance(conv_fit, xt, cg_tol=1e-11, max_iter=100000)
    s1 = O.posterior_variance(conv_fit, xt, cg_tol=1e-11, max_iter=100000, precond="jacobi")
    np.testing.assert_allclose(s1, s0, rtol=1e-6)
