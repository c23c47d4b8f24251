"""Pins for oracle steps O3/O4 (the type-1 sums v and F^*y) and O7 (the type-2 sum mu):
brute force, special cases and identities that a dropped term, wrong sign or index would break
(SURVEY §8(c) P3)."""
import cmath
import itertools
import math

import numpy as np
import pytest

import oracle as O


def _brute_v(x, h, K):
    """Pure-Python loops: v_j = sum_n exp(-2 pi i h j.x_n) for j in J_K (eq 88, sign G1)."""
    d = len(x[0])
    out = {}
    for j in itertools.product(range(-K, K + 1), repeat=d):
        s = 0j
        for xn in x:
            s += cmath.exp(-2j * math.pi * h * sum(jl * xl for jl, xl in zip(j, xn)))
        out[j] = s
    return out


@pytest.mark.parametrize("d", [1, 2, 3])
def test_toeplitz_vector_brute_force(d):
    rng = np.random.default_rng(d)
    x = rng.uniform(0, 1, (7, d))
    h, m = 0.63, 2
    v = O.toeplitz_vector(x, h, m)
    ref = _brute_v(x.tolist(), h, 2 * m)
    for j, val in ref.items():
        assert abs(v[tuple(jl + 2 * m for jl in j)] - val) < 1e-13


@pytest.mark.parametrize("d", [1, 2, 3])
def test_rhs_brute_force(d):
    rng = np.random.default_rng(10 + d)
    x = rng.uniform(0, 1, (6, d))
    y = rng.normal(size=6)
    h, m = 0.71, 2
    Fy = O.rhs_Fy(x, y, h, m)
    for j in itertools.product(range(-m, m + 1), repeat=d):
        s = sum(yn * cmath.exp(-2j * math.pi * h * float(np.dot(j, xn))) for xn, yn in zip(x, y))
        assert abs(Fy[tuple(jl + m for jl in j)] - s) < 1e-13


def test_v_invariants():
    rng = np.random.default_rng(0)
    x = rng.uniform(0, 1, (3000, 2))
    h, m = 0.62, 6
    v = O.toeplitz_vector(x, h, m)
    assert v[2 * m, 2 * m] == pytest.approx(3000.0, abs=1e-9)            # v_0 = N
    np.testing.assert_allclose(v[::-1, ::-1], v.conj(), atol=1e-10)        # v_{-j} = conj v_j
    # single point at x = 0 -> v_j = 1 for all j
    v1 = O.toeplitz_vector(np.zeros((1, 2)), h, m)
    np.testing.assert_allclose(v1, np.ones_like(v1), atol=0)


def test_type1_linearity_and_translation():
    # linear in the strengths; a shift delta of all points multiplies the output by
    # exp(-2 pi i h j.delta) (our sign, G1).
    rng = np.random.default_rng(5)
    x = rng.uniform(0, 0.8, (500, 2))
    y1, y2 = rng.normal(size=500), rng.normal(size=500)
    h, m = 0.55, 5
    a, b = 0.7, -1.3
    np.testing.assert_allclose(O.rhs_Fy(x, a * y1 + b * y2, h, m),
                               a * O.rhs_Fy(x, y1, h, m) + b * O.rhs_Fy(x, y2, h, m), rtol=1e-12, atol=1e-11)
    delta = np.array([0.11, 0.07])
    J = O.mode_indices(m, 2).reshape(2 * m + 1, 2 * m + 1, 2)
    phase = np.exp(-2j * np.pi * h * (J @ delta))
    np.testing.assert_allclose(O.rhs_Fy(x + delta, y1, h, m), phase * O.rhs_Fy(x, y1, h, m), rtol=1e-11, atol=1e-10)


def test_type2_type1_adjoint_identity():
    # <type2(c), s> = <c, conj type1(s)>; with Hermitian c the type-2 sum is real, so
    # sum_n s_n mu_n = Re sum_j c_j conj((F^* s)_j)^* ... = Re sum_j c_j sum_n s_n e^{+2 pi i h j.x_n}.
    rng = np.random.default_rng(9)
    x = rng.uniform(0, 1, (300, 2))
    s = rng.normal(size=300)
    h, m = 0.6, 4
    c = rng.normal(size=(2 * m + 1,) * 2) + 1j * rng.normal(size=(2 * m + 1,) * 2)
    c = 0.5 * (c + c[::-1, ::-1].conj())                      # Hermitian
    mu, imax = O.posterior_mean(c, np.ones_like(c.real), h, x, return_imag=True)
    assert imax < 1e-12                                        # real output for Hermitian coefficients
    Fs = O.rhs_Fy(x, s, h, m)                                  # sum_n s_n e^{-2 pi i h j.x_n}
    lhs = float(np.dot(s, mu))
    rhs = float(np.sum(c * Fs.conj()).real)
    assert lhs == pytest.approx(rhs, rel=1e-12)


def test_posterior_mean_brute_force():
    rng = np.random.default_rng(4)
    h, m = 0.5, 2
    beta = rng.normal(size=(5, 5)) + 1j * rng.normal(size=(5, 5))
    D = rng.uniform(0.1, 1, (5, 5))
    xt = rng.uniform(0, 1, (4, 2))
    mu = O.posterior_mean(beta, D, h, xt)
    for n in range(4):
        s = 0j
        for a in range(5):
            for b in range(5):
                s += D[a, b] * beta[a, b] * cmath.exp(2j * math.pi * h * ((a - 2) * xt[n, 0] + (b - 2) * xt[n, 1]))
        assert mu[n] == pytest.approx(s.real, abs=1e-13)


def test_grid_aligned_points_reduce_to_dft():
    # x_n = n/(2K+1), h = 1 -> the type-1 sum is a DFT of length 2K+1
    K = 6
    L = 2 * K + 1
    x = (np.arange(L) / L)[:, None]
    y = np.random.default_rng(1).normal(size=L)
    Fy = O.rhs_Fy(x, y, 1.0, K)
    dft = np.fft.fft(y)                                        # sum_n y_n exp(-2 pi i k n / L)
    np.testing.assert_allclose(Fy, dft[np.arange(-K, K + 1) % L], atol=1e-12)
