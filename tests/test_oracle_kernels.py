"""Pins for oracle step O1 (spectral densities, kernels, L2 norms) against closed forms, printed
values and independent numerical Fourier transforms."""
import math

import numpy as np
import pytest
import scipy.integrate
import scipy.special

import oracle as O


def test_se_khat_at_zero_spec_example():
    # (SE, d=1, l=0.1, xi=0) -> sqrt(2 pi) 0.1 = 0.250663   (eq Ghat at 0)
    assert O.khat("se", 0.0, 0.1, 1) == pytest.approx(0.250663, abs=1e-6)
    for d in (1, 2, 3):
        assert O.khat("se", 0.0, 0.37, d) == pytest.approx((math.sqrt(2 * math.pi) * 0.37) ** d, rel=1e-15)


def test_matern_half_1d_is_lorentzian():
    # (Matérn nu=1/2, d=1, l=1, xi=0) -> 2.0; in general 2l/(1+(2 pi l xi)^2), the
    # textbook Fourier transform of exp(-|x|/l).
    assert O.khat("matern", 0.0, 1.0, 1, 0.5) == pytest.approx(2.0, rel=1e-14)
    xi = np.linspace(0, 7, 31)
    for ell in (0.1, 0.4):
        ref = 2 * ell / (1 + (2 * math.pi * ell * xi) ** 2)
        np.testing.assert_allclose(O.khat("matern", xi, ell, 1, 0.5), ref, rtol=1e-13)


def test_matern_three_halves_1d_value_at_zero():
    # k^(0) = int k = int (1 + sqrt3 r/l) exp(-sqrt3 r/l) dr over R = 4 l / sqrt 3 (reading G2 pin)
    for ell in (0.1, 0.25):
        assert O.khat("matern", 0.0, ell, 1, 1.5) == pytest.approx(4 * ell / math.sqrt(3), rel=1e-13)


@pytest.mark.parametrize("kernel,nu", [("se", 0.0), ("matern", 0.5), ("matern", 1.5), ("matern", 2.5)])
@pytest.mark.parametrize("d", [1, 2, 3])
def test_khat_integrates_to_k0(kernel, nu, d):
    # int k^ = k(0) = 1.  This is the pin that rejects the printed Crecall
    # normalisation (reading G2), which integrates to (2 nu)^{-d/2}.
    if kernel == "matern" and nu == 0.5 and d == 3:
        pytest.skip("k^ ~ xi^-4: radial integrand ~ xi^-2, handled by the d<=2 cases and nu>1/2")
    ell = 0.1
    surface = {1: 2.0, 2: 2 * math.pi, 3: 4 * math.pi}[d]
    f = lambda s: float(O.khat(kernel, s, ell, d, nu)) * s ** (d - 1)
    tot = 0.0
    edges = [0, 0.5, 1, 2, 4, 8, 16, 32, 64, 128, 256, 1024, np.inf]
    for a, b in zip(edges[:-1], edges[1:]):
        tot += scipy.integrate.quad(f, a / ell, b / ell if np.isfinite(b) else np.inf, limit=500,
                                    epsrel=1e-12)[0]
    assert surface * tot == pytest.approx(1.0, rel=2e-7 if nu == 0.5 else 1e-9)


@pytest.mark.parametrize("d", [1, 3])
def test_matern_khat_matches_numerical_fourier_transform(d):
    # k^ equals a numerical Fourier transform of the radial kernel.
    #   d=1: k^(xi) = 2 int_0^inf k(r) cos(2 pi xi r) dr
    #   d=3: k^(xi) = (2/xi) int_0^inf k(r) sin(2 pi xi r) r dr
    nu, ell = 1.5, 0.1
    for xi in (0.3, 1.7, 4.2):
        w = 2 * math.pi * xi
        if d == 1:
            val = 2 * scipy.integrate.quad(lambda r: float(O.kernel_value("matern", np.array([r]), ell, nu)[0]),
                                           0, np.inf, weight="cos", wvar=w)[0]
        else:
            val = (2 / xi) * scipy.integrate.quad(
                lambda r: float(O.kernel_value("matern", np.array([r]), ell, nu)[0]) * r,
                0, np.inf, weight="sin", wvar=w)[0]
        assert float(O.khat("matern", xi, ell, d, nu)) == pytest.approx(val, rel=1e-8)


def test_se_khat_matches_numerical_fourier_transform_2d():
    # d=2 Hankel transform k^(xi) = 2 pi int_0^inf k(r) J0(2 pi xi r) r dr
    ell = 0.07
    for xi in (0.0, 1.3, 3.1):
        val = 2 * math.pi * scipy.integrate.quad(
            lambda r: math.exp(-0.5 * (r / ell) ** 2) * scipy.special.j0(2 * math.pi * xi * r) * r,
            0, 12 * ell, limit=400, epsabs=0, epsrel=1e-13)[0]
        assert float(O.khat("se", xi, ell, 2)) == pytest.approx(val, rel=1e-10)


def test_kernel_values_spec_examples():
    # SPEC S:38-40 and the nu=1/2 closed form exp(-r/l), nu=3/2 closed form.
    assert O.kernel_value("se", np.array([0.0]), 0.1)[0] == 1.0
    assert O.kernel_value("se", np.array([0.1]), 0.1)[0] == pytest.approx(math.exp(-0.5), rel=1e-15)
    assert O.kernel_value("matern", np.array([0.2]), 0.2, 0.5)[0] == pytest.approx(math.exp(-1), rel=1e-12)
    r = np.linspace(0, 3, 301)
    np.testing.assert_allclose(O.kernel_value("matern", r, 0.7, 0.5), np.exp(-r / 0.7), rtol=1e-12)
    z = math.sqrt(3) * r / 0.3
    np.testing.assert_allclose(O.kernel_value("matern", r, 0.3, 1.5), (1 + z) * np.exp(-z), rtol=1e-12, atol=1e-300)
    assert O.kernel_value("matern", np.array([0.0]), 0.3, 1.5)[0] == 1.0


@pytest.mark.parametrize("nu,d,ell", [(0.5, 1, 0.1), (1.5, 2, 0.1), (0.5, 2, 0.1), (0.5, 3, 0.2), (2.5, 3, 0.3)])
def test_matern_l2_norm_closed_form(nu, d, ell):
    # ||k||^2 = int k^2 = int k^^2 (Plancherel); closed form derived in DESIGN.md (G3):
    # (2 pi l^2/nu)^{d/4} Gamma(nu+d/2)/Gamma(nu) sqrt(Gamma(2nu+d/2)/Gamma(2nu+d)).
    closed = ((2 * math.pi * ell ** 2 / nu) ** (d / 4) * math.gamma(nu + d / 2) / math.gamma(nu)
              * math.sqrt(math.gamma(2 * nu + d / 2) / math.gamma(2 * nu + d)))
    assert O.kernel_l2_norm("matern", ell, d, nu) == pytest.approx(closed, rel=1e-9)


def test_l2_norm_special_values():
    # Matérn-1/2 in 1D: int exp(-2|x|/l) = l -> sqrt(l).  SE: int exp(-|x|^2/l^2) = (sqrt(pi) l)^d.
    assert O.kernel_l2_norm("matern", 0.1, 1, 0.5) == pytest.approx(math.sqrt(0.1), rel=1e-10)
    for d in (1, 2, 3):
        assert O.kernel_l2_norm("se", 0.2, d) == pytest.approx((math.sqrt(math.pi) * 0.2) ** (d / 2), rel=1e-10)
    # the printed formula (reading P) is not that norm: 2.44 at nu=3/2, d=2, l=0.1
    assert O.matern_l2_norm_printed(0.1, 2, 1.5) == pytest.approx(2.443, abs=1e-3)
