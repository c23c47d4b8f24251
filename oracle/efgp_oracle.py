"""EFGP oracle: a plain, slow, obviously correct CPU implementation of the EFGP hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.  It shares no code with the
CUDA path in ``paper_2210_10210_b200`` and imports nothing from it.

Everything is numpy/scipy in fp64 (complex128 for Fourier sums).  EFGP is an approximation plus
an iteration, so the oracle follows Algorithm ``a1`` step by step, with every
fast transform replaced by the sum that defines it:

  step 1  (h, m) rules ........ :func:`choose_params_se` (Cor ``c:SEparams``),
                                 :func:`choose_params_matern` (Remark ``r:heur`` eqs ``mheur``/``hheur``,
                                 P:1305-1337, with the §7.1 eps rescaling P:1982-1990, reading A)
  step 2  v_j ................. :func:`toeplitz_vector`   direct sum, eq ``88``, sign G1
  step 3  Phi^* y ............. :func:`rhs`               direct sum, eqs ``rhs``/``97``
  step 4  CG .................. :func:`cg` on :func:`system_apply`; Toeplitz product by direct
                                 convolution, CG as P:895-901, P:1973-1974;
                                 c4 only: :func:`toeplitz_apply_fft` (host pocketfft, reading G11)
  step 5/6 mu(x*) ............. :func:`posterior_mean`    direct sum, eq ``muws``
  NEXT-2  s(x*) ............... :func:`posterior_variance` one CG per target on eq ``eta``
                                 (P:571-575), then the direct sum of eq ``sws``
  NEXT-4  preconditioner ...... :func:`kron_preconditioner` + :func:`pcg` (reading G12):
                                 M = A_1 (x) ... (x) A_d + sigma^2 I from the axis lines of v and D
  NEXT-3  sigma_n ............. :func:`efgp_fit_hetero` CG on (Phi^* S^-1 Phi + I) beta = Phi^* S^-1 y,
                                 S = diag(sigma_n^2) (reading G11), Phi applied densely;
                                 :func:`toeplitz_vector_weighted` (reading G11b: Phi^* S^-1 Phi =
                                 D T(v^w) D); :func:`posterior_variance_hetero` (dense solve)

Readings where the paper is silent, garbled or inconsistent:
  G1  exponent signs: v_j = sum_n exp(-2 pi i h j.x_n), (F^*y)_j = sum_n exp(-2 pi i h j.x_n) y_n,
      mu(x) = Re sum_j D_j beta_j exp(+2 pi i h j.x).  (Phi_{n,p} = D_p exp(+2 pi i h j_p.x_n).)
  G2  Matérn spectral density uses l^d, not (l/sqrt(2 nu))^d as printed in ``Crecall``.
  G3  Matérn eps rescaling by the true ||k||_{L2(R^d)} (reading A); alternatives B (none), P (printed).
  G4  SE (h, m): Cor c:SEparams literally; h rounded down at the 12th significant digit.
  G6  CG: x0 = 0, unpreconditioned, recursive residual, Hermitian inner products.
  G11 (c4 Toeplitz product): the direct O(M^2) product is too slow at M = 4.2e5, so the oracle may use
      an independent host FFT (scipy/pocketfft, never cuFFT), validated against the direct product.
  G12 NEXT-4 preconditioner (P:2741-2745 names "Kronecker-structure Toeplitz preconditioners" only):
      v^(i)_l = v_{l e_i}, T_i = T(v^(i)) ((2m+1)^2 Toeplitz), delta_i(j) = D_{j e_i} / D_0^((d-1)/d),
      A_i = diag(delta_i) T_i diag(delta_i) / N^((d-1)/d), M = A_1 (x) ... (x) A_d + sigma^2 I, applied as
      (Q_1 (x) ... ) (Lambda + sigma^2)^-1 (Q_1 (x) ...)^* from eigh(A_i).  Exact (M = A) when the points
      form a tensor-product set and D is separable (SE); d = 1 gives M = A.  Standard PCG, same stop rule.
  G12b Jacobi preconditioner: diag(D T D + sigma^2 I) = D^2 v_0 + sigma^2 (pinned against the dense diagonal).
  G11b Phi^* S^-1 Phi = D T(v^w) D with v^w = eq 88 with strengths sigma_n^-2 (pinned densely).
  G11 heteroskedastic noise (P:2759-2763 names it, gives no formula): the weight-space posterior mean
      for y = Phi beta + e, beta ~ N(0, I), e ~ N(0, S), S = diag(sigma_n^2): beta solves
      (Phi^* S^-1 Phi + I) beta = Phi^* S^-1 y, mu(x*) = phi(x*) beta.  With sigma_n = sigma it is
      eq ``be`` divided by sigma^2 (same CG iterates); CG cap P:1766 with sigma = min sigma_n.

Pins: tests/test_oracle_*.py check every function against closed forms, printed values, invariants
and brute force.  Nothing here is "parity unpinned".
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field

import numpy as np
import scipy.fft
import scipy.integrate
import scipy.linalg
import scipy.special

__all__ = [
    "khat", "kernel_value", "kernel_l2_norm", "matern_l2_norm_printed",
    "round_down_sig", "choose_params_se", "choose_params_matern", "choose_params",
    "mode_indices", "spectral_weights", "toeplitz_vector", "toeplitz_vector_weighted", "rhs_Fy", "rhs",
    "toeplitz_matrix", "toeplitz_apply", "toeplitz_apply_fft", "system_apply", "cg", "default_max_iter",
    "posterior_mean", "posterior_variance", "design_matrix", "kernel_tilde_matrix", "dense_gp_mean",
    "dense_gp_variance", "features", "hetero_system_apply", "KronPrecond", "kron_factors",
    "kron_preconditioner", "kron_apply_inverse", "pcg", "posterior_variance_hetero", "jacobi_diagonal", "efgp_fit_hetero", "dense_gp_mean_hetero",
    "OracleFit", "efgp_fit", "efgp_predict",
]

TWO_PI = 2.0 * math.pi


# ----------------------------------------------------------------------------------------------
# Kernels and spectral densities
# ----------------------------------------------------------------------------------------------
def khat(kernel: str, xi_norm, ell: float, d: int, nu: float = 0.0):
    """Spectral density k^(xi) at |xi| = xi_norm, Fourier convention of P:674-681.

    SE   : (sqrt(2 pi) l)^d exp(-2 |pi l xi|^2)                         eq ``Ghat`` P:2812
    Matérn: c_{d,nu} l^d (2 nu + |2 pi l xi|^2)^(-nu-d/2),              eq ``Crecall`` P:2936
            c_{d,nu} = 2^d pi^{d/2} (2 nu)^nu Gamma(nu+d/2)/Gamma(nu)   eq ``hatc``
    Reading G2: the factor is l^d (the printed (l/sqrt(2nu))^d gives int k^ = (2nu)^{-d/2} != k(0)=1).
    """
    xi = np.asarray(xi_norm, dtype=np.float64)
    if kernel == "se":
        return (math.sqrt(TWO_PI) * ell) ** d * np.exp(-2.0 * (math.pi * ell * xi) ** 2)
    if kernel == "matern":
        log_c = (d * math.log(2.0) + 0.5 * d * math.log(math.pi) + nu * math.log(2.0 * nu)
                 + math.lgamma(nu + 0.5 * d) - math.lgamma(nu))
        return math.exp(log_c) * ell ** d * (2.0 * nu + (TWO_PI * ell * xi) ** 2) ** (-nu - 0.5 * d)
    raise ValueError(f"unknown kernel {kernel!r}")


def kernel_value(kernel: str, r, ell: float, nu: float = 0.0):
    """k(r), unit variance.  SE eq ``Gker``; Matérn eq ``Cker``, k(0) = 1."""
    r = np.asarray(r, dtype=np.float64)
    if kernel == "se":
        return np.exp(-0.5 * (r / ell) ** 2)
    if kernel == "matern":
        z = math.sqrt(2.0 * nu) * r / ell
        out = np.ones_like(z)
        pos = z > 1e-12
        zp = z[pos]
        out[pos] = (2.0 ** (1.0 - nu) / math.gamma(nu)) * zp ** nu * scipy.special.kv(nu, zp)
        return out
    raise ValueError(f"unknown kernel {kernel!r}")


def kernel_l2_norm(kernel: str, ell: float, d: int, nu: float = 0.0) -> float:
    """||k||_{L2(R^d)} by its definition (int k(x)^2 dx)^(1/2), as radial quadrature.

    This is the norm the §7.1 eps rescaling names (reading G3-A).  Pinned in tests
    against the closed form (2 pi l^2/nu)^{d/4} Gamma(nu+d/2)/Gamma(nu) sqrt(Gamma(2nu+d/2)/Gamma(2nu+d)).
    """
    surface = {1: 2.0, 2: TWO_PI, 3: 4.0 * math.pi}[d]      # |S^{d-1}|
    f = lambda r: float(kernel_value(kernel, np.array([r]), ell, nu)[0]) ** 2 * r ** (d - 1)
    total = 0.0
    # integrate in pieces of one length scale; tails decay at least exponentially
    edges = [0.0] + [ell * t for t in (0.5, 1, 2, 4, 8, 16, 32, 64, 128)]
    for a, b in zip(edges[:-1], edges[1:]):
        val, _ = scipy.integrate.quad(f, a, b, epsabs=0.0, epsrel=1e-13, limit=400)
        total += val
    return math.sqrt(surface * total)


def matern_l2_norm_printed(ell: float, d: int, nu: float) -> float:
    """The norm formula exactly as printed at P:1985-1986 (reading G3-P; NOT ||k||_{L2})."""
    return ((nu / (math.pi * ell ** 2)) ** (d / 4.0)
            * math.sqrt(math.gamma(d / 2.0 + 2 * nu) / (2.0 * math.gamma(d + 2 * nu))))


# ----------------------------------------------------------------------------------------------
# Step 1: discretisation parameters (h, m)
# ----------------------------------------------------------------------------------------------
def round_down_sig(x: float, digits: int = 12) -> float:
    """Round a positive x toward zero at its `digits`-th significant digit."""
    e = math.floor(math.log10(x))
    scale = 10.0 ** (digits - 1 - e)
    return math.floor(x * scale) / scale


def choose_params_se(ell: float, d: int, eps: float):
    """Cor ``c:SEparams``:  h <= (1 + l sqrt(2 log(4 d 3^d/eps)))^-1,
    m >= sqrt(1/2 log(4^{d+1} d/eps)) / (pi l h).  Reading G4: equality, h rounded down, m = ceil."""
    h = 1.0 / (1.0 + ell * math.sqrt(2.0 * math.log(4.0 * d * 3.0 ** d / eps)))
    h = round_down_sig(h)
    m = math.ceil(math.sqrt(0.5 * math.log(4.0 ** (d + 1) * d / eps)) / (math.pi * ell * h))
    return h, int(m)


def choose_params_matern(nu: float, ell: float, d: int, eps: float, rescale: str = "A"):
    """Remark ``r:heur``: h = (1 + 0.85 (l/sqrt nu) log 1/eps)^-1 (eq ``hheur``),
    m = (1/h) (pi^{nu+d/2} l^{2nu} eps/0.15)^{-1/(2nu+d/2)} (eq ``mheur``), after the §7.1 rescaling
    eps <- eps * ||k||_{L2}.  rescale: "A" true norm (default), "B" none, "P" printed."""
    if rescale == "A":
        eps_eff = eps * kernel_l2_norm("matern", ell, d, nu)
    elif rescale == "B":
        eps_eff = eps
    elif rescale == "P":
        eps_eff = eps * matern_l2_norm_printed(ell, d, nu)
    else:
        raise ValueError(rescale)
    h = 1.0 / (1.0 + 0.85 * (ell / math.sqrt(nu)) * math.log(1.0 / eps_eff))
    h = round_down_sig(h)
    m = math.ceil((1.0 / h) * (math.pi ** (nu + d / 2.0) * ell ** (2 * nu) * eps_eff / 0.15)
                  ** (-1.0 / (2 * nu + d / 2.0)))
    return h, int(m)


def choose_params(kernel: str, ell: float, d: int, eps: float, nu: float = 0.0, rescale: str = "A"):
    if kernel == "se":
        return choose_params_se(ell, d, eps)
    return choose_params_matern(nu, ell, d, eps, rescale)


def mode_indices(m: int, d: int) -> np.ndarray:
    """J_m = {-m..m}^d as an (M, d) int array, row-major with the last coordinate fastest
    (enumeration S:82)."""
    return np.array(list(itertools.product(range(-m, m + 1), repeat=d)), dtype=np.int64).reshape(-1, d)


def spectral_weights(kernel: str, ell: float, d: int, h: float, m: int, nu: float = 0.0) -> np.ndarray:
    """Diagonal D_j = sqrt(h^d k^(h |j|)), j in J_m (eq ``117``), shape (2m+1,)*d."""
    J = mode_indices(m, d)
    D = np.sqrt(h ** d * khat(kernel, h * np.linalg.norm(J, axis=1), ell, d, nu))
    return D.reshape((2 * m + 1,) * d)


# ----------------------------------------------------------------------------------------------
# Steps 2-3: the two type-1 sums, written out (no NUFFT)
# ----------------------------------------------------------------------------------------------
def _phase_factors(xcol: np.ndarray, h: float, K: int) -> np.ndarray:
    """E[n, a] = exp(-2 pi i h j x_n) for j = a - K, a = 0..2K (one coordinate)."""
    j = np.arange(-K, K + 1, dtype=np.float64)
    return np.exp(-1j * TWO_PI * h * np.outer(xcol, j))


def _signed_sum(x: np.ndarray, weights: np.ndarray | None, h: float, K: int, chunk: int = 1 << 15):
    """S_j = sum_n w_n exp(-2 pi i h j . x_n) for j in J_K, as a (2K+1,)*d complex array.

    exp(-2 pi i h j.x) = prod_l exp(-2 pi i h j_l x_l), so for d = 2 the sum over n is the matrix
    product E1^T diag(w) E2 (a library matmul serving as the sum, no other reordering)."""
    x = np.asarray(x, dtype=np.float64)
    N, d = x.shape
    S = np.zeros((2 * K + 1,) * d, dtype=np.complex128)
    for s in range(0, N, chunk):
        xs = x[s:s + chunk]
        w = np.ones(len(xs)) if weights is None else np.asarray(weights[s:s + chunk], dtype=np.float64)
        E = [_phase_factors(xs[:, l], h, K) for l in range(d)]
        if d == 1:
            S += w @ E[0]
        elif d == 2:
            S += (E[0] * w[:, None]).T @ E[1]
        elif d == 3:
            E0w = E[0] * w[:, None]
            for a in range(2 * K + 1):
                S[a] += (E0w[:, a, None] * E[1]).T @ E[2]
        else:
            raise ValueError("d must be 1, 2 or 3")
    return S


def toeplitz_vector(x: np.ndarray, h: float, m: int) -> np.ndarray:
    """v_j = sum_n exp(-2 pi i h j.x_n), j in J_{2m}  (eq ``88``; sign reading G1).
    Returned as a (4m+1,)*d array indexed by j + 2m."""
    return _signed_sum(x, None, h, 2 * m)


def toeplitz_vector_weighted(x: np.ndarray, w: np.ndarray, h: float, m: int) -> np.ndarray:
    """v^w_j = sum_n w_n exp(-2 pi i h j.x_n), j in J_{2m}: eq ``88`` with per-point weights (reading
    G11b: with w_n = sigma_n^-2, Phi^* S^-1 Phi = D T(v^w) D).  Returned indexed by j + 2m."""
    return _signed_sum(x, w, h, 2 * m)


def rhs_Fy(x: np.ndarray, y: np.ndarray, h: float, m: int) -> np.ndarray:
    """(F^* y)_j = sum_n exp(-2 pi i h j.x_n) y_n, j in J_m  (eq ``rhs``; sign G1)."""
    return _signed_sum(x, y, h, m)


def rhs(x, y, h, m, D) -> np.ndarray:
    """Right-hand side Phi^* y = D F^* y."""
    return D * rhs_Fy(x, y, h, m)


# ----------------------------------------------------------------------------------------------
# Step 4: Toeplitz product and CG
# ----------------------------------------------------------------------------------------------
def toeplitz_matrix(v: np.ndarray, m: int) -> np.ndarray:
    """Dense T with T_{p,q} = v_{j_p - j_q}  (eq ``223``: (F^*F)_{p,l} depends on j_p - j_l only)."""
    d = v.ndim
    J = mode_indices(m, d)
    diff = J[:, None, :] - J[None, :, :] + 2 * m          # index into v
    return v[tuple(diff[..., l] for l in range(d))]


def toeplitz_apply(v: np.ndarray, beta: np.ndarray, T: np.ndarray | None = None) -> np.ndarray:
    """(T beta)_p = sum_{q in J_m} v_{p-q} beta_q, p in J_m, computed directly.

    With T given: dense product.  Otherwise the same sum as a loop over q: for each q the term
    beta_q v_{p-q} over all p is the slice of v starting at index 2m - (q + m) in each axis."""
    m = (beta.shape[0] - 1) // 2
    if T is not None:
        return (T @ beta.reshape(-1)).reshape(beta.shape)
    d = beta.ndim
    out = np.zeros_like(beta, dtype=np.complex128)
    n = 2 * m + 1
    for b in itertools.product(range(n), repeat=d):
        sl = tuple(slice(2 * m - bl, 4 * m - bl + 1) for bl in b)
        out += beta[b] * v[sl]
    return out


def _prime_factors(n: int):
    out, f = [], 2
    while f * f <= n:
        while n % f == 0:
            out.append(f)
            n //= f
        f += 1
    return out + ([n] if n > 1 else [])


def toeplitz_apply_fft(v: np.ndarray, beta: np.ndarray) -> np.ndarray:
    """(T beta)_p = sum_{q in J_m} v_{p-q} beta_q by a host FFT (scipy's pocketfft), reading G11: the
    one allowed exception to the direct product, for c4 only (M = 4.2e5 makes the direct O(M^2)
    product ~1.8e11 MACs).  It is Alg ``a:FF`` written with complex FFTs of length
    L >= 4m+1 per axis (the smallest 2^a 3^b 5^c, so pocketfft avoids Bluestein for prime 4m+1): v_j
    is placed at index j mod L, beta_q at q + m (zero-padded); the circular convolution at index p + m
    equals the linear one because |p - q| <= 2m < L (no wrap-around).  Pinned against
    :func:`toeplitz_apply` (full at small m, sampled outputs at c4's m)."""
    d = beta.ndim
    m = (beta.shape[0] - 1) // 2
    L = 4 * m + 1
    while any(f > 5 for f in _prime_factors(L)):
        L += 1
    vb = np.zeros((L,) * d, dtype=np.complex128)
    idx = np.arange(-2 * m, 2 * m + 1) % L
    vb[np.ix_(*([idx] * d))] = v
    bb = np.zeros((L,) * d, dtype=np.complex128)
    bb[(slice(0, 2 * m + 1),) * d] = beta
    c = scipy.fft.ifftn(scipy.fft.fftn(vb, workers=-1) * scipy.fft.fftn(bb, workers=-1), workers=-1)
    return c[(slice(0, 2 * m + 1),) * d]       # index p + m, p in J_m


def system_apply(v, D, sigma2, beta, T=None, fft=False):
    """(Phi^*Phi + sigma^2 I) beta = D (F^*F) (D beta) + sigma^2 beta   (eq ``97``, P:766-768,
    the three steps of P:846-848).  fft=True: the Toeplitz product by :func:`toeplitz_apply_fft`
    (reading G11, c4 only)."""
    if fft:
        return D * toeplitz_apply_fft(v, D * beta) + sigma2 * beta
    return D * toeplitz_apply(v, D * beta, T) + sigma2 * beta


def default_max_iter(N: int, sigma: float, tol: float) -> int:
    """k <= log(1/eps) sqrt(N) / (2 sigma), used as the CG cap."""
    return max(10, int(math.ceil(math.log(1.0 / tol) * math.sqrt(N) / (2.0 * sigma))))


def cg(apply, b: np.ndarray, tol: float, max_iter: int):
    """Plain (unpreconditioned) conjugate gradients on the Hermitian positive definite system
    (stopping at relative residual tol; Golub & Van Loan §10.2 as cited at
    P:1758).  x0 = 0; recursive residual; Hermitian inner products (reading G6).

    Returns (x, iters, history) with history[k] = ||r_k|| / ||b|| for k = 0..iters, and iters the
    first k with history[k] <= tol (or max_iter)."""
    x = np.zeros_like(b, dtype=np.complex128)
    r = b.astype(np.complex128).copy()
    bnorm = math.sqrt(np.vdot(b, b).real)
    if bnorm == 0.0:
        return x, 0, [0.0]
    p = r.copy()
    rr = np.vdot(r, r).real
    hist = [math.sqrt(rr) / bnorm]
    k = 0
    while hist[-1] > tol and k < max_iter:
        Ap = apply(p)
        alpha = rr / np.vdot(p, Ap).real
        x = x + alpha * p
        r = r - alpha * Ap
        rr_new = np.vdot(r, r).real
        p = r + (rr_new / rr) * p
        rr = rr_new
        k += 1
        hist.append(math.sqrt(rr) / bnorm)
    return x, k, hist


# ----------------------------------------------------------------------------------------------
# NEXT-4: Kronecker preconditioner (reading G12) and preconditioned CG
# ----------------------------------------------------------------------------------------------
@dataclass
class KronPrecond:
    Q: list      # eigenvectors of A_i, (2m+1, 2m+1) each
    lam: list    # eigenvalues of A_i
    sigma2: float


def kron_factors(v: np.ndarray, D: np.ndarray):
    """The factors A_i = diag(delta_i) T(v^(i)) diag(delta_i) / N^((d-1)/d) of reading G12, where
    v^(i)_l = v_{l e_i} (the line of v through j = 0 along axis i), delta_i(j) = D_{j e_i} / D_0^((d-1)/d)
    and N = v_0 (eq ``88`` at j = 0)."""
    d = D.ndim
    m = (D.shape[0] - 1) // 2
    N = float(v[(2 * m,) * d].real)
    D0 = float(D[(m,) * d])
    out = []
    for i in range(d):
        line_v = [2 * m] * d
        line_v[i] = slice(None)
        vi = v[tuple(line_v)]                                   # l = -2m..2m
        line_d = [m] * d
        line_d[i] = slice(None)
        di = D[tuple(line_d)] / D0 ** ((d - 1) / d)
        p = np.arange(2 * m + 1)
        Ti = vi[p[:, None] - p[None, :] + 2 * m]                 # T_pq = v^(i)_{p-q}
        out.append(di[:, None] * Ti * di[None, :] / N ** ((d - 1) / d))
    return out


def kron_preconditioner(v: np.ndarray, D: np.ndarray, sigma2: float) -> KronPrecond:
    """M = A_1 (x) ... (x) A_d + sigma^2 I (reading G12), factored by numpy.linalg.eigh of each A_i."""
    Q, lam = [], []
    for A in kron_factors(v, D):
        w, V = np.linalg.eigh(A)
        Q.append(V)
        lam.append(w)
    return KronPrecond(Q, lam, sigma2)


def kron_apply_inverse(P: KronPrecond, r: np.ndarray) -> np.ndarray:
    """M^-1 r = (Q_1 (x) ... ) (Lambda_1 (x) ... + sigma^2)^-1 (Q_1 (x) ...)^* r, one axis at a time."""
    z = np.asarray(r, dtype=np.complex128)
    for i, Q in enumerate(P.Q):
        z = np.moveaxis(np.tensordot(Q.conj().T, np.moveaxis(z, i, 0), axes=1), 0, i)
    lam = P.lam[0]
    for w in P.lam[1:]:
        lam = np.multiply.outer(lam, w)
    z = z / (lam + P.sigma2)
    for i, Q in enumerate(P.Q):
        z = np.moveaxis(np.tensordot(Q, np.moveaxis(z, i, 0), axes=1), 0, i)
    return z


def jacobi_diagonal(v: np.ndarray, D: np.ndarray, sigma2: float) -> np.ndarray:
    """diag(D T D + sigma^2 I) = D_j^2 v_0 + sigma^2 (T_jj = v_0 = N, eq ``88`` at j = 0): the Jacobi
    preconditioner of reading G12b."""
    d = D.ndim
    m = (D.shape[0] - 1) // 2
    return D ** 2 * float(v[(2 * m,) * d].real) + sigma2


def pcg(apply, precond, b: np.ndarray, tol: float, max_iter: int):
    """Preconditioned CG (Golub & Van Loan Alg 11.5.1, the standard recurrences), x0 = 0, stopping
    at the first k with ||r_k|| <= tol ||b|| (the same rule as :func:`cg`, reading G6).
    Returns (x, iters, history of ||r_k|| / ||b||)."""
    x = np.zeros_like(b, dtype=np.complex128)
    r = b.astype(np.complex128).copy()
    bnorm = math.sqrt(np.vdot(b, b).real)
    if bnorm == 0.0:
        return x, 0, [0.0]
    z = precond(r)
    p = z.copy()
    rz = np.vdot(r, z).real
    hist = [1.0]
    k = 0
    while hist[-1] > tol and k < max_iter:
        Ap = apply(p)
        alpha = rz / np.vdot(p, Ap).real
        x = x + alpha * p
        r = r - alpha * Ap
        k += 1
        hist.append(math.sqrt(np.vdot(r, r).real) / bnorm)
        if hist[-1] <= tol:
            break
        z = precond(r)
        rz_new = np.vdot(r, z).real
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, k, hist


# ----------------------------------------------------------------------------------------------
# Steps 5-6: posterior mean at targets
# ----------------------------------------------------------------------------------------------
def posterior_mean(beta, D, h, xt, chunk: int = 1 << 14, return_imag: bool = False):
    """mu(x*) = sum_j beta_j phi_j(x*) = sum_j D_j beta_j exp(+2 pi i h j.x*)  (eq ``muws`` P:557,
    basis eq ``basis`` P:707), evaluated directly; the real part is returned (the exact value is
    real).  Optionally also max |Im|."""
    xt = np.asarray(xt, dtype=np.float64)
    q, d = xt.shape
    m = (beta.shape[0] - 1) // 2
    c = D * beta
    mu = np.empty(q)
    imax = 0.0
    j = np.arange(-m, m + 1, dtype=np.float64)
    for s in range(0, q, chunk):
        xs = xt[s:s + chunk]
        E = [np.exp(+1j * TWO_PI * h * np.outer(xs[:, l], j)) for l in range(d)]
        if d == 1:
            val = E[0] @ c
        elif d == 2:
            val = np.einsum("na,nb,ab->n", E[0], E[1], c, optimize=True)
        else:
            val = np.einsum("na,nb,nc,abc->n", E[0], E[1], E[2], c, optimize=True)
        mu[s:s + chunk] = val.real
        imax = max(imax, float(np.max(np.abs(val.imag))) if len(val) else 0.0)
    return (mu, imax) if return_imag else mu


def features(D, h, xt) -> np.ndarray:
    """phi_j(x*) = D_j exp(+2 pi i h j.x*) over J_m, shape (q,) + D.shape  (eq ``basis`` P:707)."""
    xt = np.asarray(xt, dtype=np.float64)
    d = D.ndim
    m = (D.shape[0] - 1) // 2
    j = np.arange(-m, m + 1, dtype=np.float64)
    E = [np.exp(+1j * TWO_PI * h * np.outer(xt[:, l], j)) for l in range(d)]
    if d == 1:
        P = E[0]
    elif d == 2:
        P = E[0][:, :, None] * E[1][:, None, :]
    else:
        P = E[0][:, :, None, None] * E[1][:, None, :, None] * E[2][:, None, None, :]
    return D[None] * P


def posterior_variance(fit, xt, cg_tol: float | None = None, max_iter: int | None = None,
                       return_iters: bool = False, precond: str | None = None):
    """s(x*) = sum_j eta_j phi_j(x*)  (eq ``sws``) where, per target,
    (Phi^*Phi + sigma^2 I) eta = sigma^2 conj(phi(x*))  (eq ``eta``), solved by the same
    plain CG and system_apply as the mean ("a new right-hand side ... per target").
    The exact value is real; the real part is returned."""
    xt = np.asarray(xt, dtype=np.float64)
    if xt.ndim == 1:
        xt = xt[:, None]
    s2 = fit.sigma ** 2
    tol = fit.eps if cg_tol is None else cg_tol
    cap = default_max_iter(max(1, int(round(fit.v[(2 * fit.m,) * fit.d].real))), fit.sigma, tol) \
        if max_iter is None else max_iter
    T = toeplitz_matrix(fit.v, fit.m) if fit.M <= 4096 else None
    Phi = features(fit.D, fit.h, xt)
    out = np.empty(len(xt))
    iters = []
    for t in range(len(xt)):
        A = lambda p: system_apply(fit.v, fit.D, s2, p, T)
        if precond == "jacobi":
            dg = jacobi_diagonal(fit.v, fit.D, s2)
            eta, k, _ = pcg(A, lambda r: r / dg, s2 * np.conj(Phi[t]), tol, cap)
        else:
            eta, k, _ = cg(A, s2 * np.conj(Phi[t]), tol, cap)
        out[t] = np.sum(eta * Phi[t]).real
        iters.append(k)
    return (out, iters) if return_iters else out


def hetero_system_apply(x, noise_sd, D, h, m, p, chunk: int = 4096):
    """(Phi^* S^-1 Phi + I) p with S = diag(noise_sd^2) (reading G11), Phi_{n,j} = D_j exp(+2 pi i h
    j.x_n) (eq ``205``).  Applied as written: a type-2 sum u = Phi p at the points (P:557's sum at the
    data points), u / sigma_n^2, then the type-1 sum Phi^* (P:855-862), the BBMM-style product of
    P:2761-2763; Phi rows are formed chunk by chunk (dense, no fast transform)."""
    x = np.asarray(x, dtype=np.float64)
    pv = np.asarray(p).reshape(-1)
    out = pv.astype(np.complex128).copy()
    for s in range(0, len(x), chunk):
        Phi = design_matrix(x[s:s + chunk], h, m, D)
        u = Phi @ pv
        out += Phi.conj().T @ (u / np.asarray(noise_sd[s:s + chunk], dtype=np.float64) ** 2)
    return out.reshape(np.shape(p))


def efgp_fit_hetero(x, y, noise_sd, kernel: str, ell: float, eps: float, nu: float = 0.0,
                    h: float | None = None, m: int | None = None, cg_tol: float | None = None,
                    max_iter: int | None = None, rescale: str = "A") -> OracleFit:
    """NEXT-3 (reading G11): per-point noise sigma_n.  Step 1 as Alg a1; right-hand side
    Phi^* S^-1 y = D F^*(y / sigma_n^2) (eq ``rhs`` with weights y_n / sigma_n^2); CG on
    hetero_system_apply.  The returned fit's sigma is min sigma_n (used only for the CG cap) and v is
    None (there is no Toeplitz vector: the structure is gone)."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    N, d = x.shape
    sd = np.asarray(noise_sd, dtype=np.float64)
    if h is None or m is None:
        h0, m0 = choose_params(kernel, ell, d, eps, nu, rescale)
        h = h0 if h is None else h
        m = m0 if m is None else m
    D = spectral_weights(kernel, ell, d, h, m, nu)
    b = rhs(x, np.asarray(y, dtype=np.float64) / sd ** 2, h, m, D)
    tol = eps if cg_tol is None else cg_tol
    smin = float(np.min(sd))
    cap = default_max_iter(N, smin, tol) if max_iter is None else max_iter
    if N * D.size <= 10_000_000:  # small enough to keep Phi: the same product, formed once
        Phi = design_matrix(x, h, m, D)
        apply = lambda p: (p.reshape(-1) + Phi.conj().T @ ((Phi @ p.reshape(-1)) / sd ** 2)).reshape(p.shape)
    else:
        apply = lambda p: hetero_system_apply(x, sd, D, h, m, p)
    beta, iters, hist = cg(apply, b, tol, cap)
    return OracleFit(kernel, nu, ell, smin, eps, d, h, m, D, None, b, beta, iters, hist)


def posterior_variance_hetero(fit: OracleFit, x, noise_sd, xt) -> np.ndarray:
    """Heteroskedastic posterior variance (reading G11 with eq ``eta`` / ``sws``, sigma^2 -> 1):
    s(x*) = phi(x*) (Phi^* S^-1 Phi + I)^-1 phi(x*)^*, by a dense LAPACK solve of the weight-space
    matrix (small problems only)."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    Phi = design_matrix(x, fit.h, fit.m, fit.D)
    A = Phi.conj().T @ (Phi / np.asarray(noise_sd, dtype=np.float64)[:, None] ** 2) + np.eye(Phi.shape[1])
    F = features(fit.D, fit.h, np.asarray(xt, dtype=np.float64)).reshape(len(xt), -1)
    eta = np.linalg.solve(A, F.conj().T)
    return np.einsum("tj,jt->t", F, eta).real


# ----------------------------------------------------------------------------------------------
# Dense references used by the oracle's own pins
# ----------------------------------------------------------------------------------------------
def design_matrix(x, h, m, D) -> np.ndarray:
    """Phi_{n,p} = D_p exp(+2 pi i h j_p.x_n), (N, M)  (eq ``205``)."""
    J = mode_indices(m, np.asarray(x).shape[1])
    return D.reshape(-1)[None, :] * np.exp(1j * TWO_PI * h * (np.asarray(x) @ J.T))


def kernel_tilde_matrix(xa, xb, h, m, D) -> np.ndarray:
    """K~_{nl} = k~(x_n - x_l) = sum_j h^d k^(hj) exp(2 pi i h j.(x_n - x_l))  (eq ``110``),
    i.e. Phi(xa) Phi(xb)^* (factorisation P:711-714).  Real part returned."""
    Pa = design_matrix(xa, h, m, D)
    Pb = design_matrix(xb, h, m, D)
    return (Pa @ Pb.conj().T).real


def dense_gp_mean(x, y, xt, kfun, sigma):
    """Function-space GP mean mu(x*) = sum_n alpha_n k(x*, x_n), (K + sigma^2 I) alpha = y
    (eqs ``mu``, ``362``) by Cholesky.  kfun(xa, xb) returns the kernel matrix."""
    K = kfun(x, x)
    c = scipy.linalg.cho_factor(K + sigma ** 2 * np.eye(len(x)))
    alpha = scipy.linalg.cho_solve(c, y)
    return kfun(xt, x) @ alpha, alpha


def dense_gp_mean_hetero(x, y, xt, kfun, noise_sd):
    """Function-space GP mean with per-point noise: mu(x*) = k(x*,X) (K + S)^{-1} y, S = diag(sigma_n^2)
    (eq ``mu`` P:98-115 with sigma^2 I replaced by S), by Cholesky."""
    K = kfun(x, x)
    c = scipy.linalg.cho_factor(K + np.diag(np.asarray(noise_sd, dtype=np.float64) ** 2))
    return kfun(xt, x) @ scipy.linalg.cho_solve(c, y)


def dense_gp_variance(x, xt, kfun, sigma):
    """Function-space GP variance s(x*) = k(x*,x*) - k(x*,X) (K + sigma^2 I)^{-1} k(X,x*)
    (eq ``s``) by Cholesky."""
    K = kfun(x, x)
    c = scipy.linalg.cho_factor(K + sigma ** 2 * np.eye(len(x)))
    Kt = kfun(xt, x)
    kss = np.array([kfun(xt[i:i + 1], xt[i:i + 1])[0, 0] for i in range(len(xt))])
    return kss - np.einsum("ij,ji->i", Kt, scipy.linalg.cho_solve(c, Kt.T))


# ----------------------------------------------------------------------------------------------
# Algorithm a1 end to end
# ----------------------------------------------------------------------------------------------
@dataclass
class OracleFit:
    kernel: str
    nu: float
    ell: float
    sigma: float
    eps: float
    d: int
    h: float
    m: int
    D: np.ndarray
    v: np.ndarray
    b: np.ndarray
    beta: np.ndarray
    iters: int
    history: list = field(default_factory=list)

    @property
    def M(self) -> int:
        return (2 * self.m + 1) ** self.d


def efgp_fit(x, y, kernel: str, ell: float, sigma: float, eps: float, nu: float = 0.0,
             h: float | None = None, m: int | None = None, cg_tol: float | None = None,
             max_iter: int | None = None, rescale: str = "A", dense_T_max: int = 4096,
             precond: str | None = None, toeplitz_fft: bool = False) -> OracleFit:
    """Algorithm ``a1`` steps 1-4: (h, m); v (eq 88); rhs Phi^*y (eq rhs); CG to
    relative residual cg_tol (default eps).  precond="kron": PCG with the NEXT-4
    preconditioner of reading G12 instead of plain CG.  toeplitz_fft=True: the Toeplitz product by
    the host FFT of reading G11 (c4 only; otherwise the direct product, dense when M <= dense_T_max)."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    N, d = x.shape
    if h is None or m is None:
        h0, m0 = choose_params(kernel, ell, d, eps, nu, rescale)
        h = h0 if h is None else h
        m = m0 if m is None else m
    D = spectral_weights(kernel, ell, d, h, m, nu)
    v = toeplitz_vector(x, h, m)
    b = rhs(x, y, h, m, D)
    tol = eps if cg_tol is None else cg_tol
    cap = default_max_iter(N, sigma, tol) if max_iter is None else max_iter
    T = toeplitz_matrix(v, m) if (2 * m + 1) ** d <= dense_T_max and not toeplitz_fft else None
    A = lambda p: system_apply(v, D, sigma ** 2, p, T, fft=toeplitz_fft)
    if precond == "kron":
        Pk = kron_preconditioner(v, D, sigma ** 2)
        beta, iters, hist = pcg(A, lambda r: kron_apply_inverse(Pk, r), b, tol, cap)
    elif precond == "jacobi":
        dg = jacobi_diagonal(v, D, sigma ** 2)
        beta, iters, hist = pcg(A, lambda r: r / dg, b, tol, cap)
    else:
        beta, iters, hist = cg(A, b, tol, cap)
    return OracleFit(kernel, nu, ell, sigma, eps, d, h, m, D, v, b, beta, iters, hist)


def efgp_predict(fit: OracleFit, xt) -> np.ndarray:
    """Algorithm ``a1`` steps 5-6: mu at the targets by the direct sum."""
    xt = np.asarray(xt, dtype=np.float64)
    if xt.ndim == 1:
        xt = xt[:, None]
    return posterior_mean(fit.beta, fit.D, fit.h, xt)
