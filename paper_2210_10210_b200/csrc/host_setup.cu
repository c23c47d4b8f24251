// Host-side setup of the EFGP plan (Alg a1 step 1 and NUFFT sizing).
// Written independently of oracle/ (which uses quadrature where this file uses closed forms).
#include <cmath>
#include <cstdio>
#include <cstring>

#include "efgp_internal.cuh"

namespace efgp {

// k^ at |xi| (P:2812 eq Ghat; P:2936-2944 eqs Crecall/hatc with the l^d reading G2).
double khat_host(const Params &p, double xi) {
  const int d = p.d;
  if (p.kernel == EFGP_SE) {
    return std::pow(std::sqrt(2.0 * kPi) * p.ell, d) * std::exp(-2.0 * std::pow(kPi * p.ell * xi, 2));
  }
  const double nu = p.nu;
  const double logc = d * std::log(2.0) + 0.5 * d * std::log(kPi) + nu * std::log(2.0 * nu) +
                      std::lgamma(nu + 0.5 * d) - std::lgamma(nu);
  const double s = 2.0 * nu + std::pow(2.0 * kPi * p.ell * xi, 2);
  return std::exp(logc + d * std::log(p.ell) + (-nu - 0.5 * d) * std::log(s));
}

static double round_down_12(double x) {
  const int e = (int)std::floor(std::log10(x));
  const double scale = std::pow(10.0, 11 - e);
  return std::floor(x * scale) / scale;
}

// ||k||_{L2(R^d)} of the Matérn kernel in closed form (G3, Plancherel):
// (2 pi l^2 / nu)^{d/4} Gamma(nu + d/2)/Gamma(nu) sqrt(Gamma(2 nu + d/2) / Gamma(2 nu + d)).
static double matern_l2(double nu, double ell, int d) {
  const double lg = std::lgamma(nu + 0.5 * d) - std::lgamma(nu) +
                    0.5 * (std::lgamma(2 * nu + 0.5 * d) - std::lgamma(2 * nu + d));
  return std::pow(2.0 * kPi * ell * ell / nu, 0.25 * d) * std::exp(lg);
}

// The norm expression as printed at P:1985-1986 (reading P).
static double matern_printed(double nu, double ell, int d) {
  return std::pow(nu / (kPi * ell * ell), 0.25 * d) *
         std::sqrt(std::tgamma(0.5 * d + 2 * nu) / (2.0 * std::tgamma(d + 2 * nu)));
}

int64_t next_smooth(int64_t n) {
  for (int64_t c = n < 1 ? 1 : n;; ++c) {
    int64_t r = c;
    for (int f : {2, 3, 5, 7})
      while (r % f == 0) r /= f;
    if (r == 1) return c;
  }
}

void gauss_legendre(int n, std::vector<double> &x, std::vector<double> &w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int i = 0; i < (n + 1) / 2; ++i) {
    double z = std::cos(kPi * (i + 0.75) / (n + 0.5)), pp = 0;
    for (int it = 0; it < 100; ++it) {
      double p1 = 1.0, p2 = 0.0;
      for (int j = 1; j <= n; ++j) {
        const double p3 = p2;
        p2 = p1;
        p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
      }
      pp = n * (z * p1 - p2) / (z * z - 1.0);
      const double dz = p1 / pp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    x[i] = -z;
    x[n - 1 - i] = z;
    w[i] = w[n - 1 - i] = 2.0 / ((1.0 - z * z) * pp * pp);
  }
}

// Piecewise-polynomial ES kernel: for cell offset a in [0, w) and
// u in [0, 1), phi_a(u) = phi((2(a+u) - w)/w) is approximated by a degree-es_degree(w) polynomial in
// s = 2u - 1 from Chebyshev interpolation, stored as monomial coefficients c[a][k].
void es_poly_fit(int w, double beta, EsPoly &out) {
  std::memset(&out, 0, sizeof(out));
  const int p = es_degree(w);  // degree
  out.deg = p;
  const int nn = p + 1;
  for (int a = 0; a < w; ++a) {
    std::vector<double> fs(nn), cheb(nn, 0.0);
    for (int j = 0; j < nn; ++j) {
      const double s = std::cos(kPi * (j + 0.5) / nn);
      const double u = 0.5 * (s + 1.0);
      const double z = (2.0 * (a + u) - w) / w;
      const double q = 1.0 - z * z;
      fs[j] = std::exp(beta * (std::sqrt(q > 0 ? q : 0.0) - 1.0));
    }
    for (int k = 0; k < nn; ++k) {
      double sacc = 0.0;
      for (int j = 0; j < nn; ++j) sacc += fs[j] * std::cos(kPi * k * (j + 0.5) / nn);
      cheb[k] = (k == 0 ? 1.0 : 2.0) * sacc / nn;
    }
    // Chebyshev -> monomial: T_0 = 1, T_1 = s, T_{k+1} = 2 s T_k - T_{k-1}
    std::vector<double> Tm1(nn, 0.0), T0(nn, 0.0), T1(nn, 0.0), mono(nn, 0.0);
    T0[0] = 1.0;
    for (int i = 0; i < nn; ++i) mono[i] += cheb[0] * T0[i];
    if (nn > 1) {
      T1[1] = 1.0;
      for (int i = 0; i < nn; ++i) mono[i] += cheb[1] * T1[i];
    }
    for (int k = 2; k < nn; ++k) {
      std::vector<double> T2(nn, 0.0);
      for (int i = 0; i < nn; ++i) {
        if (i > 0) T2[i] += 2.0 * T1[i - 1];
        T2[i] -= T0[i];
      }
      for (int i = 0; i < nn; ++i) mono[i] += cheb[k] * T2[i];
      T0 = T1;
      T1 = T2;
    }
    for (int k = 0; k < nn; ++k) out.c[a][k] = mono[k];
  }
  // exact mirror symmetry of the even ES kernel (es_weights relies on it): piece w-1-a is piece a at
  // -s, the middle piece (w odd) is even
  for (int a = 0; a < w / 2; ++a)
    for (int k = 0; k < nn; ++k) out.c[w - 1 - a][k] = (k & 1) ? -out.c[a][k] : out.c[a][k];
  if (w & 1)
    for (int k = 1; k < nn; k += 2) out.c[w / 2][k] = 0.0;
}

double es_poly_eval(const EsPoly &P, int a, double u) {
  const double s = 2.0 * u - 1.0;
  double acc = P.c[a][P.deg];
  for (int k = P.deg - 1; k >= 0; --k) acc = acc * s + P.c[a][k];
  return acc;
}

// phihat[k] = int phi~(t) cos(k t) dt over the support [-alpha, alpha], alpha = w pi / n, with phi~
// the piecewise polynomial actually used by the kernels (so deconvolution and spreading agree):
// = alpha (2/w) sum_a int_0^1 phi~_a(u) cos(k alpha (2(a+u) - w)/w) du, Gauss-Legendre per piece.
std::vector<double> es_fourier_table_poly(const EsPoly &P, int w, int64_t n, int64_t kmax) {
  const double alpha = w * kPi / (double)n;
  const int nq = 2 * P.deg + 40;
  std::vector<double> z, wq;
  gauss_legendre(nq, z, wq);
  std::vector<double> t(kmax + 1, 0.0);
  for (int a = 0; a < w; ++a) {
    for (int i = 0; i < nq; ++i) {
      const double u = 0.5 * (z[i] + 1.0), wu = 0.5 * wq[i];
      const double f = es_poly_eval(P, a, u);
      const double zz = (2.0 * (a + u) - w) / w;
      for (int64_t k = 0; k <= kmax; ++k) t[k] += wu * f * std::cos(k * alpha * zz);
    }
  }
  for (auto &v : t) v *= alpha * 2.0 / w;
  return t;
}

std::vector<double> es_fourier_table(int w, double beta, int64_t n, int64_t kmax) {
  const double alpha = w * kPi / (double)n;  // half-width of the kernel support in angle
  const int nq = 3 * w + 60;
  std::vector<double> z, wq;
  gauss_legendre(nq, z, wq);
  std::vector<double> phi(nq);
  for (int i = 0; i < nq; ++i) phi[i] = std::exp(beta * (std::sqrt(1.0 - z[i] * z[i]) - 1.0));
  std::vector<double> t(kmax + 1);
  for (int64_t k = 0; k <= kmax; ++k) {
    double s = 0.0;
    for (int i = 0; i < nq; ++i) s += wq[i] * phi[i] * std::cos(k * alpha * z[i]);
    t[k] = alpha * s;
  }
  return t;
}

std::string validate_and_choose(Params &p, const efgp_options &opt) {
  if (!(p.sigma > 0) || !std::isfinite(p.sigma)) return "sigma must be > 0";
  if (!(p.ell > 0) || !std::isfinite(p.ell)) return "ell must be > 0";
  if (!(p.eps >= 1e-14 && p.eps <= 1e-1)) return "eps must lie in [1e-14, 1e-1]";
  if (p.d < 1 || p.d > 3) return "d must be 1, 2 or 3";
  if (p.kernel != EFGP_SE && p.kernel != EFGP_MATERN) return "unknown kernel";
  if (p.kernel == EFGP_MATERN && !(p.nu >= 0.5)) return "Matern nu must be >= 1/2";
  const int d = p.d;
  p.rescale = opt.matern_rescale;
  if (opt.m > 0) {
    if (!(opt.h > 0 && opt.h < 1)) return "explicit h must lie in (0, 1)";
    p.h = opt.h;
    p.m = opt.m;
  } else if (p.kernel == EFGP_SE) {
    // Cor c:SEparams, reading G4
    p.h = round_down_12(1.0 / (1.0 + p.ell * std::sqrt(2.0 * std::log(4.0 * d * std::pow(3.0, d) / p.eps))));
    p.m = (int64_t)std::ceil(std::sqrt(0.5 * std::log(std::pow(4.0, d + 1) * d / p.eps)) / (kPi * p.ell * p.h));
  } else {
    // Remark r:heur eqs hheur/mheur after the §7.1 rescaling, reading G3
    double e = p.eps;
    if (p.rescale == EFGP_RESCALE_L2) e *= matern_l2(p.nu, p.ell, d);
    else if (p.rescale == EFGP_RESCALE_PRINTED) e *= matern_printed(p.nu, p.ell, d);
    p.h = round_down_12(1.0 / (1.0 + 0.85 * (p.ell / std::sqrt(p.nu)) * std::log(1.0 / e)));
    p.m = (int64_t)std::ceil((1.0 / p.h) *
                             std::pow(std::pow(kPi, p.nu + 0.5 * d) * std::pow(p.ell, 2 * p.nu) * e / 0.15,
                                      -1.0 / (2 * p.nu + 0.5 * d)));
  }
  if (p.m < 1) p.m = 1;
  if (!(p.h > 0 && p.h < 1)) return "grid spacing h must lie in (0, 1)";
  const int64_t n = 2 * p.m + 1;
  p.M = 1;
  p.Mh = p.m + 1;
  p.Kvh = 2 * p.m + 1;
  for (int k = 0; k < d; ++k) p.M *= n;
  for (int k = 0; k < d - 1; ++k) {
    p.Mh *= n;
    p.Kvh *= 4 * p.m + 1;
  }
  p.cg_tol = opt.cg_tol > 0 ? opt.cg_tol : p.eps;
  p.max_iter_opt = opt.max_iter;
  p.nufft_tol = opt.nufft_tol > 0 ? opt.nufft_tol : p.eps / 10.0;
  if (p.nufft_tol < 1e-15) p.nufft_tol = 1e-15;
  // ES kernel, upsampling 2: w = ceil(log10(1/tol)) + 1, beta = 2.30 w
  p.w = (int)std::ceil(std::log10(1.0 / p.nufft_tol)) + 1;
  if (p.w < 2) p.w = 2;
  if (p.w > kMaxW) p.w = kMaxW;
  p.beta_es = 2.30 * p.w;
  // grids: n >= max(2K, 2w) rounded up to 7-smooth (reading G14)
  p.n1 = next_smooth(std::max<int64_t>(2 * (4 * p.m + 1), 2 * p.w));
  p.n2 = next_smooth(std::max<int64_t>(2 * (2 * p.m + 1), 2 * p.w));
  p.L = next_smooth(4 * p.m + 1);
  p.spread_method = opt.spread_method;
  p.spread_method_requested = opt.spread_method;
  p.graph_iters = opt.graph_iters > 0 ? opt.graph_iters : 8;
  es_poly_fit(p.w, p.beta_es, p.poly);
  for (int a = 0; a < kMaxW; ++a)
    for (int k = 0; k < kMaxW + 3; ++k) p.polyf.c[a][k] = (float)p.poly.c[a][k];
  for (int q = 0; q < 3; ++q)
    for (int k = 0; k < 10; ++k) {
      const int a0 = 2 * q, a1 = 2 * q + 1;
      p.polyp.c[q][k] = make_float2(a0 < p.w && k <= p.poly.deg ? (float)p.poly.c[a0][k] : 0.f,
                                    a1 < p.w && k <= p.poly.deg ? (float)p.poly.c[a1][k] : 0.f);
    }
  // fp32 kernel weights (fp64 accumulation) only when asked for, and only where fp32 rounding of the
  // weights (~1e-7 relative) sits well below the NUFFT tolerance (DESIGN.md §7 "K1 weights")
  if (opt.spread_weights < EFGP_WEIGHTS_FP64 || opt.spread_weights > EFGP_WEIGHTS_MIXED)
    return "unknown spread_weights";
  if (opt.spread_weights != EFGP_WEIGHTS_FP64 && p.nufft_tol < 1e-6)
    return "fp32 spreading weights need nufft_tol >= 1e-6";
  p.spread_mode = opt.spread_weights;
  if (opt.precond < EFGP_PRECOND_NONE || opt.precond > EFGP_PRECOND_JACOBI) return "unknown precond";
  // AUTO: the Kronecker factors are exact in D only for a separable spectral density (SE)
  if (opt.hetero_method < EFGP_HETERO_AUTO || opt.hetero_method > EFGP_HETERO_NUFFT) return "unknown hetero_method";
  p.hetero_method = opt.hetero_method;
  p.precond = opt.precond == EFGP_PRECOND_AUTO ? (p.kernel == EFGP_SE ? EFGP_PRECOND_KRON : EFGP_PRECOND_JACOBI)
                                               : opt.precond;
  resolve_spread_method(p);
  return "";
}

}  // namespace efgp
