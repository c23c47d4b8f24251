// NEXT-3: heteroskedastic noise sigma_n (reading G11).
//
// Weight space with S = diag(sigma_n^2):  (Phi^* S^-1 Phi + I) beta = Phi^* S^-1 y,  mu = phi(x*) beta.
// S breaks the Toeplitz structure of Phi^*Phi, so every CG product is applied "as in BBMM
// methods" with one NUFFT pair over the N points:
//
//   A p = D . F^*( S^-1 . F(D . p) ) + p
//       = K2_rhs( K1( x, K9( x, C2R(K8(p)) ) / sigma^2 ) ) + p
//
// K8 places D p / phi^2 on the type-2 box, cuFFT C2R gives the fine grid, K9 interpolates it at the
// data points and divides by sigma_n^2 (fused), K1 spreads those values (the same spreader as the
// fit; its strength-y grid is the one used), cuFFT R2C + k_het_modes deconvolve, multiply by D and
// add p.  The right-hand side is the same K1 -> R2C -> k_het_modes chain on y_n / sigma_n^2.
#include <cmath>
#include <cstring>

#include "efgp_internal.cuh"

namespace efgp {

// w_n = y_n / sigma_n^2; raise dflags[2] for sigma_n <= 0 or non-finite; min sigma_n into *minbits
// (for positive doubles the IEEE bit pattern is ordered like the value)
__global__ void k_het_prep(const double *__restrict__ y, const double *__restrict__ sd, int64_t N,
                           double *__restrict__ w, unsigned long long *__restrict__ minbits, int *__restrict__ err) {
  unsigned long long lmin = ~0ull;
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const double s = sd[i];
    const bool ok = s > 0.0 && isfinite(s);
    bad |= !ok;
    w[i] = ok ? y[i] / (s * s) : 0.0;
    if (ok) {
      const unsigned long long b = (unsigned long long)__double_as_longlong(s);
      lmin = b < lmin ? b : lmin;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, lmin, o);
    lmin = t < lmin ? t : lmin;
  }
  if ((threadIdx.x & 31) == 0 && lmin != ~0ull) atomicMin(minbits, lmin);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err + 2, 1);
}

// out_q = D_q f_q + (p ? p_q : 0),  f_j = Delta^d G^(j) / prod phi(j_k) on the J_m half (type-1
// deconvolution of the strength-w grid, as K2)
template <int D>
__global__ void k_het_modes(const double2 *__restrict__ G, int64_t n, int m, const double *__restrict__ psi,
                            double sc, const double *__restrict__ Dh, const double2 *__restrict__ p,
                            double2 *__restrict__ out, int64_t Mh) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x) {
    int j[D];
    decode_half<D>(q, m, j);
    double den = 1.0;
#pragma unroll
    for (int k = 0; k < D; ++k) den *= psi[j[k] < 0 ? -j[k] : j[k]];
    const double2 g = G[box_index<D>(j, n)];
    const double f = Dh[q] * sc / den;
    double2 o = make_double2(f * g.x, f * g.y);
    if (p) {
      const double2 pp = p[q];
      o.x += pp.x;
      o.y += pp.y;
    }
    out[q] = o;
  }
}

namespace {

struct HetCtx {
  const double *x, *sd;
  double *w;
  int64_t N;
  int64_t n;           // fine grid of both transforms (n_rhs)
  const double *psi;   // its deconvolution table
  cufftHandle plan;    // its C2R plan
  double2 *box;
  double *grid;
};

unsigned grid_for(int64_t n, int sms) {
  int64_t b = (n + 255) / 256;
  const int64_t cap = (int64_t)sms * 8;
  return (unsigned)(b > cap ? cap : (b < 1 ? 1 : b));
}

// out = D . F^*(w) (+ p): spread the strengths w at x, R2C, deconvolve
efgp_status spread_to_modes(efgp_plan *pl, const double *x, const double *w, int64_t N, const double2 *p,
                            double2 *out, cudaStream_t s) {
  const Params &P = pl->P;
  EFGP_TRY(spread_begin(pl, s));
  EFGP_TRY(spread_points(pl, x, w, N, s));
  EFGP_TRY(spread_end(pl, s));
  EFGP_CUFFT(cufftSetStream(pl->plan_g2, s));
  EFGP_CUFFT(cufftExecD2Z(pl->plan_g2, pl->g2, pl->G2h));
  const int64_t nr = P.n_rhs;
  const double *psir = (nr == P.n1) ? pl->psi1 : pl->psi2;
  const double sc = std::pow(2.0 * kPi / (double)nr, P.d);
  const unsigned g = grid_for(P.Mh, pl->num_sms);
  switch (P.d) {
    case 1: k_het_modes<1><<<g, 256, 0, s>>>(pl->G2h, nr, (int)P.m, psir, sc, pl->D_half, p, out, P.Mh); break;
    case 2: k_het_modes<2><<<g, 256, 0, s>>>(pl->G2h, nr, (int)P.m, psir, sc, pl->D_half, p, out, P.Mh); break;
    case 3: k_het_modes<3><<<g, 256, 0, s>>>(pl->G2h, nr, (int)P.m, psir, sc, pl->D_half, p, out, P.Mh); break;
  }
  EFGP_CUDA(cudaGetLastError());
  return EFGP_OK;
}

// A p = D F^*(S^-1 F(D p)) + p
efgp_status het_apply(efgp_plan *pl, const double2 *p, double2 *Ap, void *vctx) {
  const HetCtx *c = static_cast<const HetCtx *>(vctx);
  cudaStream_t s = pl->stream;
  EFGP_TRY(type2_grid_on(pl, p, c->n, c->psi, c->plan, c->box, c->grid, s));
  EFGP_TRY(interp_weighted(pl, c->grid, c->n, c->x, c->N, c->sd, c->w, s));
  return spread_to_modes(pl, c->x, c->w, c->N, p, Ap, s);
}

float elapsed_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
    cudaGetLastError();
    return 0.f;
  }
  return ms;
}

}  // namespace

efgp_status fit_hetero_device(efgp_plan *pl, const double *x, const double *y, const double *sd, int64_t N) {
  const Params &P = pl->P;
  cudaStream_t s = pl->stream;
  pl->fitted = false;
  pl->op_valid = false;  // no Toeplitz operator: predict_var is refused after a heteroskedastic fit
  pl->t2_valid = false;  // the type-2 grid is rebuilt from beta by the next predict
  double *w = nullptr;
  EFGP_CUDA(cudaMallocAsync((void **)&w, sizeof(double) * N, s));
  unsigned long long *minbits = reinterpret_cast<unsigned long long *>(pl->scal + 24);
  EFGP_CUDA(cudaEventRecord(pl->ev[0], s));
  EFGP_CUDA(cudaMemsetAsync(minbits, 0xff, sizeof(unsigned long long), s));
  EFGP_CUDA(cudaMemsetAsync(pl->dflags + 2, 0, sizeof(int), s));
  k_het_prep<<<grid_for(N, pl->num_sms), 256, 0, s>>>(y, sd, N, w, minbits, pl->dflags);
  EFGP_CUDA(cudaGetLastError());
  int flags[4];
  unsigned long long mb = 0;
  EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned, pl->dflags, sizeof(int) * 4, cudaMemcpyDeviceToHost, s));
  EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned + 8, minbits, sizeof(mb), cudaMemcpyDeviceToHost, s));
  EFGP_CUDA(cudaStreamSynchronize(s));
  std::memcpy(flags, pl->h_pinned, sizeof(flags));
  std::memcpy(&mb, pl->h_pinned + 8, sizeof(mb));
  efgp_status st = EFGP_OK;
  if (flags[2]) {
    pl->err = "fit_hetero: every noise standard deviation must be finite and > 0";
    st = EFGP_ERR_INVALID;
  }
  // b = D F^*(y / sigma^2); spread_begin clears the input flags, spread_points raises dflags[0]
  if (st == EFGP_OK) st = spread_to_modes(pl, x, w, N, nullptr, pl->b, s);
  if (st == EFGP_OK) {
    EFGP_CUDA(cudaEventRecord(pl->ev[1], s));
    EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned, pl->dflags, sizeof(int) * 4, cudaMemcpyDeviceToHost, s));
    EFGP_CUDA(cudaStreamSynchronize(s));
    std::memcpy(flags, pl->h_pinned, sizeof(flags));
    if (flags[0]) {
      pl->err = "fit_hetero: a coordinate is outside [0,1] or non-finite, or an observation is non-finite";
      st = EFGP_ERR_INVALID;
    }
  }
  if (st == EFGP_OK) {
    double smin = 0;
    std::memcpy(&smin, &mb, sizeof(smin));
    int64_t max_iter = P.max_iter_opt;
    if (max_iter <= 0) {  // P:1766 with sigma = min sigma_n (reading G11)
      max_iter = (int64_t)std::ceil(std::log(1.0 / P.cg_tol) * std::sqrt((double)N) / (2.0 * smin));
      if (max_iter < 10) max_iter = 10;
    }
    // Both NUFFTs on the same fine grid n_rhs with the same kernel and deconvolution: the type-2 is
    // then the exact adjoint of the type-1, so the applied operator is exactly Hermitian (CG's
    // recurrences assume it; with the v grid n1 for the spread and n2 for the interpolation the
    // mismatch ~nufft_tol slowed parity-mode CG by ~30 %).
    HetCtx ctx{x, sd, w, N, P.n_rhs, nullptr, 0, nullptr, nullptr};
    if (P.n_rhs == P.n2) {
      ctx.psi = pl->psi2;
      ctx.plan = pl->plan_t2;
      ctx.box = pl->T2box;
      ctx.grid = pl->t2grid;
    } else {
      if (!pl->het_grid) {
        int64_t box = P.n_rhs / 2 + 1, cells = P.n_rhs;
        for (int k = 0; k < P.d - 1; ++k) {
          box *= P.n_rhs;
          cells *= P.n_rhs;
        }
        EFGP_CUDA(cudaMalloc((void **)&pl->het_box, sizeof(double2) * box));
        EFGP_CUDA(cudaMalloc((void **)&pl->het_grid, sizeof(double) * cells));
        int dims[3] = {(int)P.n_rhs, (int)P.n_rhs, (int)P.n_rhs};
        EFGP_CUFFT(cufftPlanMany(&pl->plan_het, P.d, dims, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2D, 1));
      }
      ctx.psi = pl->psi1;  // n_rhs == n1: psi1 covers k <= 2m
      ctx.plan = pl->plan_het;
      ctx.box = pl->het_box;
      ctx.grid = pl->het_grid;
    }
    st = cg_solve_op(pl, max_iter, het_apply, &ctx);
    EFGP_CUDA(cudaEventRecord(pl->ev[4], s));
    EFGP_CUDA(cudaEventSynchronize(pl->ev[4]));
    pl->t_spread = elapsed_ms(pl->ev[0], pl->ev[1]);
    pl->t_modes = 0;
    pl->t_solve = elapsed_ms(pl->ev[1], pl->ev[4]);
    if (st == EFGP_OK || st == EFGP_ERR_NOCONVERGE) {
      pl->fitted = true;
      pl->N_last = N;
    }
    if (st == EFGP_ERR_NOCONVERGE) pl->err = "CG reached max_iter before the relative residual reached cg_tol";
  }
  cudaFreeAsync(w, s);
  EFGP_CUDA(cudaStreamSynchronize(s));
  return st;
}

}  // namespace efgp
