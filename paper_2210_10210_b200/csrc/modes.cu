// K2 (deconvolve + extract), K3 (Toeplitz precompute) and K8 (type-2 pre-correction).
//
// Layouts: every mode array holds the Hermitian half j_d >= 0 only,
// row-major over (j_1 + K, ..., j_{d-1} + K, j_d) with K = 2m for v and K = m for J_m vectors.
// FFT boxes are cuFFT's half-spectrum layout n^(d-1) x (n/2 + 1), bin k_i = j_i mod n.
#include <cmath>

#include "efgp_internal.cuh"

namespace efgp {

// K2: v_j = Delta1^d G1^(j) / prod phi^1(j_k), j in J_2m;  (F^*y)_j = Delta2^d G2^(j) / prod phi^2(j_k),
// j in J_m (type-1 deconvolution; G^ = R2C of the spread grid, e^{-i} sign).
template <int D>
__global__ void k_deconv(const double2 *__restrict__ G1h, int64_t n1, const double2 *__restrict__ G2h, int64_t n2,
                         int m, const double *__restrict__ psi1, const double *__restrict__ psi2, double s1,
                         double s2, double2 *__restrict__ vh, double2 *__restrict__ fyh, int64_t Kvh, int64_t Mh) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < Kvh + Mh;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const bool first = idx < Kvh;
    const int K = first ? 2 * m : m;
    const int64_t n = first ? n1 : n2;
    const double *psi = first ? psi1 : psi2;
    const int64_t loc = first ? idx : idx - Kvh;
    int j[D];
    decode_half<D>(loc, K, j);
    double den = 1.0;
#pragma unroll
    for (int k = 0; k < D; ++k) den *= psi[j[k] < 0 ? -j[k] : j[k]];
    const double2 g = (first ? G1h : G2h)[box_index<D>(j, n)];
    const double sc = (first ? s1 : s2) / den;
    const double2 out = make_double2(g.x * sc, g.y * sc);
    if (first) vh[loc] = out;
    else fyh[loc] = out;
  }
}

// K3a: place v_j / L^d at bin j mod L of the Toeplitz box (zeros elsewhere) for C2R.
template <int D>
__global__ void k_place_v(const double2 *__restrict__ vh, int m, int64_t L, double scale, double2 *__restrict__ X,
                          int64_t box) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < box;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int j[D];
    double2 val = make_double2(0.0, 0.0);
    if (box_to_mode<D>(idx, L, 2 * m, j)) {
      const double2 v = vh[encode_half<D>(j, 2 * m)];
      val = make_double2(v.x * scale, v.y * scale);
    }
    X[idx] = val;
  }
}

// b = D F^*y
__global__ void k_make_b(const double2 *__restrict__ fyh, const double *__restrict__ Dh, double2 *__restrict__ b,
                         int64_t Mh) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < Mh; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 f = fyh[i];
    b[i] = make_double2(Dh[i] * f.x, Dh[i] * f.y);
  }
}

// K8: c'_j = Delta2^d D_j beta_j / prod phi^2(j_k) at bin j mod n2 (zeros elsewhere) for the type-2
// C2R (e^{+i} sign; Alg a1 step 6 coefficients sqrt(h^d k^(hj)) beta_j).
template <int D>
__global__ void k_place_t2(const double2 *__restrict__ beta, const double *__restrict__ Dh,
                           const double *__restrict__ psi2, int m, int64_t n2, double s2, double2 *__restrict__ X,
                           int64_t box) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < box;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int j[D];
    double2 val = make_double2(0.0, 0.0);
    if (box_to_mode<D>(idx, n2, m, j)) {
      const int64_t q = encode_half<D>(j, m);
      double den = 1.0;
#pragma unroll
      for (int k = 0; k < D; ++k) den *= psi2[j[k] < 0 ? -j[k] : j[k]];
      const double sc = s2 * Dh[q] / den;
      const double2 bb = beta[q];
      val = make_double2(bb.x * sc, bb.y * sc);
    }
    X[idx] = val;
  }
}

static unsigned grid_for(int64_t n, int threads, int sms) {
  int64_t b = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)sms * 8;
  if (b > cap) b = cap;
  return (unsigned)(b < 1 ? 1 : b);
}

efgp_status type1_modes(efgp_plan *pl, double *modes_out, cudaStream_t s) {
  const Params &P = pl->P;
  EFGP_CUFFT(cufftSetStream(pl->plan_g1, s));
  EFGP_CUFFT(cufftSetStream(pl->plan_g2, s));
  EFGP_CUFFT(cufftExecD2Z(pl->plan_g1, pl->g1, pl->G1h));
  EFGP_CUFFT(cufftExecD2Z(pl->plan_g2, pl->g2, pl->G2h));
  // the strength-y grid is n_rhs (= n1 for SORTED spreading, else n2); psi1 covers k <= 2m on n1
  const int64_t nr = P.n_rhs;
  const double *psir = (nr == P.n1) ? pl->psi1 : pl->psi2;
  const double s1 = std::pow(2.0 * kPi / (double)P.n1, P.d), s2 = std::pow(2.0 * kPi / (double)nr, P.d);
  double2 *vh = reinterpret_cast<double2 *>(modes_out);
  double2 *fyh = vh + P.Kvh;
  const unsigned g = grid_for(P.Kvh + P.Mh, 256, pl->num_sms);
  switch (P.d) {
    case 1: k_deconv<1><<<g, 256, 0, s>>>(pl->G1h, P.n1, pl->G2h, nr, (int)P.m, pl->psi1, psir, s1, s2, vh, fyh, P.Kvh, P.Mh); break;
    case 2: k_deconv<2><<<g, 256, 0, s>>>(pl->G1h, P.n1, pl->G2h, nr, (int)P.m, pl->psi1, psir, s1, s2, vh, fyh, P.Kvh, P.Mh); break;
    case 3: k_deconv<3><<<g, 256, 0, s>>>(pl->G1h, P.n1, pl->G2h, nr, (int)P.m, pl->psi1, psir, s1, s2, vh, fyh, P.Kvh, P.Mh); break;
  }
  EFGP_CUDA(cudaGetLastError());
  return EFGP_OK;
}

efgp_status type1_half(efgp_plan *pl, const double2 *G, int64_t n, int K, const double *psi, double2 *out,
                       cudaStream_t s) {
  const Params &P = pl->P;
  const double sc = std::pow(2.0 * kPi / (double)n, P.d);
  // k_deconv's first part (idx < Kvh) handles J_{2m}, its second (J_m) the rest: use one or the other
  const bool vgrid = K == 2 * P.m;
  const int64_t cnt = vgrid ? P.Kvh : P.Mh;
  const unsigned g = grid_for(cnt, 256, pl->num_sms);
  const int64_t kv = vgrid ? P.Kvh : 0, mh = vgrid ? 0 : P.Mh;
  switch (P.d) {
    case 1: k_deconv<1><<<g, 256, 0, s>>>(G, n, G, n, (int)P.m, psi, psi, sc, sc, out, out, kv, mh); break;
    case 2: k_deconv<2><<<g, 256, 0, s>>>(G, n, G, n, (int)P.m, psi, psi, sc, sc, out, out, kv, mh); break;
    case 3: k_deconv<3><<<g, 256, 0, s>>>(G, n, G, n, (int)P.m, psi, psi, sc, sc, out, out, kv, mh); break;
  }
  EFGP_CUDA(cudaGetLastError());
  return EFGP_OK;
}


// full v over J_2m ((4m+1)^2, row-major over (j1+2m, j2+2m)) from its Hermitian half (2D; the direct
// Toeplitz product of small-m CGs reads it)
__global__ void k_expand_v2(const double2 *__restrict__ vh, int m, double2 *__restrict__ vf) {
  const int K = 2 * m, n = 2 * K + 1;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n * n; idx += gridDim.x * blockDim.x) {
    int j[2] = {idx / n - K, idx % n - K};
    const bool neg = j[1] < 0;
    if (neg) {
      j[0] = -j[0];
      j[1] = -j[1];
    }
    const double2 v = vh[encode_half<2>(j, K)];
    vf[idx] = neg ? make_double2(v.x, -v.y) : v;
  }
}

efgp_status toeplitz_setup(efgp_plan *pl, const double *modes, cudaStream_t s) {
  const Params &P = pl->P;
  const double2 *vh = reinterpret_cast<const double2 *>(modes);
  const double2 *fyh = vh + P.Kvh;
  int64_t box = P.L / 2 + 1, Ld = P.L;
  for (int k = 0; k < P.d - 1; ++k) {
    box *= P.L;
    Ld *= P.L;
  }
  const double scale = 1.0 / (double)Ld;
  const unsigned g = grid_for(box, 256, pl->num_sms);
  switch (P.d) {
    case 1: k_place_v<1><<<g, 256, 0, s>>>(vh, (int)P.m, P.L, scale, pl->Xbox, box); break;
    case 2: k_place_v<2><<<g, 256, 0, s>>>(vh, (int)P.m, P.L, scale, pl->Xbox, box); break;
    case 3: k_place_v<3><<<g, 256, 0, s>>>(vh, (int)P.m, P.L, scale, pl->Xbox, box); break;
  }
  EFGP_CUDA(cudaGetLastError());
  EFGP_CUFFT(cufftSetStream(pl->plan_c2r_L, s));
  EFGP_CUFFT(cufftExecZ2D(pl->plan_c2r_L, pl->Xbox, pl->vhat));  // real: v is Hermitian (A.10)
  k_make_b<<<grid_for(P.Mh, 256, pl->num_sms), 256, 0, s>>>(fyh, pl->D_half, pl->b, P.Mh);
  EFGP_CUDA(cudaGetLastError());
  if (toeplitz_pt(P)) EFGP_TRY(pt_setup(pl, vh, s));
  if (toeplitz_dft2(P)) {  // 2D, larger m: full v, then its DFT along the second axis (cg.cu)
    const int n = (int)(4 * P.m + 1);
    if (!pl->vfull) EFGP_CUDA(cudaMalloc((void **)&pl->vfull, sizeof(double2) * n * n));
    k_expand_v2<<<grid_for((int64_t)n * n, 256, pl->num_sms), 256, 0, s>>>(vh, (int)P.m, pl->vfull);
    EFGP_CUDA(cudaGetLastError());
    EFGP_TRY(dft2_setup(pl, s));
  }
  if (toeplitz_direct(P)) {  // small m: the CG applies T by direct convolution with the full v
    const int n = (int)(4 * P.m + 1);
    if (!pl->vfull) EFGP_CUDA(cudaMalloc((void **)&pl->vfull, sizeof(double2) * n * n));
    if (!pl->toep_part) {  // split direct product (k_cg_toep2s): per-(row, split) partial rows + row counters
      const int64_t nrow = 2 * P.m + 1;
      EFGP_CUDA(cudaMalloc((void **)&pl->toep_part, sizeof(double2) * nrow * kToepSplitsHost * (P.m + 1)));
      EFGP_CUDA(cudaMalloc((void **)&pl->toep_cnt, sizeof(unsigned) * nrow));
      EFGP_CUDA(cudaMemsetAsync(pl->toep_cnt, 0, sizeof(unsigned) * nrow, s));
    }
    k_expand_v2<<<grid_for((int64_t)n * n, 256, pl->num_sms), 256, 0, s>>>(vh, (int)P.m, pl->vfull);
    EFGP_CUDA(cudaGetLastError());
  }
  return EFGP_OK;
}

efgp_status type2_grid(efgp_plan *pl, cudaStream_t s) {
  EFGP_TRY(type2_grid_from(pl, pl->x, s));
  pl->t2_valid = true;
  return EFGP_OK;
}

// The type-2 fine grid of an arbitrary Hermitian-half coefficient vector beta (weights layout):
// t2grid = C2R(c'), c'_j = Delta2^d D_j beta_j / prod phi^2(j_k)  (K8).
efgp_status type2_grid_from(efgp_plan *pl, const double2 *beta, cudaStream_t s) {
  return type2_grid_on(pl, beta, pl->P.n2, pl->psi2, pl->plan_t2, pl->T2box, pl->t2grid, s);
}

// K8 on an n^d grid with deconvolution table psi (k = 0..m at least), C2R plan `plan` (n^d Z2D).
efgp_status type2_grid_on(efgp_plan *pl, const double2 *beta, int64_t n, const double *psi, cufftHandle plan,
                          double2 *boxbuf, double *grid, cudaStream_t s) {
  const Params &P = pl->P;
  int64_t box = n / 2 + 1;
  for (int k = 0; k < P.d - 1; ++k) box *= n;
  const double sc = std::pow(2.0 * kPi / (double)n, P.d);
  const unsigned g = grid_for(box, 256, pl->num_sms);
  switch (P.d) {
    case 1: k_place_t2<1><<<g, 256, 0, s>>>(beta, pl->D_half, psi, (int)P.m, n, sc, boxbuf, box); break;
    case 2: k_place_t2<2><<<g, 256, 0, s>>>(beta, pl->D_half, psi, (int)P.m, n, sc, boxbuf, box); break;
    case 3: k_place_t2<3><<<g, 256, 0, s>>>(beta, pl->D_half, psi, (int)P.m, n, sc, boxbuf, box); break;
  }
  EFGP_CUDA(cudaGetLastError());
  EFGP_CUFFT(cufftSetStream(plan, s));
  EFGP_CUFFT(cufftExecZ2D(plan, boxbuf, grid));
  return EFGP_OK;
}

}  // namespace efgp
