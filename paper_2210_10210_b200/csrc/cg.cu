// K4-K7 + F2: conjugate gradients on (D F^*F D + sigma^2 I) beta = D F^*y (eq "be", P:570;
// Alg a1 step 4; stop at relative residual cg_tol), with the Toeplitz
// product of Alg a:FF done by real transforms:
//
//   A p = D . extract_{J_m}( R2C( C2R(pad_L(D . p)) * vhat ) ) + sigma^2 p,   vhat = C2R(v)/L^d (real)
//
// Vectors live on the Hermitian half j_d >= 0 (Mh entries); Hermitian inner products become
// sum_q w_q Re(conj(a_q) b_q) with w_q = 2 for j_d > 0 and 1 for j_d = 0.
// One iteration = C2R, k_mul, R2C, k_cg_apply, k_cg_xr, k_cg_p; a CUDA graph captures
// graph_iters iterations; the host polls a device-side "done" flag after each graph launch, so the
// reported iteration count is exact (kernels of iterations after convergence return at entry).
// Block reductions are deterministic (fixed order, no atomics).
#include <cmath>
#include <cstring>

#include "efgp_internal.cuh"

namespace efgp {

struct CGState {
  double rr;        // current ||r||^2 (weighted)
  double rr_old;    // ||r||^2 of the previous iteration (for beta_cg)
  double bnorm;     // ||b||
  double tol;
  double sigma2;
  long long iter;
  long long max_iter;
  int done;         // 1: converged, 2: hit max_iter
  int pad_;
  double rz;        // PCG: (r, z) of the current residual (NEXT-4)
};

constexpr int kCGThreads = 256;



__device__ __forceinline__ double block_sum(double v, double *sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  return t;  // valid in thread 0
}

// every block reduces the same partials in the same order -> identical value everywhere
__device__ __forceinline__ double reduce_partials(const double *__restrict__ part, int n, double *sh) {
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v += part[i];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) sh[32] = v;
  __syncthreads();
  return sh[32];
}

__global__ void k_cg_init(const double2 *__restrict__ b, double2 *__restrict__ x, double2 *__restrict__ r,
                          double2 *__restrict__ p, int64_t Mh, int m, double *__restrict__ part) {
  __shared__ double sh[40];
  double acc = 0.0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x) {
    const double2 bb = b[q];
    x[q] = make_double2(0.0, 0.0);
    r[q] = bb;
    p[q] = bb;
    const double wq = (q % (m + 1)) ? 2.0 : 1.0;
    acc += wq * (bb.x * bb.x + bb.y * bb.y);
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void k_cg_init2(CGState *st, const double *__restrict__ part, int nblk, double *hist) {
  __shared__ double sh[40];
  const double rr = reduce_partials(part, nblk, sh);
  if (threadIdx.x == 0) {
    st->rr = rr;
    st->rr_old = rr;
    st->bnorm = sqrt(rr);
    st->iter = 0;
    st->done = (rr == 0.0) ? 1 : 0;
    hist[0] = rr == 0.0 ? 0.0 : 1.0;
  }
}

// pad: Xbox = D . p at the J_m bins of the L-box, 0 elsewhere (the C2R input; cuFFT may overwrite
// it, so it is rewritten in full every iteration)
template <int D>
__device__ __forceinline__ void pad_box(const double2 *__restrict__ p, const double *__restrict__ Dh, int m,
                                        int64_t L, double2 *__restrict__ X, int64_t box) {
  const int64_t nh = L / 2 + 1;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < box;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = idx;
    const int64_t kd = rem % nh;
    rem /= nh;
    bool ok = kd <= m;
    int64_t q = kd, stride = m + 1;
#pragma unroll
    for (int k = D - 2; k >= 0; --k) {
      const int64_t kk = rem % L;
      rem /= L;
      int64_t j;
      ok = ok && bin_to_mode(kk, L, m, j);
      q += (j + m) * stride;
      stride *= (2 * m + 1);
    }
    double2 val = make_double2(0.0, 0.0);
    if (ok) {
      const double2 pp = p[q];
      const double dq = Dh[q];
      val = make_double2(dq * pp.x, dq * pp.y);
    }
    X[idx] = val;
  }
}

template <int D>
__global__ void k_cg_pad0(const double2 *__restrict__ p, const double *__restrict__ Dh, int m, int64_t L,
                          double2 *__restrict__ X, int64_t box) {
  pad_box<D>(p, Dh, m, L, X, box);
}

__global__ void k_mul(double *__restrict__ Y, const double *__restrict__ vhat, int64_t n, const CGState *st) {
  if (st->done) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    Y[i] *= vhat[i];
}

// Ap = D . Z[J_m] + sigma^2 p ; partial <p, Ap>
template <int D>
__global__ void k_cg_apply(const double2 *__restrict__ Z, const double2 *__restrict__ p, const double *__restrict__ Dh,
                           double2 *__restrict__ Ap, int64_t Mh, int m, int64_t L, const CGState *st,
                           double *__restrict__ part) {
  __shared__ double sh[40];
  pdl_trigger();
  if (st->done) return;
  const double s2 = st->sigma2;
  double acc = 0.0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = q;
    const int64_t jd = rem % (m + 1);
    rem /= (m + 1);
    int64_t zi = jd, stride = L / 2 + 1;
#pragma unroll
    for (int k = D - 2; k >= 0; --k) {
      int64_t j = rem % (2 * m + 1) - m;
      rem /= (2 * m + 1);
      zi += (j < 0 ? j + L : j) * stride;
      stride *= L;
    }
    const double2 z = Z[zi], pp = p[q];
    const double dq = Dh[q];
    const double2 a = make_double2(dq * z.x + s2 * pp.x, dq * z.y + s2 * pp.y);
    Ap[q] = a;
    const double wq = jd ? 2.0 : 1.0;
    acc += wq * (pp.x * a.x + pp.y * a.y);
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// alpha = rr / <p,Ap>; x += alpha p; r -= alpha Ap; partial ||r||^2
__global__ void k_cg_xr(double2 *__restrict__ x, double2 *__restrict__ r, const double2 *__restrict__ p,
                        const double2 *__restrict__ Ap, int64_t Mh, int m, CGState *st,
                        const double *__restrict__ part_pAp, double *__restrict__ part_rr, int nblk,
                        const double *__restrict__ part_rz = nullptr) {
  __shared__ double sh[40];
  pdl_wait();
  pdl_trigger();
  if (st->done) return;
  const double pAp = reduce_partials(part_pAp, nblk, sh);
  // CG: alpha = (r,r)/(p,Ap); PCG: alpha = (r,z)/(p,Ap), (r,z) reduced from its partials
  const double rr = part_rz ? reduce_partials(part_rz, nblk, sh) : st->rr;
  if (part_rz && blockIdx.x == 0 && threadIdx.x == 0) st->rz = rr;
  const double alpha = rr / pAp;
  double acc = 0.0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x) {
    const double2 pp = p[q], a = Ap[q];
    double2 xx = x[q], rq = r[q];
    xx.x += alpha * pp.x;
    xx.y += alpha * pp.y;
    rq.x -= alpha * a.x;
    rq.y -= alpha * a.y;
    x[q] = xx;
    r[q] = rq;
    const double wq = (q % (m + 1)) ? 2.0 : 1.0;
    acc += wq * (rq.x * rq.x + rq.y * rq.y);
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) {
    part_rr[blockIdx.x] = acc;
    if (blockIdx.x == 0 && !part_rz) st->rr_old = rr;
  }
}

// beta_cg = rr_new / rr_old; p = r + beta_cg p; pad; bookkeeping (block 0)
template <int D>
__global__ void k_cg_p(const double2 *__restrict__ r, double2 *__restrict__ p, const double *__restrict__ Dh,
                       int64_t Mh, int m, int64_t L, double2 *__restrict__ X, int64_t box, CGState *st,
                       const double *__restrict__ part_rr, int nblk, double *__restrict__ hist) {
  __shared__ double sh[40];
  pdl_wait();
  pdl_trigger();
  if (st->done) return;
  const double rr_new = reduce_partials(part_rr, nblk, sh);
  const double bcg = rr_new / st->rr_old;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x) {
    const double2 rq = r[q], pp = p[q];
    p[q] = make_double2(rq.x + bcg * pp.x, rq.y + bcg * pp.y);
  }
  // grid-wide dependency: the pad below reads p written by other blocks -> separate kernel
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->rr = rr_new;
    const long long it = st->iter + 1;
    st->iter = it;
    const double rel = sqrt(rr_new) / st->bnorm;
    hist[it] = rel;
    if (rel <= st->tol) st->done = 1;
    else if (it >= st->max_iter) st->done = 2;
  }
}

template <int D>
__global__ void k_cg_pad(const double2 *__restrict__ p, const double *__restrict__ Dh, int m, int64_t L,
                         double2 *__restrict__ X, int64_t box, const CGState *st) {
  // runs even when done was just set: harmless (the next C2R input is never used)
  pdl_wait();
  pad_box<D>(p, Dh, m, L, X, box);
}


// Toeplitz product by direct convolution (2D, small m; toeplitz_direct): CTA = output row j1.
//   out_j = sum_{k in J_m} v_{j-k} u_k,  u = D p (Hermitian completion of the half),  j = (j1, 0..m)
//   Ap_j = D_j out_j + sigma^2 p_j,  partial <p, Ap>
// Replaces pad + C2R + multiply + R2C + apply of the FFT path; the same operator (the FFT path's
// circulant embedding is exact for |j - k| <= 2m), summed directly.  c3 / c5: 25-28 -> 20-21 us per
// CG iteration (1024 threads; 256 threads gave 23-24 us, a thread per output 27 us).
constexpr int kToepThreads = 1024;
__global__ void __launch_bounds__(kToepThreads) k_cg_toep2(const double2 *__restrict__ vfull,
                                                           const double2 *__restrict__ p,
                                                           const double *__restrict__ Dh, double2 *__restrict__ Ap,
                                                           int m, const CGState *st, double *__restrict__ part) {
  extern __shared__ double2 tsm[];
  __shared__ double sh[40];
  pdl_trigger();
  if (st->done) return;
  const int n = 2 * m + 1, nv = 4 * m + 1, j1 = (int)blockIdx.x - m;
  double2 *u = tsm;                // n x n: u[(k1+m) n + (k2+m)]
  double2 *vr = tsm + n * n;       // n rows x nv: vr[(k1+m) nv + (s+2m)] = v_{j1-k1, s}
  double2 *red = vr + n * nv;      // partial sums [slices][m+1]
  // u from the canonical half (k2 > 0, or k2 = 0 and k1 >= 0): the redundant (k1 < 0, 0) entries of the
  // stored half are not read, so the product is exactly Hermitian (the FFT path's C2R projects the
  // same way); without this the CG stalls on the c3 systems (roundoff in the j2 = 0 plane)
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    int k1 = idx / n - m, k2 = idx % n - m;
    const bool neg = k2 < 0 || (k2 == 0 && k1 < 0);
    if (neg) {
      k1 = -k1;
      k2 = -k2;
    }
    const int64_t q = (int64_t)(k1 + m) * (m + 1) + k2;
    const double2 pp = p[q];
    const double dq = Dh[q];
    u[idx] = make_double2(dq * pp.x, neg ? -dq * pp.y : dq * pp.y);
  }
  for (int idx = threadIdx.x; idx < n * nv; idx += blockDim.x) {
    const int k1 = idx / nv - m, sc = idx % nv;
    vr[idx] = vfull[(int64_t)(j1 - k1 + 2 * m) * nv + sc];
  }
  __syncthreads();
  // each thread: 4 consecutive outputs j2 .. j2+3 over a slice of the k1 rows; along k2 the four
  // v_{j1-k1, j2+o-k2} form a sliding window (one new shared load per step): 2 loads per 4 MACs
  const int nout = m + 1, ngrp = (nout + 3) / 4, slices = blockDim.x / ngrp;
  const int t = threadIdx.x, g4 = t % ngrp, sl = t / ngrp, j2b = 4 * g4;
  if (sl < slices) {
    double re[4] = {0.0, 0.0, 0.0, 0.0}, im[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k1 = sl; k1 < n; k1 += slices) {  // k1 + m
      const double2 *ur = u + k1 * n;
      // v index of (j2b + o) - k2 at k2 = -m: j2b + o + m + 2m
      const double2 *vrow = vr + k1 * nv + (j2b + 3 * m);
      double2 w[4];
#pragma unroll
      for (int o = 0; o < 4; ++o) w[o] = (j2b + o <= m) ? vrow[o] : make_double2(0.0, 0.0);
      for (int k2 = 0; k2 < n; ++k2) {  // k2 + m; the window moves down by one cell per step
        const double2 b = ur[k2];
#pragma unroll
        for (int o = 0; o < 4; ++o) {
          re[o] = fma(w[o].x, b.x, fma(-w[o].y, b.y, re[o]));
          im[o] = fma(w[o].x, b.y, fma(w[o].y, b.x, im[o]));
        }
#pragma unroll
        for (int o = 3; o > 0; --o) w[o] = w[o - 1];
        const int nxt = j2b + 3 * m - (k2 + 1);  // v index of output j2b at the next k2
        w[0] = (k2 + 1 < n) ? vr[k1 * nv + nxt] : make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int o = 0; o < 4; ++o)
      if (j2b + o <= m) red[sl * nout + j2b + o] = make_double2(re[o], im[o]);
  }
  __syncthreads();
  double acc = 0.0;
  if (t < nout && !(t == 0 && j1 < 0)) {  // (j1 < 0, 0) is written by row -j1 as the conjugate
    double2 o = make_double2(0.0, 0.0);
    for (int k = 0; k < slices; ++k) {
      o.x += red[k * nout + t].x;
      o.y += red[k * nout + t].y;
    }
    const int64_t q = (int64_t)(j1 + m) * (m + 1) + t;
    const double2 pp = p[q];
    const double dq = Dh[q], s2 = st->sigma2;
    double2 a = make_double2(dq * o.x + s2 * pp.x, dq * o.y + s2 * pp.y);
    if (t == 0 && j1 == 0) a.y = s2 * pp.y;  // j = 0: (T u)_0 is real
    Ap[q] = a;
    acc = (t ? 2.0 : 1.0) * (pp.x * a.x + pp.y * a.y);
    if (t == 0 && j1 > 0) {  // the mirrored entry (-j1, 0) = conj, with the canonical p
      Ap[(int64_t)(m - j1) * (m + 1)] = make_double2(a.x, -a.y);
      acc *= 2.0;
    }
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

static size_t toep2_smem(int m) {
  const int n = 2 * m + 1, nv = 4 * m + 1;
  const int nout = m + 1, slices = kToepThreads / ((nout + 3) / 4);
  return sizeof(double2) * ((size_t)n * n + (size_t)n * nv + (size_t)slices * nout);
}

static efgp_status ensure_hist(efgp_plan *pl, int64_t max_iter) {
  if (max_iter + 1 > pl->hist_cap) {
    for (cudaGraphExec_t *e : {&pl->cg_exec, &pl->pcg_exec})  // captured graphs hold the old pointer
      if (*e) {
        cudaGraphExecDestroy(*e);
        *e = nullptr;
      }
    if (pl->hist) cudaFree(pl->hist);
    pl->hist = nullptr;
    pl->hist_cap = 0;
    EFGP_CUDA(cudaMalloc(&pl->hist, sizeof(double) * (max_iter + 1)));
    pl->hist_cap = max_iter + 1;
  }
  return EFGP_OK;
}

static unsigned nblocks(int64_t n, int sms) {
  int64_t b = (n + kCGThreads - 1) / kCGThreads;
  const int64_t cap = (int64_t)sms * 4;
  if (b > cap) b = cap;
  return (unsigned)(b < 1 ? 1 : b);
}

template <int D>
static efgp_status enqueue_iteration(efgp_plan *pl, cudaStream_t s, CGState *st, int64_t box, int64_t Ld,
                                     unsigned nb, unsigned nbox) {
  const Params &P = pl->P;
  double *part_pAp = pl->partials, *part_rr = pl->partials + pl->cg_blocks;
  const bool direct = D == 2 && toeplitz_direct(P);
  if (direct) {  // the partials come from 2m+1 CTAs
    const int nrow = (int)(2 * P.m + 1);
    k_cg_toep2<<<nrow, kToepThreads, toep2_smem((int)P.m), s>>>(pl->vfull, pl->p, pl->D_half, pl->Ap, (int)P.m, st,
                                                                part_pAp);
    EFGP_CUDA(launch_pdl(k_cg_xr, nb, kCGThreads, s, pl->x, pl->r, pl->p, pl->Ap, P.Mh, (int)P.m, st, part_pAp,
                         part_rr, nrow, (const double *)nullptr));
  } else {
  EFGP_CUFFT(cufftExecZ2D(pl->plan_c2r_L, pl->Xbox, pl->Yr));
  k_mul<<<nblocks(Ld, pl->num_sms), kCGThreads, 0, s>>>(pl->Yr, pl->vhat, Ld, st);
  EFGP_CUFFT(cufftExecD2Z(pl->plan_r2c_L, pl->Yr, pl->Zbox));
  k_cg_apply<D><<<nb, kCGThreads, 0, s>>>(pl->Zbox, pl->p, pl->D_half, pl->Ap, P.Mh, (int)P.m, P.L, st, part_pAp);
  EFGP_CUDA(launch_pdl(k_cg_xr, nb, kCGThreads, s, pl->x, pl->r, pl->p, pl->Ap, P.Mh, (int)P.m, st, part_pAp,
                       part_rr, (int)nb, (const double *)nullptr));
  }
  EFGP_CUDA(launch_pdl(k_cg_p<D>, nb, kCGThreads, s, pl->r, pl->p, pl->D_half, P.Mh, (int)P.m, P.L, pl->Xbox, box,
                       st, part_rr, (int)nb, pl->hist));
  if (!direct)
    EFGP_CUDA(launch_pdl(k_cg_pad<D>, nbox, kCGThreads, s, pl->p, pl->D_half, (int)P.m, P.L, pl->Xbox, box,
                         (const CGState *)st));
  EFGP_CUDA(cudaGetLastError());
  return EFGP_OK;
}

template <int D>
static efgp_status cg_solve_d(efgp_plan *pl, int64_t N_total) {
  const Params &P = pl->P;
  cudaStream_t s = pl->stream;
  int64_t box = P.L / 2 + 1, Ld = P.L;
  for (int k = 0; k < D - 1; ++k) {
    box *= P.L;
    Ld *= P.L;
  }
  const unsigned nb = nblocks(P.Mh, pl->num_sms);
  const unsigned nbox = nblocks(box, pl->num_sms);
  if ((int)nb > pl->cg_blocks) {
    pl->err = "internal: cg partials too small";
    return EFGP_ERR_INVALID;
  }
  int64_t max_iter = P.max_iter_opt;
  if (max_iter <= 0) {
    const double Nd = (double)(N_total > 0 ? N_total : 1);
    max_iter = (int64_t)std::ceil(std::log(1.0 / P.cg_tol) * std::sqrt(Nd) / (2.0 * pl->cap_sigma));
    if (max_iter < 10) max_iter = 10;
  }
  pl->max_iter_used = max_iter;
  EFGP_TRY(ensure_hist(pl, max_iter));
  CGState *st = reinterpret_cast<CGState *>(pl->scal);
  CGState init{};
  init.tol = P.cg_tol;
  init.sigma2 = pl->sigma2_sys;
  init.max_iter = max_iter;
  EFGP_CUDA(cudaMemcpyAsync(st, &init, sizeof(CGState), cudaMemcpyHostToDevice, s));
  k_cg_init<<<nb, kCGThreads, 0, s>>>(pl->b, pl->x, pl->r, pl->p, P.Mh, (int)P.m, pl->partials);
  k_cg_init2<<<1, kCGThreads, 0, s>>>(st, pl->partials, (int)nb, pl->hist);
  k_cg_pad0<D><<<nbox, kCGThreads, 0, s>>>(pl->p, pl->D_half, (int)P.m, P.L, pl->Xbox, box);
  EFGP_CUDA(cudaGetLastError());
  EFGP_CUFFT(cufftSetStream(pl->plan_c2r_L, s));
  EFGP_CUFFT(cufftSetStream(pl->plan_r2c_L, s));
  if (D == 2 && toeplitz_direct(P))
    EFGP_CUDA(cudaFuncSetAttribute(k_cg_toep2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)toep2_smem((int)P.m)));

  const int G = P.graph_iters;
  if (!pl->cg_exec || pl->cg_exec_iters != G) {
    if (pl->cg_exec) cudaGraphExecDestroy(pl->cg_exec);
    pl->cg_exec = nullptr;
    cudaGraph_t graph;
    EFGP_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int it = 0; it < G; ++it) {
      efgp_status e = enqueue_iteration<D>(pl, s, st, box, Ld, nb, nbox);
      if (e != EFGP_OK) {
        cudaStreamEndCapture(s, &graph);
        return e;
      }
    }
    EFGP_CUDA(cudaStreamEndCapture(s, &graph));
    EFGP_CUDA(cudaGraphInstantiate(&pl->cg_exec, graph, 0));
    cudaGraphDestroy(graph);
    pl->cg_exec_iters = G;
  }
  CGState host{};
  for (;;) {
    EFGP_CUDA(cudaGraphLaunch(pl->cg_exec, s));
    EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned, st, sizeof(CGState), cudaMemcpyDeviceToHost, s));
    EFGP_CUDA(cudaStreamSynchronize(s));
    std::memcpy(&host, pl->h_pinned, sizeof(CGState));
    if (host.done) break;
  }
  pl->iters = host.iter;
  pl->rel_resid = host.bnorm > 0 ? std::sqrt(host.rr) / host.bnorm : 0.0;
  return host.done == 2 ? EFGP_ERR_NOCONVERGE : EFGP_OK;
}

// ---- CG with a caller-applied operator (NEXT-3: the product is a type-2 + type-1 NUFFT pair, not a
// Toeplitz product).  Same recurrences and stopping rule (reading G6); host-driven, one small
// device->host read of the state per iteration (each iteration is O(N) work).
__global__ void k_dot_pAp(const double2 *__restrict__ p, const double2 *__restrict__ Ap, int64_t Mh, int m,
                          double *__restrict__ part) {
  __shared__ double sh[40];
  double acc = 0.0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x) {
    const double2 pp = p[q], a = Ap[q];
    const double wq = (q % (m + 1)) ? 2.0 : 1.0;
    acc += wq * (pp.x * a.x + pp.y * a.y);
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

template <int D>
static efgp_status cg_solve_op_d(efgp_plan *pl, int64_t max_iter, CGOp op, void *ctx) {
  const Params &P = pl->P;
  cudaStream_t s = pl->stream;
  const unsigned nb = nblocks(P.Mh, pl->num_sms);
  pl->max_iter_used = max_iter;
  EFGP_TRY(ensure_hist(pl, max_iter));
  CGState *st = reinterpret_cast<CGState *>(pl->scal);
  CGState init{};
  init.tol = P.cg_tol;
  init.max_iter = max_iter;
  double *part_pAp = pl->partials, *part_rr = pl->partials + pl->cg_blocks;
  EFGP_CUDA(cudaMemcpyAsync(st, &init, sizeof(CGState), cudaMemcpyHostToDevice, s));
  k_cg_init<<<nb, kCGThreads, 0, s>>>(pl->b, pl->x, pl->r, pl->p, P.Mh, (int)P.m, pl->partials);
  k_cg_init2<<<1, kCGThreads, 0, s>>>(st, pl->partials, (int)nb, pl->hist);
  EFGP_CUDA(cudaGetLastError());
  CGState host{};
  for (;;) {
    EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned, st, sizeof(CGState), cudaMemcpyDeviceToHost, s));
    EFGP_CUDA(cudaStreamSynchronize(s));
    std::memcpy(&host, pl->h_pinned, sizeof(CGState));
    if (host.done) break;
    EFGP_TRY(op(pl, pl->p, pl->Ap, ctx));
    k_dot_pAp<<<nb, kCGThreads, 0, s>>>(pl->p, pl->Ap, P.Mh, (int)P.m, part_pAp);
    k_cg_xr<<<nb, kCGThreads, 0, s>>>(pl->x, pl->r, pl->p, pl->Ap, P.Mh, (int)P.m, st, part_pAp, part_rr, (int)nb);
    k_cg_p<D><<<nb, kCGThreads, 0, s>>>(pl->r, pl->p, pl->D_half, P.Mh, (int)P.m, P.L, nullptr, 0, st, part_rr,
                                        (int)nb, pl->hist);
    EFGP_CUDA(cudaGetLastError());
  }
  pl->iters = host.iter;
  pl->rel_resid = host.bnorm > 0 ? std::sqrt(host.rr) / host.bnorm : 0.0;
  return host.done == 2 ? EFGP_ERR_NOCONVERGE : EFGP_OK;
}

efgp_status cg_solve_op(efgp_plan *pl, int64_t max_iter, CGOp op, void *ctx) {
  switch (pl->P.d) {
    case 1: return cg_solve_op_d<1>(pl, max_iter, op, ctx);
    case 2: return cg_solve_op_d<2>(pl, max_iter, op, ctx);
    case 3: return cg_solve_op_d<3>(pl, max_iter, op, ctx);
  }
  return EFGP_ERR_INVALID;
}

// PCG x/r update after the direct Toeplitz product: (p, Ap) partials come from its nrow CTAs, (r, z)
// partials from the previous dot over nb CTAs
__global__ void k_cg_xr_pc_direct(double2 *__restrict__ x, double2 *__restrict__ r, const double2 *__restrict__ p,
                                  const double2 *__restrict__ Ap, int64_t Mh, int m, CGState *st,
                                  const double *__restrict__ part_pAp, int npAp, double *__restrict__ part_rr,
                                  const double *__restrict__ part_rz, int nblk) {
  __shared__ double sh[40];
  pdl_wait();
  pdl_trigger();
  if (st->done) return;
  const double pAp = reduce_partials(part_pAp, npAp, sh);
  const double rz = reduce_partials(part_rz, nblk, sh);
  if (blockIdx.x == 0 && threadIdx.x == 0) st->rz = rz;
  const double alpha = rz / pAp;
  double acc = 0.0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x) {
    const double2 pp = p[q], a = Ap[q];
    double2 xx = x[q], rq = r[q];
    xx.x += alpha * pp.x;
    xx.y += alpha * pp.y;
    rq.x -= alpha * a.x;
    rq.y -= alpha * a.y;
    x[q] = xx;
    r[q] = rq;
    acc += ((q % (m + 1)) ? 2.0 : 1.0) * (rq.x * rq.x + rq.y * rq.y);
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part_rr[blockIdx.x] = acc;
}

// ---- NEXT-4: preconditioned CG with the Kronecker preconditioner of precond.cu (reading G12).
// Standard PCG recurrences; the stopping rule and history are those of CG (||r_k|| / ||b||, G6).
__global__ void k_pcg_check(CGState *st, const double *__restrict__ part_rr, int nblk, double *__restrict__ hist) {
  __shared__ double sh[40];
  pdl_wait();
  pdl_trigger();
  if (st->done) return;
  const double rr = reduce_partials(part_rr, nblk, sh);
  if (threadIdx.x == 0) {
    st->rr = rr;
    const long long it = st->iter + 1;
    st->iter = it;
    const double rel = sqrt(rr) / st->bnorm;
    hist[it] = rel;
    if (rel <= st->tol) st->done = 1;
    else if (it >= st->max_iter) st->done = 2;
  }
}

__global__ void k_pcg_dot(const double2 *__restrict__ r, const double2 *__restrict__ z, int64_t Mh, int m,
                          const CGState *st, double *__restrict__ part) {
  __shared__ double sh[40];
  pdl_wait();
  pdl_trigger();
  if (st->done) return;
  double acc = 0.0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x) {
    const double2 a = r[q], b = z[q];
    const double wq = (q % (m + 1)) ? 2.0 : 1.0;
    acc += wq * (a.x * b.x + a.y * b.y);
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// p = z + (rz_new / rz) p   (first == true: p = z)
__global__ void k_pcg_p(const double2 *__restrict__ z, double2 *__restrict__ p, int64_t Mh, const CGState *st,
                        const double *__restrict__ part_rz, int nblk, int first) {
  __shared__ double sh[40];
  pdl_wait();
  pdl_trigger();
  if (st->done) return;
  const double bcg = first ? 0.0 : reduce_partials(part_rz, nblk, sh) / st->rz;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x) {
    const double2 zq = z[q], pp = p[q];
    p[q] = make_double2(zq.x + bcg * pp.x, zq.y + bcg * pp.y);
  }
}

template <int D>
static efgp_status enqueue_pcg_iteration(efgp_plan *pl, cudaStream_t s, CGState *st, int64_t box, int64_t Ld,
                                         unsigned nb, unsigned nbox) {
  const Params &P = pl->P;
  double *part_pAp = pl->partials, *part_rr = pl->partials + pl->cg_blocks, *part_rz = pl->partials + 2 * pl->cg_blocks;
  const bool direct = D == 2 && toeplitz_direct(P);
  if (direct) {
    const int nrow = (int)(2 * P.m + 1);
    k_cg_toep2<<<nrow, kToepThreads, toep2_smem((int)P.m), s>>>(pl->vfull, pl->p, pl->D_half, pl->Ap, (int)P.m, st,
                                                                part_pAp);
    // (x, r update: alpha from the toep2 partials, (r, z) from the previous dot's partials)
    EFGP_CUDA(launch_pdl(k_cg_xr_pc_direct, nb, kCGThreads, s, pl->x, pl->r, pl->p, (const double2 *)pl->Ap, P.Mh,
                         (int)P.m, st, (const double *)part_pAp, nrow, part_rr, (const double *)part_rz, (int)nb));
  } else {
  EFGP_CUFFT(cufftExecZ2D(pl->plan_c2r_L, pl->Xbox, pl->Yr));
  k_mul<<<nblocks(Ld, pl->num_sms), kCGThreads, 0, s>>>(pl->Yr, pl->vhat, Ld, st);
  EFGP_CUFFT(cufftExecD2Z(pl->plan_r2c_L, pl->Yr, pl->Zbox));
  k_cg_apply<D><<<nb, kCGThreads, 0, s>>>(pl->Zbox, pl->p, pl->D_half, pl->Ap, P.Mh, (int)P.m, P.L, st, part_pAp);
  k_cg_xr<<<nb, kCGThreads, 0, s>>>(pl->x, pl->r, pl->p, pl->Ap, P.Mh, (int)P.m, st, part_pAp, part_rr, (int)nb,
                                    part_rz);
  }
  EFGP_CUDA(launch_pdl(k_pcg_check, 1, kCGThreads, s, st, (const double *)part_rr, (int)nb, pl->hist));
  EFGP_TRY(precond_apply(pl, pl->r, pl->z, &st->done, s, true));
  EFGP_CUDA(launch_pdl(k_pcg_dot, nb, kCGThreads, s, (const double2 *)pl->r, (const double2 *)pl->z, P.Mh, (int)P.m,
                       (const CGState *)st, part_rz));
  EFGP_CUDA(launch_pdl(k_pcg_p, nb, kCGThreads, s, (const double2 *)pl->z, pl->p, P.Mh, (const CGState *)st,
                       (const double *)part_rz, (int)nb, 0));
  if (!direct) k_cg_pad<D><<<nbox, kCGThreads, 0, s>>>(pl->p, pl->D_half, (int)P.m, P.L, pl->Xbox, box, st);
  EFGP_CUDA(cudaGetLastError());
  return EFGP_OK;
}

template <int D>
static efgp_status pcg_solve_d(efgp_plan *pl, int64_t N_total) {
  const Params &P = pl->P;
  cudaStream_t s = pl->stream;
  int64_t box = P.L / 2 + 1, Ld = P.L;
  for (int k = 0; k < D - 1; ++k) {
    box *= P.L;
    Ld *= P.L;
  }
  const unsigned nb = nblocks(P.Mh, pl->num_sms);
  const unsigned nbox = nblocks(box, pl->num_sms);
  int64_t max_iter = P.max_iter_opt;
  if (max_iter <= 0) {
    const double Nd = (double)(N_total > 0 ? N_total : 1);
    max_iter = (int64_t)std::ceil(std::log(1.0 / P.cg_tol) * std::sqrt(Nd) / (2.0 * pl->cap_sigma));
    if (max_iter < 10) max_iter = 10;
  }
  pl->max_iter_used = max_iter;
  EFGP_TRY(ensure_hist(pl, max_iter));
  CGState *st = reinterpret_cast<CGState *>(pl->scal);
  CGState init{};
  init.tol = P.cg_tol;
  init.sigma2 = pl->sigma2_sys;
  init.max_iter = max_iter;
  double *part_rz = pl->partials + 2 * pl->cg_blocks;
  EFGP_CUDA(cudaMemcpyAsync(st, &init, sizeof(CGState), cudaMemcpyHostToDevice, s));
  k_cg_init<<<nb, kCGThreads, 0, s>>>(pl->b, pl->x, pl->r, pl->p, P.Mh, (int)P.m, pl->partials);
  k_cg_init2<<<1, kCGThreads, 0, s>>>(st, pl->partials, (int)nb, pl->hist);
  EFGP_TRY(precond_apply(pl, pl->r, pl->z, &st->done, s));          // z0 = M^-1 b
  k_pcg_dot<<<nb, kCGThreads, 0, s>>>(pl->r, pl->z, P.Mh, (int)P.m, st, part_rz);
  k_pcg_p<<<nb, kCGThreads, 0, s>>>(pl->z, pl->p, P.Mh, st, part_rz, (int)nb, 1);  // p0 = z0
  k_cg_pad0<D><<<nbox, kCGThreads, 0, s>>>(pl->p, pl->D_half, (int)P.m, P.L, pl->Xbox, box);
  EFGP_CUDA(cudaGetLastError());
  EFGP_CUFFT(cufftSetStream(pl->plan_c2r_L, s));
  EFGP_CUFFT(cufftSetStream(pl->plan_r2c_L, s));
  if (D == 2 && toeplitz_direct(P))
    EFGP_CUDA(cudaFuncSetAttribute(k_cg_toep2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)toep2_smem((int)P.m)));
  const int G = P.graph_iters;
  if (!pl->pcg_exec || pl->pcg_exec_iters != G || pl->pcg_exec_sigma2 != pl->sigma2_sys) {
    pl->pcg_exec_sigma2 = pl->sigma2_sys;
    if (pl->pcg_exec) cudaGraphExecDestroy(pl->pcg_exec);
    pl->pcg_exec = nullptr;
    cudaGraph_t graph;
    EFGP_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int it = 0; it < G; ++it) {
      efgp_status e = enqueue_pcg_iteration<D>(pl, s, st, box, Ld, nb, nbox);
      if (e != EFGP_OK) {
        cudaStreamEndCapture(s, &graph);
        return e;
      }
    }
    EFGP_CUDA(cudaStreamEndCapture(s, &graph));
    EFGP_CUDA(cudaGraphInstantiate(&pl->pcg_exec, graph, 0));
    cudaGraphDestroy(graph);
    pl->pcg_exec_iters = G;
  }
  CGState host{};
  for (;;) {
    EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned, st, sizeof(CGState), cudaMemcpyDeviceToHost, s));
    EFGP_CUDA(cudaStreamSynchronize(s));
    std::memcpy(&host, pl->h_pinned, sizeof(CGState));
    if (host.done) break;
    EFGP_CUDA(cudaGraphLaunch(pl->pcg_exec, s));
  }
  pl->iters = host.iter;
  pl->rel_resid = host.bnorm > 0 ? std::sqrt(host.rr) / host.bnorm : 0.0;
  return host.done == 2 ? EFGP_ERR_NOCONVERGE : EFGP_OK;
}

efgp_status pcg_solve(efgp_plan *pl, int64_t N_total) {
  switch (pl->P.d) {
    case 1: return pcg_solve_d<1>(pl, N_total);
    case 2: return pcg_solve_d<2>(pl, N_total);
    case 3: return pcg_solve_d<3>(pl, N_total);
  }
  return EFGP_ERR_INVALID;
}

efgp_status cg_solve(efgp_plan *pl, int64_t N_total) {
  switch (pl->P.d) {
    case 1: return cg_solve_d<1>(pl, N_total);
    case 2: return cg_solve_d<2>(pl, N_total);
    case 3: return cg_solve_d<3>(pl, N_total);
  }
  return EFGP_ERR_INVALID;
}

}  // namespace efgp
