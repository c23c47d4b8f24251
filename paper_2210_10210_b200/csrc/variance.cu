// NEXT-2: posterior variance s(x*) = sum_j eta_j phi_j(x*)  (eq "sws") with, per target,
// (Phi^*Phi + sigma^2 I) eta = sigma^2 conj(phi(x*))  (eq "eta"): "an iterative solve
// similar to the above, but with a new right-hand side per target".
//
// Batched CG: B targets at a time share the Toeplitz operator of the last fit (vhat); each
// iteration is one batched C2R, the vhat multiply, one batched R2C (cuFFT, batch B), and one CTA
// per target for the vector part (extract, D, sigma^2, alpha, x, r, beta_cg, p, the padded input of
// the next product).  Each target stops at its own first k with ||r_k|| <= cg_tol ||b|| (reading
// G6); a CUDA graph holds graph_iters iterations and the host polls a device counter of finished
// targets.  phi_j(x) = D_j exp(+2 pi i h j.x) (reading G1); vectors on the Hermitian half j_d >= 0
// (the right-hand side sigma^2 D_j exp(-2 pi i h j.x*) is Hermitian, so eta is).  s is evaluated by
// the direct O(M) sum per target.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "efgp_internal.cuh"

namespace efgp {

constexpr int kVarThreads = 256;
constexpr int kVarMaxM = 256;  // per-dimension phasor tables in shared memory (<= 48 KB)

struct VarTarget {
  double rr, bnorm;
  int iters, done;
  double rz;  // PCG (NEXT-4 preconditioner): (r, z)
};

__device__ __forceinline__ double vblock_sum(double v, double *sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) sh[32] = t;
  }
  __syncthreads();
  return sh[32];
}

// half-vector index q -> signed modes (j_1 .. j_d) (row-major over (j_1+m, ..., j_{d-1}+m, j_d))
template <int D>
__device__ __forceinline__ void half_modes(int64_t q, int m, int (&j)[D]) {
  int64_t rem = q;
  j[D - 1] = (int)(rem % (m + 1));
  rem /= (m + 1);
#pragma unroll
  for (int k = D - 2; k >= 0; --k) {
    j[k] = (int)(rem % (2 * m + 1)) - m;
    rem /= (2 * m + 1);
  }
}

// per-target phasors e^{sgn 2 pi i h j x_k}, j = -m..m, for each dimension, into shared memory
template <int D>
__device__ void phasors(const double *xc, double h, int m, double sgn, double2 *E) {
  for (int idx = threadIdx.x; idx < D * (2 * m + 1); idx += blockDim.x) {
    const int k = idx / (2 * m + 1), j = idx % (2 * m + 1) - m;
    double sv, cv;
    sincospi(sgn * 2.0 * h * (double)j * xc[k], &sv, &cv);
    E[idx] = make_double2(cv, sv);
  }
}

template <int D>
__device__ __forceinline__ double2 phase_of(const double2 *E, int m, const int (&j)[D]) {
  double2 e = E[j[0] + m];
#pragma unroll
  for (int k = 1; k < D; ++k) {
    const double2 f = E[k * (2 * m + 1) + j[k] + m];
    e = make_double2(e.x * f.x - e.y * f.y, e.x * f.y + e.y * f.x);
  }
  return e;
}

// X (C2R input box of one target) = D . p at the J_m bins, 0 elsewhere
template <int D>
__device__ void pad_target(const double2 *__restrict__ p, const double *__restrict__ Dh, int m, int64_t L,
                           double2 *__restrict__ X, int64_t box) {
  const int64_t nh = L / 2 + 1;
  for (int64_t idx = threadIdx.x; idx < box; idx += blockDim.x) {
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


// NEXT-4 inside one CTA (the CTA of one target): z = M^-1 r with the Kronecker factors of the fit
// (precond.cu, reading G12) staged in shared memory: expand the half, d passes with Q^*, scale, d
// passes with Q, extract; every thread carries up to 4 outputs per pass (independent FMA chains).
// smem: Q (d n^2) | A | B (n^d each), double2.
template <int D>
__device__ void pc_apply_cta(const double2 *__restrict__ r, double2 *__restrict__ z, int m, double2 *Q, double2 *A,
                             double2 *Bf, const double *__restrict__ lam, double sigma2, int64_t Mh) {
  const int n = 2 * m + 1;
  const int total = D == 1 ? n : n * n;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    int j[D];
    int rem = idx;
#pragma unroll
    for (int k = D - 1; k >= 0; --k) {
      j[k] = rem % n - m;
      rem /= n;
    }
    const bool neg = j[D - 1] < 0;
    if (neg) {
#pragma unroll
      for (int k = 0; k < D; ++k) j[k] = -j[k];
    }
    int64_t q = j[D - 1];
    if (D == 2) q += (int64_t)(j[0] + m) * (m + 1);
    const double2 v = r[q];
    A[idx] = neg ? make_double2(v.x, -v.y) : v;
  }
  __syncthreads();
  double2 *a = A, *b = Bf;
  for (int phase = 0; phase < 2; ++phase) {
    int stride = total;
    for (int ax = 0; ax < D; ++ax) {
      stride /= n;
      const double2 *V = Q + ax * n * n;
      const bool adj = phase == 0;
      for (int base0 = 0; base0 < total; base0 += 4 * blockDim.x) {
        int jj[4], bb[4];
        double re[4], im[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int idx = base0 + threadIdx.x + t * blockDim.x;
          const int ic = idx < total ? idx : 0;
          jj[t] = (ic / stride) % n;
          bb[t] = ic - jj[t] * stride;
          re[t] = im[t] = 0.0;
        }
        for (int k = 0; k < n; ++k) {
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const double2 qv = adj ? V[jj[t] * n + k] : V[k * n + jj[t]];
            const double2 av = a[bb[t] + k * stride];
            const double qy = adj ? -qv.y : qv.y;
            re[t] = fma(qv.x, av.x, fma(-qy, av.y, re[t]));
            im[t] = fma(qv.x, av.y, fma(qy, av.x, im[t]));
          }
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int idx = base0 + threadIdx.x + t * blockDim.x;
          if (idx < total) b[idx] = make_double2(re[t], im[t]);
        }
      }
      __syncthreads();
      double2 *tmp = a;
      a = b;
      b = tmp;
    }
    if (phase == 0) {
      for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
        double pr = lam[(D - 1) * n + idx % n];
        if (D == 2) pr *= lam[idx / n];
        const double sc = 1.0 / (pr + sigma2);
        a[idx] = make_double2(a[idx].x * sc, a[idx].y * sc);
      }
      __syncthreads();
    }
  }
  for (int64_t q = threadIdx.x; q < Mh; q += blockDim.x) {
    int j[D];
    half_modes<D>(q, m, j);
    int idx = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) idx = idx * n + (j[k] + m);
    z[q] = a[idx];
  }
  __syncthreads();
}

// stage the d factors into shared memory
template <int D>
__device__ __forceinline__ void pc_load_q(const double2 *__restrict__ Qg, int m, double2 *Q) {
  const int n = 2 * m + 1;
  for (int i = threadIdx.x; i < D * n * n; i += blockDim.x) Q[i] = Qg[i];
}

// rhs = sigma^2 conj(phi(x*)) = sigma^2 D_j e^{-2 pi i h j.x*}; x = 0; r = p = rhs; first C2R input
template <int D, int PC>  // PC: 0 plain CG, 1 Kronecker (G12), 2 Jacobi (G12b)
__global__ void __launch_bounds__(kVarThreads) k_var_init(const double *__restrict__ xt, int nt, double h, int m,
                                                          double sigma2, const double *__restrict__ Dh, int64_t Mh,
                                                          int64_t L, int64_t box, double2 *__restrict__ vx,
                                                          double2 *__restrict__ vr, double2 *__restrict__ vp,
                                                          double2 *__restrict__ X, VarTarget *__restrict__ st,
                                                          unsigned *__restrict__ ndone, int *__restrict__ err,
                                                          const double2 *__restrict__ pcQ, const double *__restrict__ pcl) {
  extern __shared__ double2 E[];
  __shared__ double sh[40];
  const int t = blockIdx.x;
  double2 *x = vx + (int64_t)t * Mh, *r = vr + (int64_t)t * Mh, *p = vp + (int64_t)t * Mh;
  bool active = t < nt;
  double xc[D];
  if (active) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      xc[k] = xt[(int64_t)t * D + k];
      active = active && xc[k] >= 0.0 && xc[k] <= 1.0;  // false for NaN
    }
    if (!active && threadIdx.x == 0) atomicOr(err + 1, 1);
  }
  if (active) phasors<D>(xc, h, m, -1.0, E);
  __syncthreads();
  double acc = 0.0;
  for (int64_t q = threadIdx.x; q < Mh; q += blockDim.x) {
    double2 b = make_double2(0.0, 0.0);
    int j[D];
    half_modes<D>(q, m, j);
    if (active) {
      const double2 e = phase_of<D>(E, m, j);
      const double s = sigma2 * Dh[q];
      b = make_double2(s * e.x, s * e.y);
    }
    x[q] = make_double2(0.0, 0.0);
    r[q] = b;
    p[q] = b;
    acc += (j[D - 1] ? 2.0 : 1.0) * (b.x * b.x + b.y * b.y);
  }
  const double rr = vblock_sum(acc, sh);
  __syncthreads();
  double rz = rr;
  if constexpr (PC) {  // p0 = z0 = M^-1 r0
    if constexpr (PC == 2) {
      for (int64_t q = threadIdx.x; q < Mh; q += blockDim.x) {
        const double2 a = r[q];
        const double w = 1.0 / pcl[q];
        p[q] = make_double2(a.x * w, a.y * w);
      }
    } else {
      const int n = 2 * m + 1, total = D == 1 ? n : n * n;
      double2 *Q = E + D * n, *A = Q + D * n * n, *Bf = A + total;
      pc_load_q<D>(pcQ, m, Q);
      __syncthreads();
      pc_apply_cta<D>(r, p, m, Q, A, Bf, pcl, sigma2, Mh);
    }
    acc = 0.0;
    for (int64_t q = threadIdx.x; q < Mh; q += blockDim.x) {
      const double2 a = r[q], z = p[q];
      acc += ((q % (m + 1)) ? 2.0 : 1.0) * (a.x * z.x + a.y * z.y);
    }
    rz = vblock_sum(acc, sh);
    __syncthreads();
  }
  pad_target<D>(p, Dh, m, L, X + (int64_t)t * box, box);
  if (threadIdx.x == 0) {
    st[t].rz = rz;
    st[t].rr = rr;
    st[t].bnorm = sqrt(rr);
    st[t].iters = 0;
    const int done = (!active || rr == 0.0) ? 1 : 0;
    st[t].done = done;
    if (done) atomicAdd(ndone, 1u);
  }
}

__global__ void k_var_mul(double *__restrict__ Y, const double *__restrict__ vhat, int64_t Ld, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    Y[i] *= vhat[i % Ld];
}

// one CG iteration of one target (CTA = target)
template <int D, int PC>  // PC: 0 plain CG, 1 Kronecker (G12), 2 Jacobi (G12b)
__global__ void __launch_bounds__(kVarThreads) k_var_step(const double2 *__restrict__ Zall, const double *__restrict__ Dh,
                                                          int64_t Mh, int m, int64_t L, int64_t box, double sigma2,
                                                          double tol, int max_iter, double2 *__restrict__ vx,
                                                          double2 *__restrict__ vr, double2 *__restrict__ vp,
                                                          double2 *__restrict__ vAp, double2 *__restrict__ X,
                                                          VarTarget *__restrict__ st, unsigned *__restrict__ ndone,
                                                          const double2 *__restrict__ pcQ, const double *__restrict__ pcl) {
  extern __shared__ double2 pcsm[];  // PC: Q | A | B
  __shared__ double sh[40];
  const int t = blockIdx.x;
  if (st[t].done) return;
  const double2 *Z = Zall + (int64_t)t * box;
  double2 *x = vx + (int64_t)t * Mh, *r = vr + (int64_t)t * Mh, *p = vp + (int64_t)t * Mh, *Ap = vAp + (int64_t)t * Mh;
  const double rr = st[t].rr;
  const double num = PC ? st[t].rz : rr;  // alpha = (r, z) / (p, Ap); plain CG: z = r
  double acc = 0.0;
  for (int64_t q = threadIdx.x; q < Mh; q += blockDim.x) {
    int j[D];
    half_modes<D>(q, m, j);
    int64_t zi = j[D - 1], stride = L / 2 + 1;
#pragma unroll
    for (int k = D - 2; k >= 0; --k) {
      zi += (j[k] < 0 ? j[k] + L : j[k]) * stride;
      stride *= L;
    }
    const double2 z = Z[zi], pp = p[q];
    const double dq = Dh[q];
    const double2 a = make_double2(dq * z.x + sigma2 * pp.x, dq * z.y + sigma2 * pp.y);
    Ap[q] = a;
    acc += (j[D - 1] ? 2.0 : 1.0) * (pp.x * a.x + pp.y * a.y);
  }
  const double alpha = num / vblock_sum(acc, sh);
  acc = 0.0;
  for (int64_t q = threadIdx.x; q < Mh; q += blockDim.x) {
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
  const double rr_new = vblock_sum(acc, sh);
  const int it = st[t].iters + 1;
  const bool fin = sqrt(rr_new) <= tol * st[t].bnorm || it >= max_iter;
  if constexpr (PC) {
    if (!fin) {  // z = M^-1 r into the (now free) Ap buffer; p = z + ((r,z)_new / (r,z)) p
      if constexpr (PC == 2) {
        for (int64_t q = threadIdx.x; q < Mh; q += blockDim.x) {
          const double2 a = r[q];
          const double w = 1.0 / pcl[q];
          Ap[q] = make_double2(a.x * w, a.y * w);
        }
      } else {
        const int n = 2 * m + 1, total = D == 1 ? n : n * n;
        double2 *Q = pcsm, *A = Q + D * n * n, *Bf = A + total;
        __syncthreads();
        pc_load_q<D>(pcQ, m, Q);
        __syncthreads();
        pc_apply_cta<D>(r, Ap, m, Q, A, Bf, pcl, sigma2, Mh);
      }
      acc = 0.0;
      for (int64_t q = threadIdx.x; q < Mh; q += blockDim.x) {
        const double2 a = r[q], z = Ap[q];
        acc += ((q % (m + 1)) ? 2.0 : 1.0) * (a.x * z.x + a.y * z.y);
      }
      const double rz_new = vblock_sum(acc, sh);
      const double bcg = rz_new / num;
      for (int64_t q = threadIdx.x; q < Mh; q += blockDim.x) {
        const double2 zq = Ap[q], pp = p[q];
        p[q] = make_double2(zq.x + bcg * pp.x, zq.y + bcg * pp.y);
      }
      if (threadIdx.x == 0) st[t].rz = rz_new;
    }
  } else {
    const double bcg = rr_new / rr;
    for (int64_t q = threadIdx.x; q < Mh; q += blockDim.x) {
      const double2 rq = r[q], pp = p[q];
      p[q] = make_double2(rq.x + bcg * pp.x, rq.y + bcg * pp.y);
    }
  }
  __syncthreads();
  if (!fin) pad_target<D>(p, Dh, m, L, X + (int64_t)t * box, box);
  if (threadIdx.x == 0) {
    st[t].rr = rr_new;
    st[t].iters = it;
    if (fin) {
      st[t].done = 1;
      atomicAdd(ndone, 1u);
    }
  }
}

// s(x*) = Re sum_j eta_j phi_j(x*) over J_m = sum over the half with weight 1 (j_d = 0) or 2
template <int D>
__global__ void __launch_bounds__(kVarThreads) k_var_eval(const double *__restrict__ xt, int nt, double h, int m,
                                                          const double *__restrict__ Dh, int64_t Mh,
                                                          const double2 *__restrict__ vx,
                                                          const VarTarget *__restrict__ st, double *__restrict__ out) {
  extern __shared__ double2 E[];
  __shared__ double sh[40];
  const int t = blockIdx.x;
  if (t >= nt) return;
  double xc[D];
  bool ok = true;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    xc[k] = xt[(int64_t)t * D + k];
    ok = ok && xc[k] >= 0.0 && xc[k] <= 1.0;
  }
  if (!ok) {
    if (threadIdx.x == 0) out[t] = __longlong_as_double(0x7ff8000000000000LL);
    return;
  }
  phasors<D>(xc, h, m, +1.0, E);
  __syncthreads();
  const double2 *eta = vx + (int64_t)t * Mh;
  double acc = 0.0;
  for (int64_t q = threadIdx.x; q < Mh; q += blockDim.x) {
    int j[D];
    half_modes<D>(q, m, j);
    const double2 e = phase_of<D>(E, m, j), n = eta[q];
    acc += (j[D - 1] ? 2.0 : 1.0) * Dh[q] * (n.x * e.x - n.y * e.y);
  }
  const double s = vblock_sum(acc, sh);
  if (threadIdx.x == 0) out[t] = s;
}

static void free_var(efgp_plan *pl) {
  if (pl->var_exec) cudaGraphExecDestroy(pl->var_exec);
  pl->var_exec = nullptr;
  for (cufftHandle *h : {&pl->plan_var_c2r, &pl->plan_var_r2c})
    if (*h) {
      cufftDestroy(*h);
      *h = 0;
    }
  for (void **b : {(void **)&pl->var_x, (void **)&pl->var_r, (void **)&pl->var_p, (void **)&pl->var_Ap,
                   (void **)&pl->var_X, (void **)&pl->var_Z, (void **)&pl->var_Y, &pl->var_st})
    if (*b) {
      cudaFree(*b);
      *b = nullptr;
    }
  pl->var_B = 0;
}

// batch of targets per CG: the call's q (rounded up to 16), within min(8 GB, free / 4) of buffers
// (c4's 3D boxes are ~95 MB per target: a fixed 768 MB budget allowed 8 targets per batch); every
// batched FFT runs B wide, so B is not larger than the work (q) either
template <int D>
static int64_t var_batch_size(const efgp_plan *pl, int64_t q) {
  const Params &P = pl->P;
  int64_t box = P.L / 2 + 1, Ld = P.L;
  for (int k = 0; k < D - 1; ++k) {
    box *= P.L;
    Ld *= P.L;
  }
  const int64_t per = 4 * P.Mh * 16 + 2 * box * 16 + Ld * 8 + 64;
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
    cudaGetLastError();
    free_b = size_t(4) << 30;
  }
  const int64_t budget = std::min<int64_t>(int64_t(8) << 30, (int64_t)(free_b / 4) + (int64_t)pl->var_B * per);
  int64_t B = std::max<int64_t>(1, std::min<int64_t>({int64_t(2048), budget / per, (q + 15) / 16 * 16}));
  if (const char *e = std::getenv("EFGP_VAR_BATCH")) B = std::max<int64_t>(1, std::min<int64_t>(B, std::atoll(e)));
  return B;
}

template <int D>
static efgp_status setup_var(efgp_plan *pl, int64_t Bwant) {
  const Params &P = pl->P;
  int64_t box = P.L / 2 + 1, Ld = P.L;
  for (int k = 0; k < D - 1; ++k) {
    box *= P.L;
    Ld *= P.L;
  }
  const int64_t B = Bwant;
  pl->var_B = (int)B;
  EFGP_CUDA(cudaMalloc((void **)&pl->var_x, B * P.Mh * 16));
  EFGP_CUDA(cudaMalloc((void **)&pl->var_r, B * P.Mh * 16));
  EFGP_CUDA(cudaMalloc((void **)&pl->var_p, B * P.Mh * 16));
  EFGP_CUDA(cudaMalloc((void **)&pl->var_Ap, B * P.Mh * 16));
  EFGP_CUDA(cudaMalloc((void **)&pl->var_X, B * box * 16));
  EFGP_CUDA(cudaMalloc((void **)&pl->var_Z, B * box * 16));
  EFGP_CUDA(cudaMalloc((void **)&pl->var_Y, B * Ld * 8));
  EFGP_CUDA(cudaMalloc((void **)&pl->var_st, B * sizeof(VarTarget) + 64));
  int dims[3] = {(int)P.L, (int)P.L, (int)P.L};
  EFGP_CUFFT(cufftPlanMany(&pl->plan_var_c2r, D, dims, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2D, (int)B));
  EFGP_CUFFT(cufftPlanMany(&pl->plan_var_r2c, D, dims, nullptr, 1, 0, nullptr, 1, 0, CUFFT_D2Z, (int)B));
  return EFGP_OK;
}

template <int D>
static efgp_status var_batch(efgp_plan *pl, const double *xt, int nt, double *out, cudaStream_t s, int *iters_max,
                             int64_t *noconv) {
  const Params &P = pl->P;
  int64_t box = P.L / 2 + 1, Ld = P.L;
  for (int k = 0; k < D - 1; ++k) {
    box *= P.L;
    Ld *= P.L;
  }
  const int B = pl->var_B;
  VarTarget *st = reinterpret_cast<VarTarget *>(pl->var_st);
  unsigned *ndone = reinterpret_cast<unsigned *>(reinterpret_cast<char *>(pl->var_st) + B * sizeof(VarTarget));
  const size_t esm = sizeof(double2) * D * (2 * P.m + 1);
  const double sigma2 = pl->sigma2_sys;  // sigma^2, or 1 after a heteroskedastic Toeplitz fit (G11b)
  // NEXT-4 in the variance CGs: the fit's Kronecker factors, applied per target inside its CTA
  const int64_t n = 2 * P.m + 1, total = D == 1 ? n : n * n;
  const size_t pcsm = sizeof(double2) * (D * n * n + 2 * total);
  const int pc = pl->pc_used == EFGP_PRECOND_JACOBI && pl->pc_diag
                     ? 2
                     : (D <= 2 && pl->pc_used == EFGP_PRECOND_KRON && pl->pc_Q && esm + pcsm <= 200 * 1024 ? 1 : 0);
  pl->var_pc = pc;
  EFGP_CUDA(cudaMemsetAsync(ndone, 0, sizeof(unsigned), s));
  if (pc == 2) {
    k_var_init<D, 2><<<B, kVarThreads, esm, s>>>(xt, nt, P.h, (int)P.m, sigma2, pl->D_half, P.Mh, P.L, box, pl->var_x,
                                                 pl->var_r, pl->var_p, pl->var_X, st, ndone, pl->dflags, nullptr,
                                                 pl->pc_diag);
  } else if (pc) {
    EFGP_CUDA(cudaFuncSetAttribute(k_var_init<D, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(esm + pcsm)));
    EFGP_CUDA(cudaFuncSetAttribute(k_var_step<D, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pcsm));
    k_var_init<D, 1><<<B, kVarThreads, esm + pcsm, s>>>(xt, nt, P.h, (int)P.m, sigma2, pl->D_half, P.Mh, P.L, box,
                                                           pl->var_x, pl->var_r, pl->var_p, pl->var_X, st, ndone,
                                                           pl->dflags, pl->pc_Q, pl->pc_lam);
  } else {
    k_var_init<D, 0><<<B, kVarThreads, esm, s>>>(xt, nt, P.h, (int)P.m, sigma2, pl->D_half, P.Mh, P.L, box,
                                                     pl->var_x, pl->var_r, pl->var_p, pl->var_X, st, ndone, pl->dflags,
                                                     nullptr, nullptr);
  }
  EFGP_CUDA(cudaGetLastError());
  EFGP_CUFFT(cufftSetStream(pl->plan_var_c2r, s));
  EFGP_CUFFT(cufftSetStream(pl->plan_var_r2c, s));
  const int max_iter = (int)std::min<int64_t>(pl->max_iter_used > 0 ? pl->max_iter_used : 1000, 1 << 30);
  if (pl->var_exec && (pl->var_exec_pc != (int)pc || pl->var_exec_sigma2 != sigma2)) {
    cudaGraphExecDestroy(pl->var_exec);
    pl->var_exec = nullptr;
  }
  if (!pl->var_exec) {
    pl->var_exec_pc = (int)pc;
    pl->var_exec_sigma2 = sigma2;
    cudaGraph_t graph;
    EFGP_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int it = 0; it < P.graph_iters; ++it) {
      cufftExecZ2D(pl->plan_var_c2r, pl->var_X, pl->var_Y);
      k_var_mul<<<pl->num_sms * 4, 256, 0, s>>>(pl->var_Y, pl->vhat, Ld, Ld * B);
      cufftExecD2Z(pl->plan_var_r2c, pl->var_Y, pl->var_Z);
      if (pc == 2)
        k_var_step<D, 2><<<B, kVarThreads, 0, s>>>(pl->var_Z, pl->D_half, P.Mh, (int)P.m, P.L, box, sigma2, P.cg_tol,
                                                   max_iter, pl->var_x, pl->var_r, pl->var_p, pl->var_Ap, pl->var_X,
                                                   st, ndone, nullptr, pl->pc_diag);
      else if (pc)
        k_var_step<D, 1><<<B, kVarThreads, pcsm, s>>>(pl->var_Z, pl->D_half, P.Mh, (int)P.m, P.L, box, sigma2,
                                                         P.cg_tol, max_iter, pl->var_x, pl->var_r, pl->var_p,
                                                         pl->var_Ap, pl->var_X, st, ndone, pl->pc_Q, pl->pc_lam);
      else
        k_var_step<D, 0><<<B, kVarThreads, 0, s>>>(pl->var_Z, pl->D_half, P.Mh, (int)P.m, P.L, box, sigma2,
                                                       P.cg_tol, max_iter, pl->var_x, pl->var_r, pl->var_p,
                                                       pl->var_Ap, pl->var_X, st, ndone, nullptr, nullptr);
    }
    const cudaError_t ce = cudaStreamEndCapture(s, &graph);
    if (ce != cudaSuccess) {
      pl->err = std::string("variance graph capture: ") + cudaGetErrorString(ce);
      return EFGP_ERR_CUDA;
    }
    EFGP_CUDA(cudaGraphInstantiate(&pl->var_exec, graph, 0));
    cudaGraphDestroy(graph);
    pl->var_exec_max_iter = max_iter;
  }
  for (;;) {
    EFGP_CUDA(cudaGraphLaunch(pl->var_exec, s));
    EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned, ndone, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    EFGP_CUDA(cudaStreamSynchronize(s));
    unsigned nd;
    std::memcpy(&nd, pl->h_pinned, sizeof(nd));
    if (nd >= (unsigned)B) break;
  }
  k_var_eval<D><<<B, kVarThreads, esm, s>>>(xt, nt, P.h, (int)P.m, pl->D_half, P.Mh, pl->var_x, st, out);
  EFGP_CUDA(cudaGetLastError());
  std::vector<VarTarget> host(nt);
  EFGP_CUDA(cudaMemcpyAsync(host.data(), st, sizeof(VarTarget) * nt, cudaMemcpyDeviceToHost, s));
  EFGP_CUDA(cudaStreamSynchronize(s));
  for (const auto &h : host) {
    *iters_max = std::max(*iters_max, h.iters);
    if (h.iters >= max_iter) ++*noconv;  // stopped by the cap, not by cg_tol
  }
  return EFGP_OK;
}

template <int D>
static efgp_status var_targets_d(efgp_plan *pl, const double *xt, int64_t q, double *out, cudaStream_t s) {
  if (pl->P.m > kVarMaxM) {
    pl->err = "posterior variance: m too large for the per-target phasor tables";
    return EFGP_ERR_INVALID;
  }
  const int64_t Bw = var_batch_size<D>(pl, q);
  if (pl->var_x && (Bw > pl->var_B || 4 * Bw < pl->var_B)) free_var(pl);  // resize to the work
  if (!pl->var_x) EFGP_TRY(setup_var<D>(pl, Bw));
  if (pl->var_exec && pl->var_exec_max_iter != (int)std::min<int64_t>(pl->max_iter_used > 0 ? pl->max_iter_used : 1000, 1 << 30)) {
    cudaGraphExecDestroy(pl->var_exec);  // the cap is baked into the graph
    pl->var_exec = nullptr;
  }
  int iters_max = 0;
  int64_t noconv = 0;
  for (int64_t t0 = 0; t0 < q; t0 += pl->var_B) {
    const int nt = (int)std::min<int64_t>(pl->var_B, q - t0);
    EFGP_TRY(var_batch<D>(pl, xt + t0 * D, nt, out + t0, s, &iters_max, &noconv));
  }
  pl->var_iters_max = iters_max;
  if (noconv) {
    pl->err = "predict_var: " + std::to_string(noconv) + " of " + std::to_string(q) +
              " target CGs reached max_iter before cg_tol (their variances are CG iterates)";
    return EFGP_ERR_NOCONVERGE;
  }
  return EFGP_OK;
}

efgp_status variance_targets(efgp_plan *pl, const double *xt, int64_t q, double *out, cudaStream_t s) {
  if (q <= 0) return EFGP_OK;
  switch (pl->P.d) {
    case 1: return var_targets_d<1>(pl, xt, q, out, s);
    case 2: return var_targets_d<2>(pl, xt, q, out, s);
    case 3: return var_targets_d<3>(pl, xt, q, out, s);
  }
  return EFGP_ERR_INVALID;
}

}  // namespace efgp
