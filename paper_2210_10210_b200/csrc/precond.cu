// NEXT-4: Kronecker preconditioner for the weight-space CG ("combining EFGP
// with efficient (Kronecker-structure) Toeplitz preconditioners"; reading G12).
//
//   M = A_1 (x) ... (x) A_d + sigma^2 I,   A_i = diag(delta_i) T(v^(i)) diag(delta_i) / N^((d-1)/d),
//   v^(i)_l = v_{l e_i},  delta_i(j) = D_{j e_i} / D_0^((d-1)/d),  N = v_0.
//
// Setup (once per fit, after the Toeplitz vector v is known): the d factors (2m+1)^2 are built on the
// host from the axis lines of v and D and eigen-decomposed on the device (cuSOLVER zheevd):
// A_i = Q_i Lambda_i Q_i^*.  Apply (every PCG iteration):
//   M^-1 r = (Q_1 (x) ... (x) Q_d) (Lambda_1 (x) ... + sigma^2)^-1 (Q_1 (x) ... (x) Q_d)^* r
// on the full (2m+1)^d grid: expand the Hermitian half, d axis passes with Q^*, a diagonal scale, d
// axis passes with Q, extract the half (M maps Hermitian-symmetric vectors to Hermitian-symmetric
// vectors: T(v)_{-p,-q} = conj T(v)_{p,q}, D even).  Each axis pass is a small dense contraction
// ((2m+1) terms per output, <= 0.1 GFLOP for c4) done by a warp per output element.
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <vector>

#include "efgp_internal.cuh"

namespace efgp {

namespace {

int64_t ipow_(int64_t b, int e) {
  int64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

// index of mode j (|j_k| <= K) in a Hermitian-half array (j_d >= 0), row-major (j_1+K, ..., j_d)
int64_t half_index(const int *j, int d, int64_t K) {
  int64_t idx = 0;
  for (int k = 0; k < d - 1; ++k) idx = idx * (2 * K + 1) + (j[k] + K);
  return idx * (K + 1) + j[d - 1];
}

}  // namespace

// full[(j_1+m) ... (j_d+m)] <- half (conjugate symmetric completion)
template <int D>
__global__ void k_pc_expand(const double2 *__restrict__ half, int m, double2 *__restrict__ full, int64_t total,
                            const int *__restrict__ done) {
  if (done && *done) return;
  const int n = 2 * m + 1;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int j[D];
    int64_t rem = idx;
#pragma unroll
    for (int k = D - 1; k >= 0; --k) {
      j[k] = (int)(rem % n) - m;
      rem /= n;
    }
    bool neg = j[D - 1] < 0;
    if (neg) {
#pragma unroll
      for (int k = 0; k < D; ++k) j[k] = -j[k];
    }
    const double2 v = half[encode_half<D>(j, m)];
    full[idx] = neg ? make_double2(v.x, -v.y) : v;
  }
}

template <int D>
__global__ void k_pc_extract(const double2 *__restrict__ full, int m, double2 *__restrict__ half, int64_t Mh,
                             const int *__restrict__ done) {
  if (done && *done) return;
  const int n = 2 * m + 1;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x) {
    int j[D];
    decode_half<D>(q, m, j);
    int64_t idx = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) idx = idx * n + (j[k] + m);
    half[q] = full[idx];
  }
}

// out[.., j, ..] = sum_k Op[j, k] in[.., k, ..] along one axis (stride = n^(d-1-axis)), one warp per
// output element (lanes split the k sum, shuffle reduction): the sums are short ((2m+1) terms) and a
// thread-per-output loop is a chain of dependent L2 loads (20 us per pass on c3).
// V holds the eigenvectors column-major (V[k n + p] = Q_{p k}).  ADJ: Op = Q^* (Op[j,k] = conj Q_{k j});
// otherwise Op = Q.
template <bool ADJ>
__global__ void k_pc_axis(const double2 *__restrict__ in, double2 *__restrict__ out, const double2 *__restrict__ V,
                          int n, int64_t stride, int64_t total, const int *__restrict__ done) {
  if (done && *done) return;
  const int lane = threadIdx.x & 31;
  for (int64_t idx = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; idx < total;
       idx += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int j = (int)((idx / stride) % n);
    const int64_t base = idx - (int64_t)j * stride;
    double re = 0.0, im = 0.0;
    for (int k = lane; k < n; k += 32) {
      const double2 q = ADJ ? V[(int64_t)j * n + k] : V[(int64_t)k * n + j];
      const double2 z = in[base + (int64_t)k * stride];
      const double qy = ADJ ? -q.y : q.y;  // conj(q) z or q z
      re = fma(q.x, z.x, fma(-qy, z.y, re));
      im = fma(q.x, z.y, fma(qy, z.x, im));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      re += __shfl_xor_sync(0xffffffffu, re, o);
      im += __shfl_xor_sync(0xffffffffu, im, o);
    }
    if (lane == 0) out[idx] = make_double2(re, im);
  }
}

// z /= prod_i lambda_i(j_i) + sigma^2
template <int D>
__global__ void k_pc_scale(double2 *__restrict__ z, const double *__restrict__ lam, int n, double sigma2, int64_t total,
                           const int *__restrict__ done) {
  if (done && *done) return;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = idx;
    double p = 1.0;
#pragma unroll
    for (int k = D - 1; k >= 0; --k) {
      p *= lam[k * n + (int)(rem % n)];
      rem /= n;
    }
    const double s = 1.0 / (p + sigma2);
    const double2 v = z[idx];
    z[idx] = make_double2(v.x * s, v.y * s);
  }
}



// One axis pass with the neighbouring steps fused (fewer launches per PCG iteration): IN_HALF reads the
// input from the Hermitian half (conjugate completion) instead of an expanded grid, SCALE divides the
// output by prod lambda + sigma^2, OUT_HALF writes only the Hermitian-half entries (the extract).
template <int D, bool ADJ, bool IN_HALF, bool SCALE, bool OUT_HALF>
__global__ void k_pc_axis_f(const double2 *__restrict__ in, double2 *__restrict__ out, const double2 *__restrict__ V,
                            int m, int64_t stride, int64_t total, const double *__restrict__ lam, double sigma2,
                            const int *__restrict__ done) {
  pdl_wait();
  pdl_trigger();
  if (done && *done) return;
  const int n = 2 * m + 1;
  const int lane = threadIdx.x & 31;
  for (int64_t idx = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; idx < total;
       idx += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int j = (int)((idx / stride) % n);
    const int64_t base = idx - (int64_t)j * stride;
    double re = 0.0, im = 0.0;
    for (int k = lane; k < n; k += 32) {
      const double2 q = ADJ ? V[(int64_t)j * n + k] : V[(int64_t)k * n + j];
      double2 zv;
      const int64_t fi = base + (int64_t)k * stride;
      if constexpr (IN_HALF) {
        int jj[D];
        int64_t rem = fi;
#pragma unroll
        for (int c = D - 1; c >= 0; --c) {
          jj[c] = (int)(rem % n) - m;
          rem /= n;
        }
        const bool neg = jj[D - 1] < 0;
        if (neg) {
#pragma unroll
          for (int c = 0; c < D; ++c) jj[c] = -jj[c];
        }
        const double2 h = in[encode_half<D>(jj, m)];
        zv = neg ? make_double2(h.x, -h.y) : h;
      } else {
        zv = in[fi];
      }
      const double qy = ADJ ? -q.y : q.y;  // conj(q) z or q z
      re = fma(q.x, zv.x, fma(-qy, zv.y, re));
      im = fma(q.x, zv.y, fma(qy, zv.x, im));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      re += __shfl_xor_sync(0xffffffffu, re, o);
      im += __shfl_xor_sync(0xffffffffu, im, o);
    }
    if (lane == 0) {
      int jj[D];
      int64_t rem = idx;
#pragma unroll
      for (int c = D - 1; c >= 0; --c) {
        jj[c] = (int)(rem % n);
        rem /= n;
      }
      if constexpr (SCALE) {
        double pr = 1.0;
#pragma unroll
        for (int c = 0; c < D; ++c) pr *= lam[c * n + jj[c]];
        const double sc = 1.0 / (pr + sigma2);
        re *= sc;
        im *= sc;
      }
      if constexpr (OUT_HALF) {
        if (jj[D - 1] >= m) {  // j_d >= 0
#pragma unroll
          for (int c = 0; c < D; ++c) jj[c] -= m;
          out[encode_half<D>(jj, m)] = make_double2(re, im);
        }
      } else {
        out[idx] = make_double2(re, im);
      }
    }
  }
}


// Jacobi (reading G12b): diag_q = D_q^2 v_0 + sigma^2 on the Hermitian half; z = r / diag
template <int D>
__global__ void k_jacobi_diag(const double2 *__restrict__ vh, const double *__restrict__ Dh, int64_t Mh, int m,
                              double sigma2, double *__restrict__ diag) {
  int j0[D];
#pragma unroll
  for (int k = 0; k < D; ++k) j0[k] = 0;
  const double v0 = vh[encode_half<D>(j0, 2 * m)].x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x)
    diag[q] = Dh[q] * Dh[q] * v0 + sigma2;
}

__global__ void k_pc_jacobi(const double2 *__restrict__ r, double2 *__restrict__ z, const double *__restrict__ diag,
                            int64_t Mh, const int *__restrict__ done) {
  pdl_wait();
  pdl_trigger();
  if (done && *done) return;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x) {
    const double2 a = r[q];
    const double w = 1.0 / diag[q];
    z[q] = make_double2(a.x * w, a.y * w);
  }
}

static unsigned pc_grid(int64_t n, int sms) {
  int64_t b = (n + 255) / 256;
  const int64_t cap = (int64_t)sms * 8;
  return (unsigned)(b > cap ? cap : (b < 1 ? 1 : b));
}

efgp_status precond_setup(efgp_plan *pl, const double *modes) {
  const Params &P = pl->P;
  if (P.precond == EFGP_PRECOND_JACOBI) {
    if (!pl->pc_diag) EFGP_CUDA(cudaMalloc((void **)&pl->pc_diag, sizeof(double) * P.Mh));
    if (!pl->z) EFGP_CUDA(cudaMalloc((void **)&pl->z, sizeof(double2) * P.Mh));
    const double2 *vh = reinterpret_cast<const double2 *>(modes);
    const unsigned g = pc_grid(P.Mh, pl->num_sms);
    switch (P.d) {
      case 1: k_jacobi_diag<1><<<g, 256, 0, pl->stream>>>(vh, pl->D_half, P.Mh, (int)P.m, pl->sigma2_sys, pl->pc_diag); break;
      case 2: k_jacobi_diag<2><<<g, 256, 0, pl->stream>>>(vh, pl->D_half, P.Mh, (int)P.m, pl->sigma2_sys, pl->pc_diag); break;
      case 3: k_jacobi_diag<3><<<g, 256, 0, pl->stream>>>(vh, pl->D_half, P.Mh, (int)P.m, pl->sigma2_sys, pl->pc_diag); break;
    }
    EFGP_CUDA(cudaGetLastError());
    return EFGP_OK;
  }
  const int d = P.d;
  const int64_t m = P.m, n = 2 * m + 1, K = 2 * m;
  cudaStream_t s = pl->stream;
  // v half (Kvh complex) to the host
  std::vector<std::complex<double>> vh(P.Kvh);
  EFGP_CUDA(cudaMemcpyAsync(vh.data(), modes, sizeof(double2) * P.Kvh, cudaMemcpyDeviceToHost, s));
  EFGP_CUDA(cudaStreamSynchronize(s));
  auto v_at = [&](int axis, int64_t l) {  // v_{l e_axis}
    int j[3] = {0, 0, 0};
    j[axis] = (int)l;
    if (j[d - 1] < 0) {
      for (int k = 0; k < d; ++k) j[k] = -j[k];
      return std::conj(vh[half_index(j, d, K)]);
    }
    return vh[half_index(j, d, K)];
  };
  const double N = v_at(0, 0).real();
  if (!(N > 0)) {
    pl->err = "precond: v_0 (the number of points) is not positive";
    return EFGP_ERR_INVALID;
  }
  const double D0 = std::sqrt(std::pow(P.h, d) * khat_host(P, 0.0));
  const double dpow = (double)(d - 1) / d;
  if (!pl->pc_solver) {
    cusolverDnHandle_t hs;
    if (cusolverDnCreate(&hs) != CUSOLVER_STATUS_SUCCESS) {
      pl->err = "cusolverDnCreate failed";
      return EFGP_ERR_CUDA;
    }
    pl->pc_solver = hs;
  }
  cusolverDnHandle_t hs = static_cast<cusolverDnHandle_t>(pl->pc_solver);
  cusolverDnSetStream(hs, s);
  if (!pl->pc_Q) {
    EFGP_CUDA(cudaMalloc((void **)&pl->pc_Q, sizeof(double2) * d * n * n));
    EFGP_CUDA(cudaMalloc((void **)&pl->pc_lam, sizeof(double) * d * n));
    EFGP_CUDA(cudaMalloc((void **)&pl->pc_F0, sizeof(double2) * ipow_(n, d)));
    EFGP_CUDA(cudaMalloc((void **)&pl->pc_F1, sizeof(double2) * ipow_(n, d)));
    EFGP_CUDA(cudaMalloc((void **)&pl->z, sizeof(double2) * P.Mh));
    EFGP_CUDA(cudaMalloc((void **)&pl->pc_info, sizeof(int)));
  }
  std::vector<std::complex<double>> A(n * n);
  int lwork = 0;
  for (int i = 0; i < d; ++i) {
    std::vector<double> delta(n);
    for (int64_t j = -m; j <= m; ++j)
      delta[j + m] = std::sqrt(std::pow(P.h, d) * khat_host(P, P.h * std::fabs((double)j))) / std::pow(D0, dpow);
    const double sc = 1.0 / std::pow(N, dpow);
    for (int64_t p = 0; p < n; ++p)
      for (int64_t q = 0; q < n; ++q)  // column-major: A[q n + p] = A_pq
        A[q * n + p] = delta[p] * v_at(i, p - q) * delta[q] * sc;
    double2 *Qi = pl->pc_Q + (size_t)i * n * n;
    double *li = pl->pc_lam + (size_t)i * n;
    EFGP_CUDA(cudaMemcpyAsync(Qi, A.data(), sizeof(double2) * n * n, cudaMemcpyHostToDevice, s));
    int lw = 0;
    if (cusolverDnZheevd_bufferSize(hs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)n,
                                    reinterpret_cast<cuDoubleComplex *>(Qi), (int)n, li, &lw) != CUSOLVER_STATUS_SUCCESS) {
      pl->err = "cusolverDnZheevd_bufferSize failed";
      return EFGP_ERR_CUDA;
    }
    if (lw > lwork) {
      if (pl->pc_work) cudaFree(pl->pc_work);
      pl->pc_work = nullptr;
      EFGP_CUDA(cudaMalloc((void **)&pl->pc_work, sizeof(double2) * lw));
      lwork = lw;
    }
    if (cusolverDnZheevd(hs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)n,
                         reinterpret_cast<cuDoubleComplex *>(Qi), (int)n, li,
                         reinterpret_cast<cuDoubleComplex *>(pl->pc_work), lwork, pl->pc_info) != CUSOLVER_STATUS_SUCCESS) {
      pl->err = "cusolverDnZheevd failed";
      return EFGP_ERR_CUDA;
    }
    int info = 0;
    EFGP_CUDA(cudaMemcpyAsync(&info, pl->pc_info, sizeof(int), cudaMemcpyDeviceToHost, s));
    EFGP_CUDA(cudaStreamSynchronize(s));  // (A reused for the next factor)
    if (info != 0) {
      pl->err = "precond: eigen-decomposition did not converge";
      return EFGP_ERR_CUDA;
    }
  }
  return EFGP_OK;
}

// z = M^-1 r on Hermitian halves; kernels return at entry when *done (captured in the CG graph)
template <int D>
static efgp_status precond_apply_d(efgp_plan *pl, const double2 *r, double2 *z, const int *done, cudaStream_t s,
                                   bool pdl) {
  const Params &P = pl->P;
  const int m = (int)P.m, n = 2 * m + 1;
  const int64_t total = ipow_(n, D);
  const unsigned g = pc_grid(total, pl->num_sms);
  const unsigned gw = (unsigned)std::min<int64_t>((total * 32 + 255) / 256, (int64_t)pl->num_sms * 8);
  double2 *a = pl->pc_F0, *b = pl->pc_F1;
  const double2 *Q = pl->pc_Q;
  const double s2 = pl->sigma2_sys;
  const int64_t st0 = total / n;  // axis-0 stride
  // (pdl: the passes are launched as programmatic dependents of their predecessors; they wait before
  // reading anything)
  auto L = [&](auto kern, const double2 *in, double2 *out, const double2 *V, int64_t stride) {
    if (pdl) return launch_pdl(kern, gw, 256, s, in, out, V, m, stride, total, (const double *)pl->pc_lam, s2, done);
    kern<<<gw, 256, 0, s>>>(in, out, V, m, stride, total, pl->pc_lam, s2, done);
    return cudaGetLastError();
  };
  if constexpr (D == 2) {  // 4 fused passes: (half -> Q0^*) (Q1^*, scale) (Q0) (Q1 -> half)
    EFGP_CUDA(L(k_pc_axis_f<2, true, true, false, false>, r, a, Q, st0));
    EFGP_CUDA(L(k_pc_axis_f<2, true, false, true, false>, a, b, Q + (size_t)n * n, 1));
    EFGP_CUDA(L(k_pc_axis_f<2, false, false, false, false>, b, a, Q, st0));
    EFGP_CUDA(L(k_pc_axis_f<2, false, false, false, true>, a, z, Q + (size_t)n * n, 1));
    return EFGP_OK;
  } else if constexpr (D == 1) {  // (half -> Q^*, scale) (Q -> half)
    EFGP_CUDA(L(k_pc_axis_f<1, true, true, true, false>, r, a, Q, 1));
    EFGP_CUDA(L(k_pc_axis_f<1, false, false, false, true>, a, z, Q, 1));
    return EFGP_OK;
  }
  // D = 3: expand, three Q^* passes, scale, three Q passes, extract
  k_pc_expand<D><<<g, 256, 0, s>>>(r, m, a, total, done);
  int64_t stride = total;
  for (int i = 0; i < D; ++i) {
    stride /= n;
    k_pc_axis<true><<<gw, 256, 0, s>>>(a, b, pl->pc_Q + (size_t)i * n * n, n, stride, total, done);
    std::swap(a, b);
  }
  k_pc_scale<D><<<g, 256, 0, s>>>(a, pl->pc_lam, n, pl->sigma2_sys, total, done);
  stride = total;
  for (int i = 0; i < D; ++i) {
    stride /= n;
    k_pc_axis<false><<<gw, 256, 0, s>>>(a, b, pl->pc_Q + (size_t)i * n * n, n, stride, total, done);
    std::swap(a, b);
  }
  k_pc_extract<D><<<pc_grid(P.Mh, pl->num_sms), 256, 0, s>>>(a, m, z, P.Mh, done);
  EFGP_CUDA(cudaGetLastError());
  return EFGP_OK;
}

efgp_status precond_apply(efgp_plan *pl, const double2 *r, double2 *z, const int *done, cudaStream_t s, bool pdl) {
  if (pl->P.precond == EFGP_PRECOND_JACOBI) {
    const unsigned g = pc_grid(pl->P.Mh, pl->num_sms);
    if (pdl) EFGP_CUDA(launch_pdl(k_pc_jacobi, g, 256, s, r, z, (const double *)pl->pc_diag, pl->P.Mh, done));
    else k_pc_jacobi<<<g, 256, 0, s>>>(r, z, pl->pc_diag, pl->P.Mh, done);
    EFGP_CUDA(cudaGetLastError());
    return EFGP_OK;
  }
  switch (pl->P.d) {
    case 1: return precond_apply_d<1>(pl, r, z, done, s, pdl);
    case 2: return precond_apply_d<2>(pl, r, z, done, s, pdl);
    case 3: return precond_apply_d<3>(pl, r, z, done, s, pdl);
  }
  return EFGP_ERR_INVALID;
}

}  // namespace efgp
