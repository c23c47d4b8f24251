// K1: type-1 spreading of the N points onto the fine grids (Alg a1 steps 2-3; the type-1 NUFFTs of
// eqs "88" and "rhs").
//
// Point coordinate theta = 2 pi h x in [0, 2 pi h) with h < 1; in units of the grid spacing
// Delta = 2 pi / n it is t = h x n.  The footprint of a point is the W cells i0 .. i0+W-1 with
// i0 = ceil(t - W/2) per dimension (periodic wrap), weights = the piecewise-polynomial ES kernel
// (es_weights).  Strength 1 goes to g1 (n1^d, modes J_2m) and strength
// y to g2 (n_rhs^d, modes J_m).
//
// Strategies (DESIGN.md §7 "K1"):
//   GLOBAL: one thread per point, fp64 RED into L2 (any d, any grid).
//   SMEM  : one CTA per SM keeps a private copy of the *occupied* part of both grids (cells reachable
//           from x in [0,1]^d) in shared memory, CAS-accumulates, flushes once with RED.
//   SORTED: d = 2, W <= 6, bin-sorted register accumulation (spread_sorted.cu).
//   CELLSORT: d = 2 (any W) or 3 (W <= 6): counting sort by (super-)cell, warp-per-run accumulation
//           with shared-memory weight rows (spread_cellsort.cu).
// Every thread also validates its point (x in [0,1]^d, finite y) and raises dflags[0] otherwise.
#include <cstdio>

#include "efgp_internal.cuh"

namespace efgp {

#define EFGP_W_CASES(MACRO) \
  MACRO(2) MACRO(3) MACRO(4) MACRO(5) MACRO(6) MACRO(7) MACRO(8) MACRO(9) MACRO(10) MACRO(11) MACRO(12) MACRO(13) MACRO(14) MACRO(15) MACRO(16)

template <int D>
__device__ __forceinline__ bool load_point(const double *__restrict__ x, const double *__restrict__ y,
                                           int64_t i, double (&xc)[D], double &yv) {
  bool ok = true;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    xc[k] = __ldg(x + i * D + k);
    ok = ok && (xc[k] >= 0.0) && (xc[k] <= 1.0);  // false for NaN
  }
  yv = __ldg(y + i);
  return ok && isfinite(yv);
}

template <int D, int W>
__device__ __forceinline__ void point_weights(const double (&xc)[D], double h, int n, const EsPoly &P,
                                              int (&base)[D], double (&wt)[D][W]) {
#pragma unroll
  for (int k = 0; k < D; ++k) base[k] = es_weights<W>(h * xc[k] * (double)n, P, wt[k]);
}

__device__ __forceinline__ int wrap(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

template <int D, int W>
__device__ __forceinline__ void add_global(double *__restrict__ g, int n, const int (&base)[D],
                                           const double (&wt)[D][W], double c) {
  if constexpr (D == 1) {
#pragma unroll
    for (int a = 0; a < W; ++a) atomicAdd(g + wrap(base[0] + a, n), c * wt[0][a]);
  } else if constexpr (D == 2) {
#pragma unroll
    for (int a = 0; a < W; ++a) {
      double *row = g + (int64_t)wrap(base[0] + a, n) * n;
      const double ca = c * wt[0][a];
#pragma unroll
      for (int b = 0; b < W; ++b) atomicAdd(row + wrap(base[1] + b, n), ca * wt[1][b]);
    }
  } else {
#pragma unroll 1
    for (int a = 0; a < W; ++a) {
      const double ca = c * wt[0][a];
      const int64_t ia = wrap(base[0] + a, n);
#pragma unroll
      for (int b = 0; b < W; ++b) {
        double *row = g + (ia * n + wrap(base[1] + b, n)) * n;
        const double cab = ca * wt[1][b];
#pragma unroll
        for (int e = 0; e < W; ++e) atomicAdd(row + wrap(base[2] + e, n), cab * wt[2][e]);
      }
    }
  }
}

template <int D, int W>
__global__ void __launch_bounds__(256) k_spread_global(const double *__restrict__ x, const double *__restrict__ y,
                                                       int64_t N, double *__restrict__ g1, int n1,
                                                       double *__restrict__ g2, int n2, double h, EsPoly P,
                                                       int *__restrict__ err) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride) {
    double xc[D], yv;
    if (!load_point<D>(x, y, i, xc, yv)) {
      atomicOr(err, 1);
      continue;
    }
    int base[D];
    double wt[D][W];
    point_weights<D, W>(xc, h, n1, P, base, wt);
    add_global<D, W>(g1, n1, base, wt, 1.0);
    if (n2 != n1) point_weights<D, W>(xc, h, n2, P, base, wt);
    add_global<D, W>(g2, n2, base, wt, yv);
  }
}

// Occupied range of a grid: cells lo .. lo+A-1 (unwrapped) can receive mass from x in [0,1].
struct Occ {
  int lo, A;
};
__host__ __device__ inline Occ occupied(double h, int n, int W) {
  const int lo = -(W / 2);                       // ceil(-W/2)
  const int hi0 = (int)ceil(h * n - 0.5 * W);    // largest first cell (x = 1)
  return Occ{lo, hi0 + W - 1 - lo + 1};
}

template <int D, int W>
__device__ __forceinline__ void add_smem(double *s, int A, int lo, const int (&base)[D], const double (&wt)[D][W],
                                         double c) {
  if constexpr (D == 1) {
#pragma unroll
    for (int a = 0; a < W; ++a) atomicAdd(s + (base[0] + a - lo), c * wt[0][a]);
  } else if constexpr (D == 2) {
#pragma unroll
    for (int a = 0; a < W; ++a) {
      double *row = s + (base[0] + a - lo) * A + (base[1] - lo);
      const double ca = c * wt[0][a];
#pragma unroll
      for (int b = 0; b < W; ++b) atomicAdd(row + b, ca * wt[1][b]);
    }
  } else {
#pragma unroll 1
    for (int a = 0; a < W; ++a) {
      const double ca = c * wt[0][a];
#pragma unroll
      for (int b = 0; b < W; ++b) {
        double *row = s + ((base[0] + a - lo) * A + (base[1] + b - lo)) * A + (base[2] - lo);
        const double cab = ca * wt[1][b];
#pragma unroll
        for (int e = 0; e < W; ++e) atomicAdd(row + e, cab * wt[2][e]);
      }
    }
  }
}

template <int D>
__device__ void flush_smem(const double *s, int A, int lo, double *g, int n) {
  int64_t cells = A;
  for (int k = 1; k < D; ++k) cells *= A;
  for (int64_t c = threadIdx.x; c < cells; c += blockDim.x) {
    const double v = s[c];
    if (v == 0.0) continue;
    int64_t rem = c, gi = 0;
    int idx[D];
#pragma unroll
    for (int k = D - 1; k >= 0; --k) {
      idx[k] = (int)(rem % A);
      rem /= A;
    }
#pragma unroll
    for (int k = 0; k < D; ++k) {
      int i = idx[k] + lo;
      i %= n;
      if (i < 0) i += n;
      gi = gi * n + i;
    }
    atomicAdd(g + gi, v);
  }
}

template <int D, int W>
__global__ void __launch_bounds__(512) k_spread_smem(const double *__restrict__ x, const double *__restrict__ y,
                                                     int64_t N, double *__restrict__ g1, int n1,
                                                     double *__restrict__ g2, int n2, double h, EsPoly P,
                                                     int *__restrict__ err) {
  extern __shared__ double sm[];
  const Occ o1 = occupied(h, n1, W), o2 = occupied(h, n2, W);
  int64_t c1 = o1.A, c2 = o2.A;
  for (int k = 1; k < D; ++k) {
    c1 *= o1.A;
    c2 *= o2.A;
  }
  double *s1 = sm, *s2 = sm + c1;
  for (int64_t c = threadIdx.x; c < c1 + c2; c += blockDim.x) sm[c] = 0.0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride) {
    double xc[D], yv;
    if (!load_point<D>(x, y, i, xc, yv)) {
      atomicOr(err, 1);
      continue;
    }
    int base[D];
    double wt[D][W];
    point_weights<D, W>(xc, h, n1, P, base, wt);
    add_smem<D, W>(s1, o1.A, o1.lo, base, wt, 1.0);
    point_weights<D, W>(xc, h, n2, P, base, wt);
    add_smem<D, W>(s2, o2.A, o2.lo, base, wt, yv);
  }
  __syncthreads();
  flush_smem<D>(s1, o1.A, o1.lo, g1, n1);
  flush_smem<D>(s2, o2.A, o2.lo, g2, n2);
}

static size_t smem_bytes(const Params &P) {
  const Occ o1 = occupied(P.h, (int)P.n1, P.w), o2 = occupied(P.h, (int)P.n2, P.w);
  size_t c1 = o1.A, c2 = o2.A;
  for (int k = 1; k < P.d; ++k) {
    c1 *= o1.A;
    c2 *= o2.A;
  }
  return (c1 + c2) * sizeof(double);
}

void resolve_spread_method(Params &p) {
  int m = p.spread_method;
  // SORTED: 2D, register windows up to 6 x 6, start-cell lookup tables up to 2048 per dimension
  const bool sorted_ok = p.d == 2 && p.w <= 6 && p.h * p.n1 + p.w < 2048 && !p.sorted_disabled;
  const bool smem_ok = smem_bytes(p) <= 200 * 1024;
  int lo, S, ncell;
  const bool cellsort_ok = cellsort_geometry(p, lo, S, ncell);
  const int fallback = cellsort_ok ? EFGP_SPREAD_CELLSORT : (smem_ok ? EFGP_SPREAD_SMEM : EFGP_SPREAD_GLOBAL);
  if (m == EFGP_SPREAD_AUTO) m = sorted_ok ? EFGP_SPREAD_SORTED : fallback;
  if (m == EFGP_SPREAD_SORTED && !sorted_ok) m = fallback;
  if (m == EFGP_SPREAD_CELLSORT && !cellsort_ok) m = smem_ok ? EFGP_SPREAD_SMEM : EFGP_SPREAD_GLOBAL;
  if (m == EFGP_SPREAD_SMEM && !smem_ok) m = EFGP_SPREAD_GLOBAL;
  p.spread_method = m;
  // SORTED and CELLSORT spread both strengths onto the n1 grid (psi1 covers |j| <= 2m >= m)
  p.n_rhs = (m == EFGP_SPREAD_SORTED || m == EFGP_SPREAD_CELLSORT) ? p.n1 : p.n2;
}

template <int D, int W>
static efgp_status launch_spread(efgp_plan *pl, const double *x, const double *y, int64_t N, cudaStream_t s,
                                 int method) {
  const Params &P = pl->P;
  if (method == EFGP_SPREAD_SMEM) {
    const size_t sb = smem_bytes(P);
    EFGP_CUDA(cudaFuncSetAttribute(k_spread_smem<D, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
    k_spread_smem<D, W><<<pl->num_sms, 512, sb, s>>>(x, y, N, pl->g1, (int)P.n1, pl->g2, (int)P.n_rhs, P.h,
                                                     P.poly, pl->dflags);
  } else {
    int64_t blocks = (N + 255) / 256;
    const int64_t cap = (int64_t)pl->num_sms * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    k_spread_global<D, W><<<(unsigned)blocks, 256, 0, s>>>(x, y, N, pl->g1, (int)P.n1, pl->g2, (int)P.n_rhs, P.h,
                                                           P.poly, pl->dflags);
  }
  EFGP_CUDA(cudaGetLastError());
  return EFGP_OK;
}

template <int D>
static efgp_status dispatch_w(efgp_plan *pl, const double *x, const double *y, int64_t N, cudaStream_t s,
                              int method) {
  switch (pl->P.w) {
#define EFGP_CASE(WW) \
  case WW:            \
    return launch_spread<D, WW>(pl, x, y, N, s, method);
    EFGP_W_CASES(EFGP_CASE)
#undef EFGP_CASE
  }
  pl->err = "unsupported ES width";
  return EFGP_ERR_INVALID;
}

efgp_status spread_begin(efgp_plan *pl, cudaStream_t s) {
  const Params &P = pl->P;
  size_t c1 = 1, c2 = 1;
  for (int k = 0; k < P.d; ++k) {
    c1 *= P.n1;
    c2 *= P.n_rhs;
  }
  EFGP_CUDA(cudaMemsetAsync(pl->g1, 0, c1 * sizeof(double), s));
  EFGP_CUDA(cudaMemsetAsync(pl->g2, 0, c2 * sizeof(double), s));
  EFGP_CUDA(cudaMemsetAsync(pl->dflags, 0, sizeof(int) * 4, s));
  pl->spread_used = P.spread_method;
  pl->spread_fallback = EFGP_FALLBACK_NONE;
  return EFGP_OK;
}

efgp_status spread_points(efgp_plan *pl, const double *x, const double *y, int64_t N, cudaStream_t s,
                          const double *s1, unsigned long long *raw_minbits) {
  if (N <= 0) return EFGP_OK;
  int method = pl->P.spread_method;
  if (s1) {  // weighted strength 1: the SORTED kernel's one-pass mode, or CELLSORT; nothing else
    if (method == EFGP_SPREAD_SORTED && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
                                          reinterpret_cast<uintptr_t>(s1)) & 15) == 0)
      return spread_sorted2(pl, x, y, N, s, s1, raw_minbits);
    if (raw_minbits) return EFGP_ERR_RESOURCE;  // raw (y, sigma_n) strengths: the SORTED kernel only
    if (method == EFGP_SPREAD_CELLSORT) return spread_cellsort(pl, x, y, N, s, s1);
    return EFGP_ERR_RESOURCE;
  }
  if (method == EFGP_SPREAD_SORTED) {
    // the binning bulk-copies x and y (16-byte alignment); unaligned inputs fall back to GLOBAL
    // (same grids, same kernel)
    // (same grids, same kernel); the fallback is recorded in efgp_info.spread_fallback
    if (((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0) {
      const efgp_status st = spread_sorted2(pl, x, y, N, s);
      if (st != EFGP_ERR_RESOURCE) return st;
      pl->err.clear();  // co-residency not available now: same grids, direct spreading below
      pl->spread_fallback = EFGP_FALLBACK_CORESIDENCY;
    } else {
      pl->spread_fallback = EFGP_FALLBACK_UNALIGNED;
    }
    method = EFGP_SPREAD_GLOBAL;
    pl->spread_used = method;
  } else if (method == EFGP_SPREAD_CELLSORT) {
    const efgp_status st = spread_cellsort(pl, x, y, N, s);
    if (st != EFGP_ERR_RESOURCE) return st;
    pl->err.clear();  // (N >= 2^32 in one call): same grids, direct spreading below
    pl->spread_fallback = EFGP_FALLBACK_TOO_MANY_POINTS;
    method = EFGP_SPREAD_GLOBAL;
    pl->spread_used = method;
  }
  switch (pl->P.d) {
    case 1: return dispatch_w<1>(pl, x, y, N, s, method);
    case 2: return dispatch_w<2>(pl, x, y, N, s, method);
    case 3: return dispatch_w<3>(pl, x, y, N, s, method);
  }
  return EFGP_ERR_INVALID;
}

}  // namespace efgp
