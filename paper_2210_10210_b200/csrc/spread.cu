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
//   SORTED (d = 2, W <= 6): per chunk of points, k_bin2 bins the points by tile of start cells
//           (T x T start cells) into an L2-resident record buffer; k_tiles2 gives each start cell of a
//           tile to one thread, which accumulates the W x W footprints of all its points (identical
//           windows) in registers for both strengths; windows are combined in shared memory in W^2
//           conflict-free steps and flushed once per work item with RED.  Both strengths use g1's grid.
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

// ------------------------------------------------------------------------------------------------
// SORTED (2D)
// ------------------------------------------------------------------------------------------------
constexpr int kBinThreads = 256, kBinPPT = 8, kBinBatch = kBinThreads * kBinPPT;  // 2048 points / CTA
constexpr int kTileSide = 16, kTileThreads = kTileSide * kTileSide;                // 256 start cells
constexpr int kRound = 8192;                                                       // points per round

// exclusive scan of n ints in shared memory by a whole block (n arbitrary)
__device__ void block_exclusive_scan(int *a, int n, int *total, int *warp_sums) {
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int beg = threadIdx.x * per, end = min(n, beg + per);
  int s = 0;
  for (int i = beg; i < end; ++i) s += a[i];
  // inclusive scan of s across the block
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int v = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) warp_sums[wid] = v;
  __syncthreads();
  if (wid == 0) {
    int w = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    if (lane < nw) warp_sums[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  int run = v - s + (wid > 0 ? warp_sums[wid - 1] : 0);  // exclusive prefix of this thread's range
  for (int i = beg; i < end; ++i) {
    const int c = a[i];
    a[i] = run;
    run += c;
  }
  if (threadIdx.x == blockDim.x - 1) *total = run;
  __syncthreads();
}

// Bin one batch of kBinBatch points of the chunk by tile; records land in the batch's own region,
// ordered by tile; seg[tile * nbmax + batch] = (offset in the region, count).
template <int W>
__global__ void __launch_bounds__(kBinThreads) k_bin2(const double *__restrict__ x, const double *__restrict__ y,
                                                      int64_t n, double h, int n1, int s_lo, int nt1, int ntiles,
                                                      int nbmax, double2 *__restrict__ rec_x,
                                                      double *__restrict__ rec_y, int2 *__restrict__ seg,
                                                      int *__restrict__ err) {
  extern __shared__ int bsh[];
  int *cnt = bsh, *wsum = bsh + ntiles + 1;
  __shared__ int total;
  for (int i = threadIdx.x; i < ntiles; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  const int b = blockIdx.x;
  const int64_t base = (int64_t)b * kBinBatch;
  const double2 *x2 = reinterpret_cast<const double2 *>(x);
  double2 px[kBinPPT];
  double py[kBinPPT];
  int tl[kBinPPT], rk[kBinPPT];
#pragma unroll
  for (int k = 0; k < kBinPPT; ++k) {
    const int64_t i = base + k * kBinThreads + threadIdx.x;
    tl[k] = -1;
    if (i < n) {
      px[k] = __ldcs(x2 + i);  // streamed once: evict-first
      py[k] = __ldcs(y + i);
    }
  }
#pragma unroll
  for (int k = 0; k < kBinPPT; ++k) {
    const int64_t i = base + k * kBinThreads + threadIdx.x;
    if (i >= n) continue;
    const bool ok = px[k].x >= 0.0 && px[k].x <= 1.0 && px[k].y >= 0.0 && px[k].y <= 1.0 && isfinite(py[k]);
    if (!ok) {
      atomicOr(err, 1);
      continue;
    }
    const int i1 = (int)ceil(h * px[k].x * n1 - 0.5 * W) - s_lo;
    const int i2 = (int)ceil(h * px[k].y * n1 - 0.5 * W) - s_lo;
    const int t = (i1 / kTileSide) * nt1 + (i2 / kTileSide);
    tl[k] = t;
    rk[k] = atomicAdd(&cnt[t], 1);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) seg[(int64_t)t * nbmax + b].y = cnt[t];
  __syncthreads();
  block_exclusive_scan(cnt, ntiles, &total, wsum);
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) seg[(int64_t)t * nbmax + b].x = cnt[t];
#pragma unroll
  for (int k = 0; k < kBinPPT; ++k) {
    if (tl[k] < 0) continue;
    const int64_t pos = base + cnt[tl[k]] + rk[k];
    rec_x[pos] = px[k];
    rec_y[pos] = py[k];
  }
}

// Work item = (tile, part): the part-th 1/Q of the tile's records of this chunk.  Thread = start cell.
template <int W>
__global__ void __launch_bounds__(kTileThreads) k_tiles2(const double2 *__restrict__ rec_x,
                                                         const double *__restrict__ rec_y,
                                                         const int2 *__restrict__ seg, int nb, int nbmax, int nt1,
                                                         int Q, double h, int n1, int s_lo, EsPoly P,
                                                         double *__restrict__ g1, double *__restrict__ gy) {
  constexpr int T = kTileSide, NT = kTileThreads, A = T + W - 1;
  extern __shared__ int tsh[];
  int *pre = tsh;                                   // nbmax + 1
  int *offb = pre + (nbmax + 1);                    // nbmax
  int *ccnt = offb + nbmax;                         // NT
  int *wsum = ccnt + NT;                            // 32
  unsigned short *segof = reinterpret_cast<unsigned short *>(wsum + 32);  // kRound
  unsigned short *rank = segof + kRound;
  unsigned short *sidx = rank + kRound;
  unsigned char *cell = reinterpret_cast<unsigned char *>(sidx + kRound);  // kRound
  double *accs = reinterpret_cast<double *>(
      (reinterpret_cast<uintptr_t>(cell + kRound) + 15) & ~uintptr_t(15));   // 2 A^2
  __shared__ int total, bfirst;

  const int tile = blockIdx.x / Q, part = blockIdx.x % Q;
  const int r0 = (tile / nt1) * T, c0 = (tile % nt1) * T;  // tile origin in start-cell units (0-based)
  for (int b = threadIdx.x; b < nb; b += NT) {
    const int2 s = seg[(int64_t)tile * nbmax + b];
    pre[b] = s.y;
    offb[b] = s.x;
  }
  __syncthreads();
  block_exclusive_scan(pre, nb, &total, wsum);
  if (threadIdx.x == 0) pre[nb] = total;
  __syncthreads();
  const int begin = (int)((int64_t)part * total / Q), end = (int)((int64_t)(part + 1) * total / Q);

  double a1[W][W], ay[W][W];
#pragma unroll
  for (int a = 0; a < W; ++a)
#pragma unroll
    for (int b = 0; b < W; ++b) a1[a][b] = ay[a][b] = 0.0;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = NT / 32;
  for (int rs = begin; rs < end; rs += kRound) {
    const int nr = min(kRound, end - rs);
    ccnt[threadIdx.x] = 0;
    if (threadIdx.x == 0) {  // last segment starting at or before rs
      int lo = 0, hi = nb;   // pre[lo] <= rs < pre[hi]
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (pre[mid] <= rs) lo = mid;
        else hi = mid;
      }
      bfirst = lo;
    }
    __syncthreads();
    for (int b = bfirst + warp; b < nb && pre[b] < rs + nr; b += nwarps) {
      const int lo = max(pre[b], rs), hi = min(pre[b + 1], rs + nr);
      for (int gi = lo + lane; gi < hi; gi += 32) {
        const int64_t pos = (int64_t)b * kBinBatch + offb[b] + (gi - pre[b]);
        const double2 xx = rec_x[pos];
        const int i1 = (int)ceil(h * xx.x * n1 - 0.5 * W) - s_lo - r0;
        const int i2 = (int)ceil(h * xx.y * n1 - 0.5 * W) - s_lo - c0;
        const int c = i1 * T + i2;
        const int j = gi - rs;
        cell[j] = (unsigned char)c;
        segof[j] = (unsigned short)b;
        rank[j] = (unsigned short)atomicAdd(&ccnt[c], 1);
      }
    }
    __syncthreads();
    const int mycnt = ccnt[threadIdx.x];
    block_exclusive_scan(ccnt, NT, &total, wsum);  // ccnt <- start offsets
    for (int j = threadIdx.x; j < nr; j += NT) sidx[ccnt[cell[j]] + rank[j]] = (unsigned short)j;
    __syncthreads();
    const int st = ccnt[threadIdx.x];
    for (int k = st; k < st + mycnt; ++k) {
      const int j = sidx[k], b = segof[j];
      const int64_t pos = (int64_t)b * kBinBatch + offb[b] + (rs + j - pre[b]);
      const double2 xx = rec_x[pos];
      const double yv = rec_y[pos];
      double w1[W], w2[W];
      es_weights<W>(h * xx.x * n1, P, w1);
      es_weights<W>(h * xx.y * n1, P, w2);
#pragma unroll
      for (int a = 0; a < W; ++a) {
        const double ca = w1[a], cy = yv * w1[a];
#pragma unroll
        for (int b2 = 0; b2 < W; ++b2) {
          a1[a][b2] = fma(ca, w2[b2], a1[a][b2]);
          ay[a][b2] = fma(cy, w2[b2], ay[a][b2]);
        }
      }
    }
    __syncthreads();
  }
  // combine the threads' windows in shared memory: W^2 steps, each conflict-free
  for (int i = threadIdx.x; i < 2 * A * A; i += NT) accs[i] = 0.0;
  __syncthreads();
  const int my_r = threadIdx.x / T, my_c = threadIdx.x % T;
#pragma unroll
  for (int a = 0; a < W; ++a) {
#pragma unroll
    for (int b2 = 0; b2 < W; ++b2) {
      const int idx = (my_r + a) * A + (my_c + b2);
      accs[idx] += a1[a][b2];
      accs[A * A + idx] += ay[a][b2];
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < A * A; i += NT) {
    const double v1 = accs[i], vy = accs[A * A + i];
    if (v1 == 0.0 && vy == 0.0) continue;
    const int r = wrap(s_lo + r0 + i / A, n1), c = wrap(s_lo + c0 + i % A, n1);
    const int64_t gi = (int64_t)r * n1 + c;
    if (v1 != 0.0) atomicAdd(g1 + gi, v1);
    if (vy != 0.0) atomicAdd(gy + gi, vy);
  }
}

static size_t tiles_smem_bytes(int nbmax, int W) {
  const int A = kTileSide + W - 1;
  size_t b = sizeof(int) * (size_t)(nbmax + 1 + nbmax + kTileThreads + 32);
  b += sizeof(unsigned short) * 3 * kRound + kRound;
  b = (b + 15) & ~size_t(15);
  b += sizeof(double) * 2 * A * A;
  return b;
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
  const bool sorted_ok = p.d == 2 && p.w <= 6;
  const bool smem_ok = smem_bytes(p) <= 200 * 1024;
  if (m == EFGP_SPREAD_AUTO) m = sorted_ok ? EFGP_SPREAD_SORTED : (smem_ok ? EFGP_SPREAD_SMEM : EFGP_SPREAD_GLOBAL);
  if (m == EFGP_SPREAD_SORTED && !sorted_ok) m = smem_ok ? EFGP_SPREAD_SMEM : EFGP_SPREAD_GLOBAL;
  if (m == EFGP_SPREAD_SMEM && !smem_ok) m = EFGP_SPREAD_GLOBAL;
  p.spread_method = m;
  p.n_rhs = (m == EFGP_SPREAD_SORTED) ? p.n1 : p.n2;
  if (m == EFGP_SPREAD_SORTED) {
    p.s_lo = -(p.w / 2);
    const int hi0 = (int)std::ceil(p.h * p.n1 - 0.5 * p.w);
    p.s_count = hi0 - p.s_lo + 1;
    p.tile = kTileSide;
    p.ntile1 = (p.s_count + kTileSide - 1) / kTileSide;
    p.bin_batch = kBinBatch;
    p.chunk = int64_t(1) << 21;
  }
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
  } else if (method == EFGP_SPREAD_SORTED) {
    if constexpr (D == 2 && W <= 6) {
      const int nt1 = P.ntile1, ntiles = nt1 * nt1;
      const int nbmax = (int)((P.chunk + kBinBatch - 1) / kBinBatch);
      const size_t bsm = sizeof(int) * (size_t)(ntiles + 1 + 32);
      const size_t tsm = tiles_smem_bytes(nbmax, W);
      EFGP_CUDA(cudaFuncSetAttribute(k_bin2<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
      EFGP_CUDA(cudaFuncSetAttribute(k_tiles2<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
      const int Q = std::max(1, (2 * pl->num_sms + ntiles - 1) / ntiles);
      for (int64_t c0 = 0; c0 < N; c0 += P.chunk) {
        const int64_t nc = std::min<int64_t>(P.chunk, N - c0);
        const int nb = (int)((nc + kBinBatch - 1) / kBinBatch);
        k_bin2<W><<<nb, kBinThreads, bsm, s>>>(x + c0 * 2, y + c0, nc, P.h, (int)P.n1, P.s_lo, nt1, ntiles, nbmax,
                                               pl->rec_x, pl->rec_y, pl->seg, pl->dflags);
        k_tiles2<W><<<ntiles * Q, kTileThreads, tsm, s>>>(pl->rec_x, pl->rec_y, pl->seg, nb, nbmax, nt1, Q, P.h,
                                                          (int)P.n1, P.s_lo, P.poly, pl->g1, pl->g2);
      }
    } else {
      pl->err = "internal: SORTED spreading needs d = 2 and w <= 6";
      return EFGP_ERR_INVALID;
    }
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
  return EFGP_OK;
}

efgp_status spread_points(efgp_plan *pl, const double *x, const double *y, int64_t N, cudaStream_t s) {
  if (N <= 0) return EFGP_OK;
  int method = pl->P.spread_method;
  // the SORTED binning loads points as 16-byte pairs
  if (method == EFGP_SPREAD_SORTED && (reinterpret_cast<uintptr_t>(x) & 15)) method = EFGP_SPREAD_GLOBAL;
  switch (pl->P.d) {
    case 1: return dispatch_w<1>(pl, x, y, N, s, method);
    case 2: return dispatch_w<2>(pl, x, y, N, s, method);
    case 3: return dispatch_w<3>(pl, x, y, N, s, method);
  }
  return EFGP_ERR_INVALID;
}

efgp_status spread_end(efgp_plan *pl, cudaStream_t s) {
  (void)pl;
  (void)s;
  return EFGP_OK;
}

}  // namespace efgp
