// K1, CELLSORT strategy: type-1 spreading for the kernels the SORTED register windows cannot hold
// (2D with W >= 7, e.g. c3 at nufft_tol 1e-7, W = 8; and 3D, e.g. c4) — the cases that otherwise fall
// back to one fp64 RED per (point, cell): 2 W^d atomics per point (c3: 5.4e8 points/s).
//
// Both strengths (1 and y) go to the n1 grid (n_rhs = n1, like SORTED).  Per call:
//   1. k_cs_count   : per-CTA shared-memory histogram of the points' super-cells (G^d start cells;
//                     G = 1 in 2D (2 for large grids), 4 in 3D so the key space fits shared memory).
//   2. k_het_colscan / k_het_offsets (hetero.cu): bucket offsets per CTA.
//   3. k_cs_scatter : counting-sort scatter of 32-byte records, one STG.256 (a full sector) per point:
//                     2D (x1, x2, y, w), 3D (x1, x2, x3, y) (+ w in its own array when given).  (The
//                     r01 structure-of-arrays scatter wrote 3-4 partial 8-byte sectors per point: 3.5-4x
//                     its algorithmic DRAM bytes.)
//   4. k_cs_spread  : a warp per run of <= kCsRun points of one super-cell.  Batches of 32 points: lane
//                     p evaluates the ES weights of point p and writes them, padded to the union window
//                     U = W + G - 1 per dimension, to shared memory; then every lane accumulates the
//                     U^d window elements it owns (e = lane + 32 t) over the 32 points in registers
//                     (strengths 1 and y).  One RED per owned element per run.
// Traffic: x, y read twice (count, scatter) + the sorted 32-byte records written and read, against
// 2 W^d L2 atomics per point for GLOBAL.
#include <algorithm>
#include <cmath>
#include <vector>

#include "efgp_internal.cuh"

namespace efgp {

constexpr int kCsRun = 1024;     // points per warp work item
constexpr int kCsThreads = 128;  // spread kernel CTA (static weight rows: <= 34 KB)

struct CsItem {
  long long begin, end;
  int cell, pad_;
};


// super-cell key of point i; validates x in [0,1]^d and finite y (raises *err)
template <int D, int W, int G>
__device__ __forceinline__ int cs_key(const double *__restrict__ x, const double *__restrict__ y, int64_t i, double h,
                                      int n, int lo, int S, int *__restrict__ err) {
  int key = 0;
  bool ok = isfinite(__ldg(y + i));
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const double xv = __ldg(x + i * D + k);
    ok = ok && xv >= 0.0 && xv <= 1.0;
    const double t = h * xv * (double)n;  // the expression es_weights' callers use (K1, K9)
    int c = ((int)ceil(__dsub_rn(t, 0.5 * W)) - lo) / G;
    c = c < 0 ? 0 : (c >= S ? S - 1 : c);
    key = key * S + c;
  }
  if (!ok) atomicOr(err, 1);
  return key;
}

__device__ __forceinline__ void cs_range(int64_t N, int64_t &a, int64_t &e) {
  const int64_t per = (N + gridDim.x - 1) / gridDim.x;
  a = (int64_t)blockIdx.x * per;
  e = a + per < N ? a + per : N;
}

template <int D, int W, int G>
__global__ void k_cs_count(const double *__restrict__ x, const double *__restrict__ y, int64_t N, double h, int n,
                           int lo, int S, int ncell, unsigned *__restrict__ hist, int *__restrict__ err) {
  extern __shared__ unsigned cs_h[];
  for (int i = threadIdx.x; i < ncell; i += blockDim.x) cs_h[i] = 0;
  __syncthreads();
  int64_t a, e;
  cs_range(N, a, e);
  for (int64_t i = a + threadIdx.x; i < e; i += blockDim.x) atomicAdd(&cs_h[cs_key<D, W, G>(x, y, i, h, n, lo, S, err)], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < ncell; i += blockDim.x) hist[(size_t)blockIdx.x * ncell + i] = cs_h[i];
}

__device__ __forceinline__ void cs_st256(double4 *p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

template <int D, int W, int G>
__global__ void k_cs_scatter(const double *__restrict__ x, const double *__restrict__ y, int64_t N, double h, int n,
                             int lo, int S, int ncell, const unsigned *__restrict__ hist,
                             const long long *__restrict__ off, double4 *__restrict__ rec, int *__restrict__ err,
                             const double *__restrict__ w1, double *__restrict__ ws1) {
  extern __shared__ unsigned cs_c[];  // cursor relative to the bucket start (< 2^32 points per call)
  for (int i = threadIdx.x; i < ncell; i += blockDim.x) cs_c[i] = hist[(size_t)blockIdx.x * ncell + i];
  __syncthreads();
  int64_t a, e;
  cs_range(N, a, e);
  for (int64_t i = a + threadIdx.x; i < e; i += blockDim.x) {
    const int key = cs_key<D, W, G>(x, y, i, h, n, lo, S, err);
    EFGP_DCHECK(key >= 0 && key < ncell);
    const long long pos = off[key] + (long long)atomicAdd(&cs_c[key], 1u);
    EFGP_DCHECK(pos >= off[key] && pos < off[key + 1]);
    if constexpr (D == 2) {
      cs_st256(rec + pos, __ldg(x + 2 * i), __ldg(x + 2 * i + 1), __ldg(y + i), w1 ? __ldg(w1 + i) : 1.0);
    } else {
      cs_st256(rec + pos, __ldg(x + 3 * i), __ldg(x + 3 * i + 1), __ldg(x + 3 * i + 2), __ldg(y + i));
      if (w1) ws1[pos] = __ldg(w1 + i);
    }
  }
}

__device__ __forceinline__ int cs_wrap(int i, int n) {
  i %= n;
  return i < 0 ? i + n : i;
}

template <int D, int W, int G>
__global__ void __launch_bounds__(kCsThreads) k_cs_spread(const CsItem *__restrict__ items, int64_t nitems,
                                                          const double4 *__restrict__ rec,
                                                          const double *__restrict__ ws1, int64_t N,
                                                          double *__restrict__ g1, double *__restrict__ g2,
                                                          double h, int n, int lo, int S, EsPoly P) {
  constexpr int U = W + G - 1;                   // union window per dimension of a super-cell
  constexpr int UD = D == 2 ? U * U : U * U * U;
  constexpr int E = (UD + 31) / 32;              // window elements per lane
  __shared__ double wsm[kCsThreads / 32][32][D * U + 2];  // padded weight rows, y, strength-1 weight
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double(*ws)[D * U + 2] = wsm[wid];
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t it = warp; it < nitems; it += nwarps) {
    const CsItem item = items[it];
    int sc[D];
    {
      int rem = item.cell;
#pragma unroll
      for (int k = D - 1; k >= 0; --k) {
        sc[k] = rem % S;
        rem /= S;
      }
    }
    double a1[E], ay[E];
#pragma unroll
    for (int t = 0; t < E; ++t) a1[t] = ay[t] = 0.0;
    for (long long b0 = item.begin; b0 < item.end; b0 += 32) {
      const long long r = b0 + lane;
      __syncwarp();
      if (r < item.end) {
        const double4 rv = rec[r];
        const double xr[3] = {rv.x, rv.y, rv.z};
        double row[D * U];
#pragma unroll
        for (int q = 0; q < D * U; ++q) row[q] = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) {
          double w[W];
          const int i0 = es_weights<W>(h * xr[k] * (double)n, P, w);
          int off = i0 - lo - sc[k] * G;         // start cell within the super-cell, 0..G-1
          off = off < 0 ? 0 : (off > G - 1 ? G - 1 : off);
#pragma unroll
          for (int a = 0; a < W; ++a)
#pragma unroll
            for (int o = 0; o < G; ++o)
              if (o == off) row[k * U + o + a] = w[a];
        }
#pragma unroll
        for (int q = 0; q < D * U; ++q) ws[lane][q] = row[q];
        ws[lane][D * U] = D == 2 ? rv.z : rv.w;
        ws[lane][D * U + 1] = D == 2 ? rv.w : (ws1 ? __ldg(ws1 + r) : 1.0);
      } else {
#pragma unroll
        for (int q = 0; q <= D * U + 1; ++q) ws[lane][q] = 0.0;
      }
      __syncwarp();
      const int np = (int)min(32LL, item.end - b0);
      for (int p = 0; p < np; ++p) {
        const double yv = ws[p][D * U], wv = ws[p][D * U + 1];
#pragma unroll
        for (int t = 0; t < E; ++t) {
          const int e = lane + 32 * t;
          if (e < UD) {
            double f;
            if constexpr (D == 2) {
              f = ws[p][e / U] * ws[p][U + e % U];
            } else {
              f = ws[p][e / (U * U)] * ws[p][U + (e / U) % U] * ws[p][2 * U + e % U];
            }
            a1[t] = fma(f, wv, a1[t]);
            ay[t] = fma(f, yv, ay[t]);
          }
        }
      }
    }
#pragma unroll
    for (int t = 0; t < E; ++t) {
      const int e = lane + 32 * t;
      if (e < UD && (a1[t] != 0.0 || ay[t] != 0.0)) {
        int64_t gi;
        if constexpr (D == 2) {
          gi = (int64_t)cs_wrap(sc[0] * G + lo + e / U, n) * n + cs_wrap(sc[1] * G + lo + e % U, n);
        } else {
          gi = ((int64_t)cs_wrap(sc[0] * G + lo + e / (U * U), n) * n + cs_wrap(sc[1] * G + lo + (e / U) % U, n)) * n +
               cs_wrap(sc[2] * G + lo + e % U, n);
        }
        atomicAdd(g1 + gi, a1[t]);
        atomicAdd(g2 + gi, ay[t]);
      }
    }
  }
}

// super-cell size: 1 in 2D (2 when the start-cell count does not fit the shared-memory histogram,
// e.g. m = 94), 4 in 3D
bool cellsort_geometry(const Params &p, int &lo, int &S, int &ncell, int &G) {
  if (p.d < 2 || p.d > 3 || (p.d == 3 && p.w > 6)) return false;
  lo = -(p.w / 2);
  const int hi = (int)std::ceil(p.h * (double)p.n1 - 0.5 * p.w);
  const int cells = hi - lo + 2;  // start cells per dimension (+1 spare)
  for (G = (p.d == 3 ? 4 : 1); G <= (p.d == 3 ? 4 : 2); ++G) {
    S = (cells + G - 1) / G;
    ncell = p.d == 2 ? S * S : S * S * S;
    if ((size_t)ncell * 4 <= 200 * 1024) return true;
  }
  return false;
}
bool cellsort_geometry(const Params &p, int &lo, int &S, int &ncell) {
  int G;
  return cellsort_geometry(p, lo, S, ncell, G);
}

template <int D, int W, int G>
static efgp_status cellsort_t(efgp_plan *pl, const double *x, const double *y, const double *w1, int64_t N,
                              cudaStream_t s) {
  const Params &P = pl->P;
  int lo, S, ncell, Gs;
  if (!cellsort_geometry(P, lo, S, ncell, Gs) || Gs != G) return EFGP_ERR_RESOURCE;
  const int B = sort_ctas(pl->num_sms), T = 1024, n = (int)P.n1;
  unsigned *hist = nullptr;
  long long *tot = nullptr, *off = nullptr;
  double4 *rec = nullptr;
  double *ws1 = nullptr;
  CsItem *items = nullptr;
  EFGP_PALLOC(&hist, sizeof(unsigned) * B * ncell, s);
  EFGP_PALLOC(&tot, sizeof(long long) * ncell, s);
  EFGP_PALLOC(&off, sizeof(long long) * (ncell + 1), s);
  EFGP_PALLOC(&rec, sizeof(double4) * N, s);
  if (w1 && D == 3) EFGP_PALLOC(&ws1, sizeof(double) * N, s);
  const size_t sm = sizeof(unsigned) * ncell;
  EFGP_CUDA(cudaFuncSetAttribute(k_cs_count<D, W, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  EFGP_CUDA(cudaFuncSetAttribute(k_cs_scatter<D, W, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  k_cs_count<D, W, G><<<B, T, sm, s>>>(x, y, N, P.h, n, lo, S, ncell, hist, pl->dflags);
  k_het_colscan<<<(ncell + 255) / 256, 256, 0, s>>>(hist, B, ncell, tot);
  k_het_offsets<<<1, 1024, 0, s>>>(tot, ncell, off);
  k_cs_scatter<D, W, G><<<B, T, sm, s>>>(x, y, N, P.h, n, lo, S, ncell, hist, off, rec, pl->dflags, w1, ws1);
  EFGP_CUDA(cudaGetLastError());
  std::vector<long long> offh(ncell + 1);
  EFGP_CUDA(cudaMemcpyAsync(offh.data(), off, sizeof(long long) * (ncell + 1), cudaMemcpyDeviceToHost, s));
  EFGP_CUDA(cudaStreamSynchronize(s));
  std::vector<CsItem> it;
  for (int c = 0; c < ncell; ++c)
    for (long long b = offh[c]; b < offh[c + 1]; b += kCsRun)
      it.push_back(CsItem{b, std::min<long long>(b + kCsRun, offh[c + 1]), c, 0});
  const int64_t nitems = (int64_t)it.size();
  EFGP_PALLOC(&items, sizeof(CsItem) * std::max<size_t>(it.size(), 1), s);
  EFGP_CUDA(cudaMemcpyAsync(items, it.data(), sizeof(CsItem) * it.size(), cudaMemcpyHostToDevice, s));
  int per_sm = 1;
  EFGP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cs_spread<D, W, G>, kCsThreads, 0));
  int64_t blocks = std::min<int64_t>((int64_t)pl->num_sms * std::max(per_sm, 1), (nitems * 32 + kCsThreads - 1) / kCsThreads);
  if (nitems > 0)
    k_cs_spread<D, W, G><<<(unsigned)std::max<int64_t>(blocks, 1), kCsThreads, 0, s>>>(items, nitems, rec, ws1, N, pl->g1,
                                                                                     pl->g2, P.h, n, lo, S, P.poly);
  EFGP_CUDA(cudaGetLastError());
  EFGP_CUDA(cudaStreamSynchronize(s));  // the host item vector is consumed by the copy above
  for (void *p : {(void *)hist, (void *)tot, (void *)off, (void *)rec, (void *)items}) cudaFreeAsync(p, s);
  if (ws1) cudaFreeAsync(ws1, s);
  return EFGP_OK;
}

efgp_status spread_cellsort(efgp_plan *pl, const double *x, const double *y, int64_t N, cudaStream_t s,
                            const double *w1) {
  if (N >= (1ll << 32)) return EFGP_ERR_RESOURCE;  // 32-bit bucket cursors
  const int W = pl->P.w;
  int lo, S, ncell, G;
  if (!cellsort_geometry(pl->P, lo, S, ncell, G)) return EFGP_ERR_RESOURCE;
  if (pl->P.d == 2 && G == 1) {
    switch (W) {
#define C2(WW) case WW: return cellsort_t<2, WW, 1>(pl, x, y, w1, N, s);
      C2(2) C2(3) C2(4) C2(5) C2(6) C2(7) C2(8) C2(9) C2(10) C2(11) C2(12) C2(13) C2(14) C2(15) C2(16)
#undef C2
    }
  } else if (pl->P.d == 2 && G == 2) {
    switch (W) {
#define C2(WW) case WW: return cellsort_t<2, WW, 2>(pl, x, y, w1, N, s);
      C2(2) C2(3) C2(4) C2(5) C2(6) C2(7) C2(8) C2(9) C2(10) C2(11) C2(12) C2(13) C2(14) C2(15) C2(16)
#undef C2
    }
  } else if (pl->P.d == 3) {
    switch (W) {
#define C3(WW) case WW: return cellsort_t<3, WW, 4>(pl, x, y, w1, N, s);
      C3(2) C3(3) C3(4) C3(5) C3(6)
#undef C3
    }
  }
  return EFGP_ERR_RESOURCE;
}

}  // namespace efgp
