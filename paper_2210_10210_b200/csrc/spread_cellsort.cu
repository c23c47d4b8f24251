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


// super-cell key of a point from its loaded coordinates; ok is false for x outside [0,1]^d or a
// non-finite y (the caller raises *err once per batch: an atomic between the loads of a batch would
// keep the compiler from hoisting the later loads above it)
template <int D, int W, int G>
__device__ __forceinline__ int cs_key_of(const double (&xv)[D], double yv, double h, int n, int lo, int S, bool &ok) {
  int key = 0;
  ok = isfinite(yv);
#pragma unroll
  for (int k = 0; k < D; ++k) {
    ok = ok && xv[k] >= 0.0 && xv[k] <= 1.0;
    const double t = h * xv[k] * (double)n;  // the expression es_weights' callers use (K1, K9)
    int c = ((int)ceil(__dsub_rn(t, 0.5 * W)) - lo) / G;
    c = c < 0 ? 0 : (c >= S ? S - 1 : c);
    key = key * S + c;
  }
  return key;
}

// kCsBatch points per thread per step: all loads first, then keys, cursor atomics and stores
constexpr int kCsBatch = 4;
template <int D>
struct CsPts {
  double x[kCsBatch][D], y[kCsBatch], w[kCsBatch];
  int key[kCsBatch];
};
template <int D, int W, int G>
__device__ __forceinline__ bool cs_load_batch(const double *__restrict__ x, const double *__restrict__ y,
                                              const double *__restrict__ w1, int64_t i0, int64_t stride, int64_t e,
                                              double h, int n, int lo, int S, CsPts<D> &P) {
#pragma unroll
  for (int u = 0; u < kCsBatch; ++u) {
    const int64_t i = i0 + u * stride;
    const int64_t j = i < e ? i : i0;  // (i0 < e: a valid index for the masked lanes)
#pragma unroll
    for (int k = 0; k < D; ++k) P.x[u][k] = __ldg(x + j * D + k);
    P.y[u] = y ? __ldg(y + j) : 0.0;
    P.w[u] = w1 ? __ldg(w1 + j) : 1.0;
  }
  bool bad = false;
#pragma unroll
  for (int u = 0; u < kCsBatch; ++u) {
    bool ok;
    const int k = cs_key_of<D, W, G>(P.x[u], P.y[u], h, n, lo, S, ok);
    const bool in = i0 + u * stride < e;
    bad |= in && !ok;
    P.key[u] = in ? k : -1;
  }
  return bad;
}

__device__ __forceinline__ void cs_range(int64_t N, int64_t &a, int64_t &e) {
  const int64_t per = (N + gridDim.x - 1) / gridDim.x;
  a = (int64_t)blockIdx.x * per;
  e = a + per < N ? a + per : N;
}

template <int D, int W, int G>
__global__ void __launch_bounds__(1024) k_cs_count(const double *__restrict__ x, const double *__restrict__ y, int64_t N, double h, int n,
                           int lo, int S, int ncell, unsigned *__restrict__ hist, int *__restrict__ err) {
  extern __shared__ unsigned cs_h[];
  for (int i = threadIdx.x; i < ncell; i += blockDim.x) cs_h[i] = 0;
  __syncthreads();
  int64_t a, e;
  cs_range(N, a, e);
  bool bad = false;
  for (int64_t i0 = a + threadIdx.x; i0 < e; i0 += kCsBatch * (int64_t)blockDim.x) {
    CsPts<D> P;
    bad |= cs_load_batch<D, W, G>(x, y, nullptr, i0, blockDim.x, e, h, n, lo, S, P);
#pragma unroll
    for (int u = 0; u < kCsBatch; ++u)
      if (P.key[u] >= 0) atomicAdd(&cs_h[P.key[u]], 1u);
  }
  if (bad) atomicOr(err, 1);
  __syncthreads();
  for (int i = threadIdx.x; i < ncell; i += blockDim.x) hist[(size_t)blockIdx.x * ncell + i] = cs_h[i];
}

__device__ __forceinline__ void cs_st256(double4 *p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

template <int D, int W, int G>
__global__ void __launch_bounds__(1024) k_cs_scatter(const double *__restrict__ x, const double *__restrict__ y, int64_t N, double h, int n,
                             int lo, int S, int ncell, const unsigned *__restrict__ hist,
                             const long long *__restrict__ off, double4 *__restrict__ rec, int *__restrict__ err,
                             const double *__restrict__ w1, double *__restrict__ ws1) {
  // absolute cursor of this CTA in each bucket, off[c] + (this CTA's prefix), as 32 bits (< 2^32 points
  // per call): the scatter position needs no dependent global load of off[key]
  extern __shared__ unsigned cs_c[];
  for (int i = threadIdx.x; i < ncell; i += blockDim.x) cs_c[i] = (unsigned)(off[i] + hist[(size_t)blockIdx.x * ncell + i]);
  __syncthreads();
  int64_t a, e;
  cs_range(N, a, e);
  bool bad = false;
  for (int64_t i0 = a + threadIdx.x; i0 < e; i0 += kCsBatch * (int64_t)blockDim.x) {
    CsPts<D> P;
    bad |= cs_load_batch<D, W, G>(x, y, w1, i0, blockDim.x, e, h, n, lo, S, P);
    unsigned pos[kCsBatch];
#pragma unroll
    for (int u = 0; u < kCsBatch; ++u) {
      EFGP_DCHECK(P.key[u] < ncell);
      pos[u] = P.key[u] >= 0 ? atomicAdd(&cs_c[P.key[u]], 1u) : 0u;
    }
#pragma unroll
    for (int u = 0; u < kCsBatch; ++u) {
      if (P.key[u] < 0) continue;
      EFGP_DCHECK(pos[u] >= off[P.key[u]] && pos[u] < off[P.key[u] + 1]);
      if constexpr (D == 2) {
        cs_st256(rec + pos[u], P.x[u][0], P.x[u][1], P.y[u], P.w[u]);
      } else {
        cs_st256(rec + pos[u], P.x[u][0], P.x[u][1], P.x[u][2], P.y[u]);
        if (w1) ws1[pos[u]] = P.w[u];
      }
    }
  }
  if (bad) atomicOr(err, 1);
}

// off[c] = exclusive prefix of the bucket sizes tot[c] (off[ncell] = N), iof[c] = exclusive prefix of
// the work items per bucket ceil(tot[c] / kCsRun) (iof[ncell] = item count): one CTA of 1024
// threads, each scanning a contiguous slice serially, one block scan of the slice totals
__global__ void k_cs_offsets(const long long *__restrict__ tot, int ncell, long long *__restrict__ off,
                             long long *__restrict__ iof) {
  extern __shared__ unsigned cs_t[];  // bucket sizes (< 2^32: N < 2^32 per call), staged coalesced
  __shared__ long long wsum[2][32];
  for (int c = threadIdx.x; c < ncell; c += blockDim.x) cs_t[c] = (unsigned)tot[c];
  __syncthreads();
  const int t = threadIdx.x, nt = blockDim.x, lane = t & 31, wid = t >> 5;
  const int per = (ncell + nt - 1) / nt, a = t * per, e = min(ncell, a + per);
  long long s = 0, si = 0;
  for (int c = a; c < e; ++c) {
    const unsigned v = cs_t[c];
    s += v;
    si += (v + kCsRun - 1) / kCsRun;
  }
  long long incl = s, incli = si;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long v = __shfl_up_sync(0xffffffffu, incl, o), vi = __shfl_up_sync(0xffffffffu, incli, o);
    if (lane >= o) {
      incl += v;
      incli += vi;
    }
  }
  if (lane == 31) {
    wsum[0][wid] = incl;
    wsum[1][wid] = incli;
  }
  __syncthreads();
  if (wid < 2) {
    long long w = lane < (nt >> 5) ? wsum[wid][lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long v = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += v;
    }
    wsum[wid][lane] = w;
  }
  __syncthreads();
  long long run = incl - s + (wid > 0 ? wsum[0][wid - 1] : 0);
  long long runi = incli - si + (wid > 0 ? wsum[1][wid - 1] : 0);
  for (int c = a; c < e; ++c) {
    const unsigned v = cs_t[c];
    iof[c] = runi;
    runi += (v + kCsRun - 1) / kCsRun;
    cs_t[c] = (unsigned)run;  // exclusive offset (< 2^32), written out coalesced below
    run += v;
  }
  if (t == nt - 1) {
    off[ncell] = run;
    iof[ncell] = runi;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < ncell; c += blockDim.x) off[c] = cs_t[c];
}

// the work items of bucket c: runs of <= kCsRun records (thread per bucket)
__global__ void k_cs_items(const long long *__restrict__ off, const long long *__restrict__ iof, int ncell,
                           CsItem *__restrict__ items) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncell) return;
  long long it = iof[c];
  for (long long b = off[c]; b < off[c + 1]; b += kCsRun, ++it)
    items[it] = CsItem{b, b + kCsRun < off[c + 1] ? b + kCsRun : off[c + 1], c, 0};
}

// Column scan of the per-CTA histograms, global bucket offsets and work items in one kernel (r02;
// replaces k_het_colscan + k_cs_offsets (one CTA) + k_cs_items: 22 + 37 + 5 us cold on c3).  CTA b
// (logical index from a ticket, so every predecessor has started) owns cells [256 b, 256 b + 256):
// thread c scans its column of hist over the B histogram rows (exclusive, in place) to the bucket size
// tot_c, the CTA scans (tot, ceil(tot / kCsRun)) and publishes its aggregate, then looks back over the
// predecessors' published words (decoupled look-back) for its exclusive prefix.  A status word packs
// flag (2 bits: 1 aggregate, 2 inclusive prefix) | items (30 bits) | points (32 bits): one 64-bit
// store publishes it, no torn reads (N < 2^32 and fewer than 2^30 items per call).
constexpr int kScanThreads = 256;
__global__ void __launch_bounds__(kScanThreads) k_cs_scan(unsigned *__restrict__ hist, int nblk, int ncell,
                                                          long long N, long long *__restrict__ off,
                                                          long long *__restrict__ iof, CsItem *__restrict__ items,
                                                          unsigned long long *st) {
  __shared__ unsigned ws_p[kScanThreads / 32], ws_i[kScanThreads / 32];
  __shared__ unsigned long long pre_s;
  __shared__ int bid_s;
  if (threadIdx.x == 0) bid_s = (int)atomicAdd(reinterpret_cast<unsigned *>(st + gridDim.x), 1u);
  __syncthreads();
  const int b = bid_s, t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int c = b * kScanThreads + t;
  unsigned tot = 0;
  if (c < ncell) {  // column scan (loads of a chunk of rows before any store, as k_het_colscan)
    constexpr int kChunk = 16;
    unsigned run = 0;
    for (int b0 = 0; b0 < nblk; b0 += kChunk) {
      unsigned v[kChunk];
#pragma unroll
      for (int k = 0; k < kChunk; ++k) v[k] = b0 + k < nblk ? __ldcg(hist + (size_t)(b0 + k) * ncell + c) : 0u;
#pragma unroll
      for (int k = 0; k < kChunk; ++k) {
        if (b0 + k < nblk) hist[(size_t)(b0 + k) * ncell + c] = run;
        run += v[k];
      }
    }
    tot = run;
  }
  const unsigned nit = (tot + kCsRun - 1) / kCsRun;
  // CTA scan of (tot, nit)
  unsigned ip = tot, ii = nit;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned vp = __shfl_up_sync(0xffffffffu, ip, o), vi = __shfl_up_sync(0xffffffffu, ii, o);
    if (lane >= o) {
      ip += vp;
      ii += vi;
    }
  }
  if (lane == 31) {
    ws_p[wid] = ip;
    ws_i[wid] = ii;
  }
  __syncthreads();
  unsigned bp = 0, bi = 0, ap = 0, ai = 0;  // warp prefix, CTA aggregate
  for (int w = 0; w < kScanThreads / 32; ++w) {
    if (w < wid) {
      bp += ws_p[w];
      bi += ws_i[w];
    }
    ap += ws_p[w];
    ai += ws_i[w];
  }
  if (t == 0) {
    const unsigned long long agg = (unsigned long long)ai << 32 | ap;
    unsigned long long excl = 0;  // (items << 32 | points) of the predecessors
    if (b == 0) {
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(st + b), "l"(agg | (2ull << 62)) : "memory");
    } else {
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(st + b), "l"(agg | (1ull << 62)) : "memory");
      for (int p = b - 1; p >= 0;) {
        unsigned long long w;
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(st + p) : "memory");
        const unsigned fl = (unsigned)(w >> 62);
        if (fl == 0) continue;  // not published yet: spin
        excl += w & ~(3ull << 62);
        if (fl == 2) break;
        --p;
      }
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(st + b), "l"((excl + agg) | (2ull << 62)) : "memory");
    }
    pre_s = excl;
  }
  __syncthreads();
  const unsigned long long pre = pre_s;
  if (c < ncell) {
    const long long o = (long long)(pre & 0xFFFFFFFFull) + bp + (ip - tot);
    const long long io = (long long)(pre >> 32) + bi + (ii - nit);
    off[c] = o;
    iof[c] = io;
    long long it = io;
    for (long long a = o; a < o + tot; a += kCsRun, ++it)
      items[it] = CsItem{a, a + kCsRun < o + tot ? a + kCsRun : o + tot, c, 0};
    if (c == ncell - 1) {
      off[ncell] = N;
      iof[ncell] = io + nit;
    }
  }
}

__device__ __forceinline__ int cs_wrap(int i, int n) {
  i %= n;
  return i < 0 ? i + n : i;
}

template <int D, int W, int G>
__global__ void __launch_bounds__(kCsThreads) k_cs_spread(const CsItem *__restrict__ items, const long long *__restrict__ nitems_dev,
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
  const int64_t nitems = *nitems_dev;
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
      if constexpr (D == 3 && U == 8) {
        // 3D, U = 8 (c4: W = 5, G = 4): element t = 2a + k of lane l is (a, b = l/8 + 4k, c = l%8), so
        // the strengths and the (b, c) weights fold into two per-point column factors and every
        // element costs 2 FMAs; the row weights w1[a] are broadcast loads (r01: 2 products, 2 FMAs
        // and 3 shared loads per element)
        const int cc = lane & 7, bb = lane >> 3;
#pragma unroll 2
        for (int p = 0; p < np; ++p) {
          const double *wr = ws[p];
          const double yv = wr[3 * U], wv = wr[3 * U + 1];
          const double w3 = wr[2 * U + cc], w3s = w3 * wv, w3y = w3 * yv;
          const double w2a = wr[U + bb], w2b = wr[U + bb + 4];
          const double gs0 = w2a * w3s, gy0 = w2a * w3y, gs1 = w2b * w3s, gy1 = w2b * w3y;
#pragma unroll
          for (int a = 0; a < U; ++a) {
            const double w1 = wr[a];
            a1[2 * a] = fma(w1, gs0, a1[2 * a]);
            ay[2 * a] = fma(w1, gy0, ay[2 * a]);
            a1[2 * a + 1] = fma(w1, gs1, a1[2 * a + 1]);
            ay[2 * a + 1] = fma(w1, gy1, ay[2 * a + 1]);
          }
        }
        continue;
      }
#pragma unroll 4
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

// 2D spread with a quarter-warp layout (c3): batches of 32 points as in k_cs_spread (lane p evaluates
// point p's weights into a shared row), then the warp accumulates 4 points at a time: quarter q = lane / 8
// takes point 4 i + q, lane c = lane % 8 owns the window columns b = c, c + 8, .. (< U) and every row a.
// Per point a lane loads w2[b] once and the U row weights w1[.] as broadcast 16-byte pairs, so a point
// costs ~2 shared wavefronts instead of 5 (r01 layout: every lane two elements, two loads each; the
// shared-memory pipe was the limit), with the same 2 U^2 FMAs.  The four quarters' partial windows are
// summed by shuffles at the end of a run; quarter q then issues the REDs of rows a = q mod 4.
template <int W, int G>
__global__ void __launch_bounds__(kCsThreads) k_cs_spread2q(const CsItem *__restrict__ items,
                                                            const long long *__restrict__ nitems_dev,
                                                            const double4 *__restrict__ rec, double *__restrict__ g1,
                                                            double *__restrict__ g2, double h, int n, int lo, int S,
                                                            EsPoly P) {
  constexpr int U = W + G - 1;                  // union window per dimension of a super-cell
  constexpr int RW = (2 * U + 2 + 1) / 2 * 2;   // row: w1[U], w2[U], y, strength-1 weight (16-byte multiple)
  constexpr int NB = (U + 7) / 8;               // columns per lane
  __shared__ __align__(16) double wsm[kCsThreads / 32][32][RW];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, qd = lane >> 3, c8 = lane & 7;
  double(*ws)[RW] = wsm[wid];
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nitems = *nitems_dev;
  for (int64_t it = warp; it < nitems; it += nwarps) {
    const CsItem item = items[it];
    const int sc0 = item.cell / S, sc1 = item.cell % S;
    double a1[U][NB], ay[U][NB];
#pragma unroll
    for (int a = 0; a < U; ++a)
#pragma unroll
      for (int k = 0; k < NB; ++k) a1[a][k] = ay[a][k] = 0.0;
    for (long long b0 = item.begin; b0 < item.end; b0 += 32) {
      const long long r = b0 + lane;
      __syncwarp();
      double *myrow = ws[lane];
      if (r < item.end) {
        const double4 rv = rec[r];  // (x1, x2, y, strength-1 weight)
        const double xr[2] = {rv.x, rv.y};
        const int scs[2] = {sc0, sc1};
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          double w[W];
          const int i0 = es_weights<W>(h * xr[k] * (double)n, P, w);
          if constexpr (G == 1) {
#pragma unroll
            for (int a = 0; a < W; ++a) myrow[k * U + a] = w[a];
          } else {
            int off = i0 - lo - scs[k] * G;  // start cell within the super-cell, 0..G-1
            off = off < 0 ? 0 : (off > G - 1 ? G - 1 : off);
#pragma unroll
            for (int a = 0; a < U; ++a) {
              double v = 0.0;
#pragma unroll
              for (int o = 0; o < G; ++o)
                if (o == off && a - o >= 0 && a - o < W) v = w[a - o];
              myrow[k * U + a] = v;
            }
          }
        }
        *reinterpret_cast<double2 *>(myrow + 2 * U) = make_double2(rv.z, rv.w);
      } else {
#pragma unroll
        for (int q = 0; q < RW; q += 2) *reinterpret_cast<double2 *>(myrow + q) = make_double2(0.0, 0.0);
      }
      __syncwarp();
      const int np = (int)min(32LL, item.end - b0);
      for (int p0 = 0; p0 < np; p0 += 4) {
        const double *wr = ws[p0 + qd];  // rows past np are zero, so they add nothing
        double w2[NB];
#pragma unroll
        for (int k = 0; k < NB; ++k) w2[k] = c8 + 8 * k < U ? wr[U + c8 + 8 * k] : 0.0;
        const double2 yw = *reinterpret_cast<const double2 *>(wr + 2 * U);
        // the strengths folded into the column weight once per point: 2 FMAs per (row, column)
        // instead of a product and 2 FMAs
        double w2s[NB], w2y[NB];
#pragma unroll
        for (int k = 0; k < NB; ++k) {
          w2s[k] = w2[k] * yw.y;
          w2y[k] = w2[k] * yw.x;
        }
#pragma unroll
        for (int a = 0; a < U; a += 2) {
          const double2 wa = *reinterpret_cast<const double2 *>(wr + a);  // (w1[a], w1[a+1]); w1[U] = w2[0] if U odd
#pragma unroll
          for (int k = 0; k < NB; ++k) {
            a1[a][k] = fma(wa.x, w2s[k], a1[a][k]);
            ay[a][k] = fma(wa.x, w2y[k], ay[a][k]);
            if (a + 1 < U) {
              a1[a + 1][k] = fma(wa.y, w2s[k], a1[a + 1][k]);
              ay[a + 1][k] = fma(wa.y, w2y[k], ay[a + 1][k]);
            }
          }
        }
      }
    }
    // sum the four quarters (butterfly: every lane gets the totals of its columns), then quarter qd
    // adds rows a = qd mod 4 to the fine grids
#pragma unroll
    for (int a = 0; a < U; ++a)
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        a1[a][k] += __shfl_xor_sync(0xffffffffu, a1[a][k], 8);
        a1[a][k] += __shfl_xor_sync(0xffffffffu, a1[a][k], 16);
        ay[a][k] += __shfl_xor_sync(0xffffffffu, ay[a][k], 8);
        ay[a][k] += __shfl_xor_sync(0xffffffffu, ay[a][k], 16);
      }
#pragma unroll
    for (int a = 0; a < U; ++a) {
      if ((a & 3) != qd) continue;
      const int64_t rowi = (int64_t)cs_wrap(sc0 * G + lo + a, n) * n;
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        const int b = c8 + 8 * k;
        if (b < U && (a1[a][k] != 0.0 || ay[a][k] != 0.0)) {
          const int64_t gi = rowi + cs_wrap(sc1 * G + lo + b, n);
          atomicAdd(g1 + gi, a1[a][k]);
          atomicAdd(g2 + gi, ay[a][k]);
        }
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
  long long *tot = nullptr, *off = nullptr, *iof = nullptr;
  double4 *rec = nullptr;
  double *ws1 = nullptr;
  CsItem *items = nullptr;
  EFGP_PALLOC(&hist, sizeof(unsigned) * B * ncell, s);
  EFGP_PALLOC(&tot, sizeof(long long) * ncell, s);
  EFGP_PALLOC(&off, sizeof(long long) * (ncell + 1), s);
  EFGP_PALLOC(&iof, sizeof(long long) * (ncell + 1), s);
  EFGP_PALLOC(&items, sizeof(CsItem) * ((N + kCsRun - 1) / kCsRun + ncell), s);
  EFGP_PALLOC(&rec, sizeof(double4) * N, s);
  if (w1 && D == 3) EFGP_PALLOC(&ws1, sizeof(double) * N, s);
  const size_t sm = sizeof(unsigned) * ncell;
  EFGP_CUDA(cudaFuncSetAttribute(k_cs_count<D, W, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  EFGP_CUDA(cudaFuncSetAttribute(k_cs_scatter<D, W, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  // (the count reads x only: y does not change a key, and the scatter validates y)
  k_cs_count<D, W, G><<<B, T, sm, s>>>(x, nullptr, N, P.h, n, lo, S, ncell, hist, pl->dflags);
  if (getenv("EFGP_CS_SCAN3")) {  // r02 before the fused scan: three launches
    k_het_colscan<<<(ncell + 255) / 256, 256, 0, s>>>(hist, B, ncell, tot);
    EFGP_CUDA(cudaFuncSetAttribute(k_cs_offsets, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_cs_offsets<<<1, 1024, sm, s>>>(tot, ncell, off, iof);
    k_cs_scatter<D, W, G><<<B, T, sm, s>>>(x, y, N, P.h, n, lo, S, ncell, hist, off, rec, pl->dflags, w1, ws1);
    k_cs_items<<<(ncell + 255) / 256, 256, 0, s>>>(off, iof, ncell, items);
  } else {
    // column scan + global bucket offsets (decoupled look-back) + work items in ONE kernel
    const int nsb = (ncell + kScanThreads - 1) / kScanThreads;
    unsigned long long *scan_st = nullptr;
    EFGP_PALLOC(&scan_st, sizeof(unsigned long long) * (nsb + 1), s);
    EFGP_CUDA(cudaMemsetAsync(scan_st, 0, sizeof(unsigned long long) * (nsb + 1), s));
    k_cs_scan<<<nsb, kScanThreads, 0, s>>>(hist, B, ncell, N, off, iof, items, scan_st);
    k_cs_scatter<D, W, G><<<B, T, sm, s>>>(x, y, N, P.h, n, lo, S, ncell, hist, off, rec, pl->dflags, w1, ws1);
    cudaFreeAsync(scan_st, s);
  }
  // (work items on the device, no host round trip: at most ceil(N / kCsRun) + ncell of them)
  EFGP_CUDA(cudaGetLastError());
  int per_sm = 1;
  // quarter-warp 2D layout for union windows up to 12 (EFGP_CS_R01: the r01 layout)
  constexpr bool kQ2 = D == 2 && W + G - 1 <= 12;
  const bool q2 = kQ2 && !getenv("EFGP_CS_R01");
  if constexpr (kQ2) {
    if (q2) EFGP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cs_spread2q<W, G>, kCsThreads, 0));
  }
  if (!q2) EFGP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cs_spread<D, W, G>, kCsThreads, 0));
  const int64_t max_items = (N + kCsRun - 1) / kCsRun + ncell;
  int64_t blocks = std::min<int64_t>((int64_t)pl->num_sms * std::max(per_sm, 1), (max_items * 32 + kCsThreads - 1) / kCsThreads);
  if constexpr (kQ2) {
    if (q2)
      k_cs_spread2q<W, G><<<(unsigned)std::max<int64_t>(blocks, 1), kCsThreads, 0, s>>>(items, iof + ncell, rec, pl->g1,
                                                                                      pl->g2, P.h, n, lo, S, P.poly);
  }
  if (!q2)
    k_cs_spread<D, W, G><<<(unsigned)std::max<int64_t>(blocks, 1), kCsThreads, 0, s>>>(items, iof + ncell, rec, ws1, N,
                                                                                       pl->g1, pl->g2, P.h, n, lo, S, P.poly);
  EFGP_CUDA(cudaGetLastError());
  for (void *p : {(void *)hist, (void *)tot, (void *)off, (void *)iof, (void *)rec, (void *)items}) cudaFreeAsync(p, s);
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
