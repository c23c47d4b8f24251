// K1, SORTED strategy (d = 2, W <= 6): tile-binned spreading with register accumulation.
//
// Why: a 2D point touches W^2 cells per strength; accumulating each touch with an atomic is bounded
// by the atomic units (shared fp64 atomicAdd is a CAS loop on sm_100a), far below HBM speed
// (DESIGN.md §7).  All points whose footprint starts at the same cell (the "start cell" i0 = ceil(t -
// W/2) per dimension) share one W x W window, so a thread that owns a start cell accumulates all of
// its points in registers and pays the window update once per tile segment.
//
// The start cells reachable from x in [0,1]^2 form an S x S square (S = s_count); it is cut into
// tiles of T1 x T2 start cells (T1 T2 <= 256, one thread per start cell).  Per chunk of C points
// (double-buffered on two streams, so binning of chunk k+1 overlaps accumulation of chunk k):
//   k_bin3  : each CTA streams 2048 points from HBM (evict-first), validates them, ranks them per
//             tile in shared memory, reserves room in each tile's list with ONE global atomic per
//             (CTA, tile), and writes the (x1, x2, y) records contiguously per tile (the chunk's
//             records, 24 B per point, stay in L2).  A tile list that would exceed its capacity
//             spills the point to direct fp64 RED spreading (correct for any data, fast for spread data).
//   k_tiles3: persistent; CTA b takes the b-th equal share of the concatenated tile lists.  Per round
//             of R records: one bulk async copy (cp.async.bulk + mbarrier, double-buffered) stages the
//             raw records in shared memory; phase A (thread per record, balanced) computes the start
//             cell, its rank (shared int atomics) and, for fp32 weights, the 2W kernel weights; phase B
//             scans the per-cell counts into a sorted index; phase C (thread per start cell)
//             accumulates its records into two W x W fp64 register windows (strength 1 and y, both
//             on the n1 grid).  At a tile change the windows are summed in shared memory in W^2
//             conflict-free steps and flushed with one RED per cell.
// Weights: WF = double evaluates the piecewise polynomial in fp64 (in phase C);  WF = float
// evaluates it in fp32 (phase A) from the fp64 reduced coordinate; accumulation is fp64 in both.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "efgp_internal.cuh"

namespace efgp {

constexpr int kBinThreads = 256, kBinPPT = 8, kBinBatch = kBinThreads * kBinPPT;  // 2048 points / CTA
constexpr int kTileThreads = 256;                                                  // T1 T2 <= 256

__device__ __forceinline__ int wrap_s(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

// grid coordinate of a point in units of the fine-grid spacing: t = h x n (theta / Delta)
// (explicit roundings: binning, classification and weights must agree on the start cell bit for bit)
__device__ __forceinline__ double grid_t(double h, double x, int n) { return __dmul_rn(__dmul_rn(h, x), (double)n); }
template <int W>
__device__ __forceinline__ int start_cell(double t) {
  return (int)ceil(__dsub_rn(t, 0.5 * W));
}

// exclusive scan of n ints in shared memory by a whole block (n arbitrary, blockDim multiple of 32)
__device__ void block_exclusive_scan(int *a, int n, int *total, int *warp_sums) {
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int beg = threadIdx.x * per, end = min(n, beg + per);
  int s = 0;
  for (int i = beg; i < end; ++i) s += a[i];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
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
    if (lane < nw) warp_sums[lane] = w;
  }
  __syncthreads();
  int run = v - s + (wid > 0 ? warp_sums[wid - 1] : 0);
  for (int i = beg; i < end; ++i) {
    const int c = a[i];
    a[i] = run;
    run += c;
  }
  if (threadIdx.x == blockDim.x - 1) *total = run;
  __syncthreads();
}

// fp32 kernel weights from the fp64 grid coordinate: the reduced coordinate s = 2(i0 - t + W/2) - 1
// in [-1, 1] is formed in fp64, the polynomial is evaluated in fp32.
template <int W>
__device__ __forceinline__ void es_weights_f32(double t, const EsPolyF &P, float (&w)[W]) {
  const double tm = __dsub_rn(t, 0.5 * W);
  const float s = (float)(2.0 * (ceil(tm) - tm) - 1.0);
#pragma unroll
  for (int a = 0; a < W; ++a) {
    float acc = P.c[a][W + 2];
#pragma unroll
    for (int k = W + 1; k >= 0; --k) acc = fmaf(acc, s, P.c[a][k]);
    w[a] = acc;
  }
}

// the same for both coordinates of a 2D point at once, with packed fp32x2 FMAs (FFMA2)
template <int W>
__device__ __forceinline__ void es_weights_f32x2(double t1, double t2, const EsPolyF &P, float (&w1)[W],
                                                 float (&w2)[W]) {
  const double tm1 = __dsub_rn(t1, 0.5 * W), tm2 = __dsub_rn(t2, 0.5 * W);
  const float2 s = make_float2((float)(2.0 * (ceil(tm1) - tm1) - 1.0), (float)(2.0 * (ceil(tm2) - tm2) - 1.0));
#pragma unroll
  for (int a = 0; a < W; ++a) {
    float2 acc = make_float2(P.c[a][W + 2], P.c[a][W + 2]);
#pragma unroll
    for (int k = W + 1; k >= 0; --k) acc = __ffma2_rn(acc, s, make_float2(P.c[a][k], P.c[a][k]));
    w1[a] = acc.x;
    w2[a] = acc.y;
  }
}

// direct fp64 RED spreading of one point (overflow path; the polynomial is read from global memory so
// the kernel parameters are not copied to the stack)
template <int W>
__device__ __noinline__ void spread_point_red(double x1, double x2, double yv, double h, int n1,
                                              const EsPoly *__restrict__ Pg, double *__restrict__ g1,
                                              double *__restrict__ gy) {
  double w1[W], w2[W];
  const int b1 = es_weights<W>(grid_t(h, x1, n1), *Pg, w1);
  const int b2 = es_weights<W>(grid_t(h, x2, n1), *Pg, w2);
#pragma unroll 1
  for (int a = 0; a < W; ++a) {
    const int64_t row = (int64_t)wrap_s(b1 + a, n1) * n1;
#pragma unroll
    for (int b = 0; b < W; ++b) {
      const int64_t gi = row + wrap_s(b2 + b, n1);
      const double p = w1[a] * w2[b];
      atomicAdd(g1 + gi, p);
      atomicAdd(gy + gi, p * yv);
    }
  }
}

// ---- bulk async copy global -> shared with an mbarrier (TMA engine, 1D) -----------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// exclusive scan of one int per thread over the block (blockDim = 256); returns the exclusive prefix
__device__ __forceinline__ int block_scan_256(int v, int *wsum) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int s = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, s, o);
    if (lane >= o) s += t;
  }
  if (lane == 31) wsum[wid] = s;
  __syncthreads();
  if (wid == 0) {
    int w = lane < 8 ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    if (lane < 8) wsum[lane] = w;
  }
  __syncthreads();
  return s - v + (wid > 0 ? wsum[wid - 1] : 0);
}

// K1a: bin the chunk's points by tile.  Persistent CTAs (2 per SM) walk the chunk's batches of
// kBinBatch points; the next batch's x and y arrive by bulk async copy (TMA engine, mbarrier) while
// the current one is processed, so HBM reads stay in flight without holding registers.  Per batch:
// validate, start cells -> tile (shared lookup tables, no integer division), rank per tile (shared
// int atomics), ONE global atomic per non-empty tile reserves room in its list, then the records
// (x1, x2, y) are written tile-contiguously with coalesced stores (24 B per point, into L2).
constexpr int kBinMaxS = 8192;  // start cells per dimension supported by the lookup tables

template <int W>
__global__ void __launch_bounds__(kBinThreads, 2)
    k_bin5(const double *__restrict__ x, const double *__restrict__ y, int64_t n, double h, int n1, int s_lo, int S,
           int T1, int T2, int nt2, int ntiles, int cap, double *__restrict__ rec, int *__restrict__ gcnt,
           const EsPoly *__restrict__ Pg, double *__restrict__ g1, double *__restrict__ gy, int *__restrict__ err) {
  extern __shared__ __align__(16) unsigned char bsm[];
  double *xin = reinterpret_cast<double *>(bsm);                     // [2][kBinBatch * 2]
  double *yin = xin + 2 * 2 * kBinBatch;                             // [2][kBinBatch]
  int *perm = reinterpret_cast<int *>(yin + 2 * kBinBatch);          // [kBinBatch] slot -> j | t << 16
  int *cnt = perm + kBinBatch;                                       // ntiles
  int *loc = cnt + ntiles;                                           // ntiles
  int *base = loc + ntiles;                                          // ntiles
  int *rowt = base + ntiles;                                         // S: (c1 / T1) * nt2
  int *colt = rowt + S;                                              // S: c2 / T2
  __shared__ int wsum[32], total;
  __shared__ __align__(8) uint64_t bar[2];
  const int tid = threadIdx.x;
  const int64_t nbatch = (n + kBinBatch - 1) / kBinBatch;
  for (int c = tid; c < S; c += kBinThreads) {
    rowt[c] = (c / T1) * nt2;
    colt[c] = c / T2;
  }
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t b, int buf) {
    if (tid == 0 && b < nbatch) {
      const int64_t i0 = b * kBinBatch;
      const int nb = (int)(n - i0 < (int64_t)kBinBatch ? n - i0 : (int64_t)kBinBatch);
      const int ne = nb & ~1;  // y copies need a multiple of 16 bytes; an odd tail is loaded below
      const uint32_t bytes = (uint32_t)(nb * 16 + ne * 8);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[buf])), "r"(bytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(xin + buf * 2 * kBinBatch)),
          "l"(x + 2 * i0), "r"((uint32_t)(nb * 16)), "r"(smem_u32(&bar[buf]))
          : "memory");
      if (ne > 0)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(yin + buf * kBinBatch)),
            "l"(y + i0), "r"((uint32_t)(ne * 8)), "r"(smem_u32(&bar[buf]))
            : "memory");
    }
  };
  uint32_t phase[2] = {0u, 0u};
  int buf = 0;
  issue(blockIdx.x, 0);
  issue(blockIdx.x + gridDim.x, 1);
  for (int64_t b = blockIdx.x; b < nbatch; b += gridDim.x, buf ^= 1) {
    const int64_t i0 = b * kBinBatch;
    const int nb = (int)(n - i0 < (int64_t)kBinBatch ? n - i0 : (int64_t)kBinBatch);
    for (int t = tid; t < ntiles; t += kBinThreads) cnt[t] = 0;
    mbar_wait(&bar[buf], phase[buf]);
    phase[buf] ^= 1u;
    const double *xs = xin + buf * 2 * kBinBatch;
    double *ys = yin + buf * kBinBatch;
    if ((nb & 1) && tid == 0) ys[nb - 1] = y[i0 + nb - 1];
    __syncthreads();
    int tl[kBinPPT], rk[kBinPPT];
#pragma unroll
    for (int k = 0; k < kBinPPT; ++k) {
      const int j = k * kBinThreads + tid;
      tl[k] = -1;
      if (j >= nb) continue;
      const double2 p = *reinterpret_cast<const double2 *>(xs + 2 * j);
      const double yv = ys[j];
      const bool ok = p.x >= 0.0 && p.x <= 1.0 && p.y >= 0.0 && p.y <= 1.0 && isfinite(yv);
      if (!ok) {
        atomicOr(err, 1);
        continue;
      }
      const int c1 = start_cell<W>(grid_t(h, p.x, n1)) - s_lo;
      const int c2 = start_cell<W>(grid_t(h, p.y, n1)) - s_lo;
      const int t = rowt[c1] + colt[c2];
      tl[k] = t;
      rk[k] = atomicAdd(&cnt[t], 1);
    }
    __syncthreads();
    for (int t = tid; t < ntiles; t += kBinThreads) {
      const int c = cnt[t];
      loc[t] = c;
      base[t] = c ? atomicAdd(gcnt + t, c) : 0;
    }
    __syncthreads();
    block_exclusive_scan(loc, ntiles, &total, wsum);
#pragma unroll
    for (int k = 0; k < kBinPPT; ++k)
      if (tl[k] >= 0) perm[loc[tl[k]] + rk[k]] = (k * kBinThreads + tid) | (tl[k] << 16);
    __syncthreads();
    const int nv = total;
    for (int e = tid; e < 3 * nv; e += kBinThreads) {
      const int slot = e / 3, comp = e - 3 * slot;
      const int v = perm[slot];
      const int j = v & 0xFFFF, t = v >> 16;
      const int p = base[t] + slot - loc[t];
      const double val = comp < 2 ? xs[2 * j + comp] : ys[j];
      if (p < cap) {
        rec[((int64_t)t * cap + p) * 3 + comp] = val;
      } else if (comp == 0) {
        spread_point_red<W>(xs[2 * j], xs[2 * j + 1], ys[j], h, n1, Pg, g1, gy);
      }
    }
    __syncthreads();  // this buffer is consumed: refill it with the batch after next
    issue(b + 2 * (int64_t)gridDim.x, buf);
  }
}

// Spreading modes of the accumulation kernel
constexpr int kModeF64 = 0;   // fp64 weights (evaluated per record in phase C), fp64 accumulation
constexpr int kModeW32 = 1;   // fp32 weights (phase A), fp64 accumulation
constexpr int kModeA32 = 2;   // fp32 weights, fp32 (packed FFMA2) accumulation within a round, fp64 across

template <int W, int MODE>
struct StageRec {
  // MODE 0: sorted copy of (x1, x2, y); else: w1[W], w2[W] (fp32) then y (fp64), 16-byte padded
  static constexpr int kBytes = MODE == kModeF64 ? 24 : ((8 * W + 8) + 15) / 16 * 16;
};

template <int W, int MODE>
__device__ __forceinline__ void load_stage_w(const unsigned char *sp, float (&w1)[W], float (&w2)[W], double &yv) {
  constexpr int NF = 2 * W, NV = (NF + 3) / 4;
  float f[NV * 4];
  const float4 *q = reinterpret_cast<const float4 *>(sp);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const float4 v = q[i];
    f[4 * i] = v.x;
    f[4 * i + 1] = v.y;
    f[4 * i + 2] = v.z;
    f[4 * i + 3] = v.w;
  }
#pragma unroll
  for (int a = 0; a < W; ++a) {
    w1[a] = f[a];
    w2[a] = f[W + a];
  }
  yv = *reinterpret_cast<const double *>(sp + 8 * W);
}

// K1b: persistent accumulation.  CTA b takes the b-th equal share of the concatenated tile lists.
template <int W, int MODE>
__global__ void __launch_bounds__(kTileThreads, 1)
    k_tiles4(const double *__restrict__ rec, const int *__restrict__ gcnt, int cap, int ntiles, int T1, int T2,
             int nt2, int R, double h, int n1, int s_lo, EsPoly P, EsPolyF PF, double *__restrict__ g1,
             double *__restrict__ gy) {
  constexpr int SB = StageRec<W, MODE>::kBytes;
  extern __shared__ __align__(16) unsigned char tsm[];
  // layout: raw[(R + 2) * 3] doubles | stage[R * SB] | kr[R] | cnt[256] | tpre[ntiles + 1]
  double *raw = reinterpret_cast<double *>(tsm);
  unsigned char *stage = tsm + sizeof(double) * (size_t)(R + 2) * 3;
  int *kr = reinterpret_cast<int *>(stage + (size_t)R * SB);
  int *cnt = kr + R;
  int *tpre = cnt + kTileThreads;
  __shared__ int wsum[32];
  __shared__ int total;
  __shared__ __align__(8) uint64_t bar;

  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int t = tid; t < ntiles; t += kTileThreads) tpre[t] = min(gcnt[t], cap);
  __syncthreads();
  block_exclusive_scan(tpre, ntiles, &total, wsum);
  if (tid == 0) tpre[ntiles] = total;
  __syncthreads();
  const int all = tpre[ntiles];
  const int gb = (int)((int64_t)blockIdx.x * all / gridDim.x), ge = (int)((int64_t)(blockIdx.x + 1) * all / gridDim.x);
  if (gb >= ge) return;
  int t_first = 0;  // last tile with tpre[t] <= gb (binary search; identical in all threads)
  {
    int lo = 0, hi = ntiles;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (tpre[mid] <= gb) lo = mid;
      else hi = mid;
    }
    t_first = lo;
    while (tpre[t_first + 1] <= gb) ++t_first;  // skip empty tiles ending at gb
  }
  const int NT = T1 * T2;
  const bool own = tid < NT;
  const int my_r = own ? tid / T2 : 0, my_c = own ? tid % T2 : 0;
  const int A1 = T1 + W - 1, A2 = T2 + W - 1;
  uint32_t phase = 0u;

  struct Rd {
    int tile, lo, n;
  };
  auto round_at = [&](int t, int lo) -> Rd {
    const int hi = min(tpre[t + 1], ge) - tpre[t];
    return Rd{t, lo, min(R, hi - lo)};
  };
  auto next_round = [&](Rd r) -> Rd {
    const int tile_hi = min(tpre[r.tile + 1], ge) - tpre[r.tile];
    if (r.lo + r.n < tile_hi) return round_at(r.tile, r.lo + r.n);
    int t = r.tile + 1;
    while (t < ntiles && tpre[t] < ge && tpre[t + 1] == tpre[t]) ++t;
    if (t >= ntiles || tpre[t] >= ge) return Rd{-1, 0, 0};
    return round_at(t, 0);
  };
  // bulk copy of round r into raw (aligned superset: records are 24 B, copies need 16 B alignment)
  auto issue = [&](Rd r) {
    if (tid == 0 && r.tile >= 0) {
      const int64_t first = (int64_t)r.tile * cap + r.lo;
      const int64_t a0 = first & ~int64_t(1), a1 = (first + r.n + 1) & ~int64_t(1);
      bulk_load(raw, rec + a0 * 3, (uint32_t)((a1 - a0) * 24), &bar);
    }
  };

  double a1[W][W], ay[W][W];
#pragma unroll
  for (int a = 0; a < W; ++a)
#pragma unroll
    for (int b = 0; b < W; ++b) a1[a][b] = ay[a][b] = 0.0;

  Rd cur = round_at(t_first, gb - tpre[t_first]);
  issue(cur);
  while (cur.tile >= 0) {
    const Rd nxt = next_round(cur);
    const int r0 = (cur.tile / nt2) * T1, c0 = (cur.tile % nt2) * T2;
    const int nr = cur.n;
    const double *rw = raw + 3 * (int)(((int64_t)cur.tile * cap + cur.lo) & 1);
    cnt[tid] = 0;
    mbar_wait(&bar, phase);
    phase ^= 1u;
    __syncthreads();
    // pass 1 (thread per record): start cell within the tile and its rank
    for (int j = tid; j < nr; j += kTileThreads) {
      const double t1 = grid_t(h, rw[3 * j], n1), t2 = grid_t(h, rw[3 * j + 1], n1);
      const int key = (start_cell<W>(t1) - s_lo - r0) * T2 + (start_cell<W>(t2) - s_lo - c0);
      kr[j] = key | (atomicAdd(&cnt[key], 1) << 8);
    }
    __syncthreads();
    const int mycnt = cnt[tid];
    const int myoff = block_scan_256(mycnt, wsum);
    cnt[tid] = myoff;
    __syncthreads();
    // pass 2 (thread per record): write the record (MODE 0) or its fp32 weights at its sorted slot
    for (int j = tid; j < nr; j += kTileThreads) {
      const int v = kr[j];
      const int pos = cnt[v & 255] + (v >> 8);
      unsigned char *sp = stage + (size_t)pos * SB;
      if constexpr (MODE == kModeF64) {
        double *d = reinterpret_cast<double *>(sp);
        d[0] = rw[3 * j];
        d[1] = rw[3 * j + 1];
        d[2] = rw[3 * j + 2];
      } else {
        float w1[W], w2[W];
        es_weights_f32x2<W>(grid_t(h, rw[3 * j], n1), grid_t(h, rw[3 * j + 1], n1), PF, w1, w2);
        float f[4 * ((2 * W + 3) / 4)];
#pragma unroll
        for (int a = 0; a < W; ++a) {
          f[a] = w1[a];
          f[W + a] = w2[a];
        }
#pragma unroll
        for (int i = 2 * W; i < 4 * ((2 * W + 3) / 4); ++i) f[i] = 0.f;
        float4 *q = reinterpret_cast<float4 *>(sp);
#pragma unroll
        for (int i = 0; i < (2 * W + 3) / 4; ++i) q[i] = make_float4(f[4 * i], f[4 * i + 1], f[4 * i + 2], f[4 * i + 3]);
        *reinterpret_cast<double *>(sp + 8 * W) = rw[3 * j + 2];
      }
    }
    __syncthreads();
    issue(nxt);  // raw is free: the next round's copy lands during phase C
    // phase C (thread per start cell): register accumulation of its records
    if (mycnt > 0) {
      const unsigned char *sp = stage + (size_t)myoff * SB;
      if constexpr (MODE == kModeF64) {
        for (int k = 0; k < mycnt; ++k, sp += SB) {
          const double *d = reinterpret_cast<const double *>(sp);
          const double yv = d[2];
          double w1[W], w2[W];
          es_weights<W>(grid_t(h, d[0], n1), P, w1);
          es_weights<W>(grid_t(h, d[1], n1), P, w2);
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
      } else if constexpr (MODE == kModeW32) {
        for (int k = 0; k < mycnt; ++k, sp += SB) {
          float w1[W], w2[W];
          double yv;
          load_stage_w<W, MODE>(sp, w1, w2, yv);
#pragma unroll
          for (int a = 0; a < W; ++a) {
            const double ca = (double)w1[a], cy = yv * (double)w1[a];
#pragma unroll
            for (int b2 = 0; b2 < W; ++b2) {
              const double wb = (double)w2[b2];
              a1[a][b2] = fma(ca, wb, a1[a][b2]);
              ay[a][b2] = fma(cy, wb, ay[a][b2]);
            }
          }
        }
      } else {
        float2 acc[W][W];
#pragma unroll
        for (int a = 0; a < W; ++a)
#pragma unroll
          for (int b2 = 0; b2 < W; ++b2) acc[a][b2] = make_float2(0.f, 0.f);
        for (int k = 0; k < mycnt; ++k, sp += SB) {
          float w1[W], w2[W];
          double yv;
          load_stage_w<W, MODE>(sp, w1, w2, yv);
          const float yf = (float)yv;
#pragma unroll
          for (int a = 0; a < W; ++a) {
            const float2 pa = make_float2(w1[a], yf * w1[a]);
#pragma unroll
            for (int b2 = 0; b2 < W; ++b2) acc[a][b2] = __ffma2_rn(pa, make_float2(w2[b2], w2[b2]), acc[a][b2]);
          }
        }
#pragma unroll
        for (int a = 0; a < W; ++a)
#pragma unroll
          for (int b2 = 0; b2 < W; ++b2) {
            a1[a][b2] += (double)acc[a][b2].x;
            ay[a][b2] += (double)acc[a][b2].y;
          }
      }
    }
    __syncthreads();  // stage, kr, cnt free
    // flush the windows at the end of a tile segment: W^2 conflict-free steps into shared memory,
    // then one RED per cell
    if (nxt.tile != cur.tile) {
      double *acc = reinterpret_cast<double *>(stage);
      for (int i = tid; i < 2 * A1 * A2; i += kTileThreads) acc[i] = 0.0;
      __syncthreads();
#pragma unroll
      for (int a = 0; a < W; ++a) {
#pragma unroll
        for (int b2 = 0; b2 < W; ++b2) {
          if (own) {
            const int idx = (my_r + a) * A2 + (my_c + b2);
            acc[idx] += a1[a][b2];
            acc[A1 * A2 + idx] += ay[a][b2];
          }
          a1[a][b2] = ay[a][b2] = 0.0;
          __syncthreads();
        }
      }
      for (int i = tid; i < A1 * A2; i += kTileThreads) {
        const double v1 = acc[i], vy = acc[A1 * A2 + i];
        const int r = wrap_s(s_lo + r0 + i / A2, n1), c = wrap_s(s_lo + c0 + i % A2, n1);
        const int64_t gi = (int64_t)r * n1 + c;
        if (v1 != 0.0) atomicAdd(g1 + gi, v1);
        if (vy != 0.0) atomicAdd(gy + gi, vy);
      }
      __syncthreads();
    }
    cur = nxt;
  }
}

template <int W, int MODE>
static size_t tiles_smem_bytes(int R, int ntiles) {
  size_t b = sizeof(double) * (size_t)(R + 2) * 3;        // raw
  b += (size_t)R * StageRec<W, MODE>::kBytes;             // stage
  b += 4 * (size_t)R;                                     // kr
  b += 4 * (size_t)(kTileThreads + ntiles + 1);           // cnt, tpre
  return b;
}
static size_t bin_smem_bytes(int ntiles, int S) {
  return sizeof(double) * 2 * 3 * kBinBatch + sizeof(int) * kBinBatch + sizeof(int) * (3 * (size_t)ntiles + 2 * S);
}

// Tile shape (T1 x T2 start cells, T1 T2 <= 256, least covered area), chunk, capacity, round size.
void sorted_geometry(Params &p, int num_sms) {
  p.s_lo = -(p.w / 2);
  const int hi0 = (int)std::ceil(p.h * p.n1 - 0.5 * p.w);
  p.s_count = hi0 - p.s_lo + 1;
  const int S = p.s_count;
  int64_t best = -1;
  for (int T2 = 6; T2 <= 64; ++T2) {
    const int T1 = std::min(kTileThreads / T2, S);
    if (T1 < 4) continue;
    const int64_t nt1 = (S + T1 - 1) / T1, nt2 = (S + T2 - 1) / T2;
    const int64_t cover = nt1 * T1 * nt2 * T2;
    if (nt1 * nt2 > 4096) continue;
    if (best < 0 || cover < best) {
      best = cover;
      p.T1 = T1;
      p.T2 = T2;
      p.nt1 = (int)nt1;
      p.nt2 = (int)nt2;
    }
  }
  if (const char *e = std::getenv("EFGP_SORTED_T2")) {
    p.T2 = std::max(4, std::min(64, std::atoi(e)));
    p.T1 = std::min(kTileThreads / p.T2, S);
    p.nt1 = (S + p.T1 - 1) / p.T1;
    p.nt2 = (S + p.T2 - 1) / p.T2;
  }
  p.ntiles = p.nt1 * p.nt2;
  p.chunk = int64_t(1) << 21;
  if (const char *e = std::getenv("EFGP_SORTED_CHUNK")) p.chunk = std::max<int64_t>(kBinBatch, std::atoll(e));
  // capacity per tile list: 2x the uniform share + slack; overflow spills to direct RED spreading
  const double share = (double)p.chunk * p.T1 * p.T2 / ((double)S * S);
  p.cap = (int)std::min<double>((double)p.chunk, 2.0 * share + 8192.0);
  p.cap = (p.cap + 1) & ~1;
  p.tiles_grid = num_sms;
  p.bin_grid = 2 * num_sms;
  if (const char *e = std::getenv("EFGP_BIN_GRID")) p.bin_grid = std::max(1, std::atoi(e));
  if (const char *e = std::getenv("EFGP_SORTED_GRID")) p.tiles_grid = std::max(1, std::atoi(e));
  // round size: the largest multiple of 256 whose shared memory fits 227 KB
  const size_t lim = 224 * 1024;
  int R = 256;
  for (int r = 256; r <= 16384; r += 256) {
    size_t need = 0;
    switch (p.w) {
#define EFGP_SZ(WW)                                                   \
  case WW:                                                            \
    need = p.spread_mode == 0   ? tiles_smem_bytes<WW, 0>(r, p.ntiles) \
           : p.spread_mode == 1 ? tiles_smem_bytes<WW, 1>(r, p.ntiles) \
                                : tiles_smem_bytes<WW, 2>(r, p.ntiles); \
    break;
      EFGP_SZ(2) EFGP_SZ(3) EFGP_SZ(4) EFGP_SZ(5) EFGP_SZ(6)
#undef EFGP_SZ
    }
    if (need <= lim) R = r;
  }
  if (const char *e = std::getenv("EFGP_SORTED_R")) R = std::max(256, std::min(R, std::atoi(e) / 256 * 256));
  p.round = R;
}

template <int W>
static efgp_status run_sorted(efgp_plan *pl, const double *x, const double *y, int64_t N, cudaStream_t s) {
  const Params &P = pl->P;
  const int ntiles = P.ntiles, R = P.round;
  const size_t bsm = bin_smem_bytes(ntiles, P.s_count);
  const int mode = P.spread_mode;
  const size_t tsm = mode == 0 ? tiles_smem_bytes<W, 0>(R, ntiles)
                     : mode == 1 ? tiles_smem_bytes<W, 1>(R, ntiles) : tiles_smem_bytes<W, 2>(R, ntiles);
  auto ktiles = mode == 0 ? k_tiles4<W, 0> : mode == 1 ? k_tiles4<W, 1> : k_tiles4<W, 2>;
  EFGP_CUDA(cudaFuncSetAttribute(k_bin5<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
  EFGP_CUDA(cudaFuncSetAttribute(ktiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
  cudaStream_t sb = pl->bin_stream;
  EFGP_CUDA(cudaEventRecord(pl->ev_sp, s));
  EFGP_CUDA(cudaStreamWaitEvent(sb, pl->ev_sp, 0));
  int k = 0;
  for (int64_t c0 = 0; c0 < N; c0 += P.chunk, ++k) {
    const int buf = k & 1;
    const int64_t nc = std::min<int64_t>(P.chunk, N - c0);
    const int nb = (int)((nc + kBinBatch - 1) / kBinBatch);
    if (k >= 2) EFGP_CUDA(cudaStreamWaitEvent(sb, pl->ev_tiles[buf], 0));
    EFGP_CUDA(cudaMemsetAsync(pl->tcnt[buf], 0, sizeof(int) * ntiles, sb));
    const int bgrid = (int)std::min<int64_t>((int64_t)P.bin_grid, nb);
    k_bin5<W><<<bgrid, kBinThreads, bsm, sb>>>(x + c0 * 2, y + c0, nc, P.h, (int)P.n1, P.s_lo, P.s_count, P.T1, P.T2,
                                               P.nt2, ntiles, P.cap, pl->rec[buf], pl->tcnt[buf], pl->poly_dev, pl->g1,
                                               pl->g2, pl->dflags);
    EFGP_CUDA(cudaEventRecord(pl->ev_bin[buf], sb));
    EFGP_CUDA(cudaStreamWaitEvent(s, pl->ev_bin[buf], 0));
    ktiles<<<P.tiles_grid, kTileThreads, tsm, s>>>(pl->rec[buf], pl->tcnt[buf], P.cap, ntiles, P.T1, P.T2, P.nt2, R,
                                                   P.h, (int)P.n1, P.s_lo, P.poly, P.polyf, pl->g1, pl->g2);
    EFGP_CUDA(cudaEventRecord(pl->ev_tiles[buf], s));
  }
  EFGP_CUDA(cudaGetLastError());
  return EFGP_OK;
}

efgp_status spread_sorted2(efgp_plan *pl, const double *x, const double *y, int64_t N, cudaStream_t s) {
  switch (pl->P.w) {
    case 2: return run_sorted<2>(pl, x, y, N, s);
    case 3: return run_sorted<3>(pl, x, y, N, s);
    case 4: return run_sorted<4>(pl, x, y, N, s);
    case 5: return run_sorted<5>(pl, x, y, N, s);
    case 6: return run_sorted<6>(pl, x, y, N, s);
  }
  pl->err = "internal: SORTED spreading needs w <= 6";
  return EFGP_ERR_INVALID;
}

}  // namespace efgp
