// K1, SORTED strategy (d = 2, W <= 6): bin-sorted spreading with register accumulation.
//
// Why: a 2D point touches W^2 cells per strength; accumulating each touch with an atomic is bounded
// by the atomic units (shared fp64 atomicAdd is a CAS loop on sm_100a), far below HBM speed
// (DESIGN.md §7).  All points whose footprint starts at the same cell (the "start cell" i0 = ceil(t -
// W/2) per dimension) share one W x W window, so a thread that owns a start cell can accumulate all of
// its points in registers and pay the window update once.
//
// Per chunk of C input points (double-buffered, two streams, so binning of chunk k+1 overlaps the
// accumulation of chunk k):
//   k_bin2   : each CTA loads kBinBatch points (streamed, evict-first), validates them, computes the
//              tile (T x T start cells) of each, counts per tile in shared memory and writes the
//              records (x1, x2, y) into its own region ordered by tile; seg[tile][batch] = (offset,
//              count).  Records stay in L2 for k_tiles2.
//   k_tiles2 : work item = (tile, part of Q).  The tile's records of the chunk are the concatenation of
//              its segments; the work item takes a contiguous 1/Q of them, in rounds of kRound:
//              positions -> load x, classify by start cell (shared counters) -> counting sort ->
//              thread (start cell) accumulates its points into two W x W fp64 register windows
//              (strength 1 and strength y; both on the n1 grid).  At the end the T^2 windows are summed
//              in shared memory in W^2 conflict-free steps and flushed with one RED per cell.
// Geometry (T, Q, C) is chosen on the host (sorted_geometry) for whole waves at 2 CTAs per SM.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "efgp_internal.cuh"

namespace efgp {

constexpr int kBinThreads = 256, kBinPPT = 8, kBinBatch = kBinThreads * kBinPPT;  // 2048 points / CTA
constexpr int kMaxTile = 16;                                                       // T <= 16 (T^2 <= 256)
constexpr int kRound = 8192;                                                       // records per round
constexpr int kClassUnroll = 8;

__device__ __forceinline__ int wrap_s(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

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

template <int W>
__global__ void __launch_bounds__(kBinThreads) k_bin2(const double *__restrict__ x, const double *__restrict__ y,
                                                      int64_t n, double h, int n1, int s_lo, int T, int nt1,
                                                      int ntiles, int nbmax, double2 *__restrict__ rec_x,
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
      px[k] = __ldcs(x2 + i);  // read once: evict-first, keep L2 for the records
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
    const int t = (i1 / T) * nt1 + (i2 / T);
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
    const int64_t p = base + cnt[tl[k]] + rk[k];
    rec_x[p] = px[k];
    rec_y[p] = py[k];
  }
}

template <int W>
__global__ void __launch_bounds__(kMaxTile * kMaxTile, 1)
    k_tiles2(const double2 *__restrict__ rec_x, const double *__restrict__ rec_y, const int2 *__restrict__ seg,
             int nb, int nbmax, int T, int nt1, int Q, double h, int n1, int s_lo, EsPoly P,
             double *__restrict__ g1, double *__restrict__ gy) {
  // NT start cells, NB = blockDim.x = NT rounded up to whole warps (threads >= NT own no cell)
  const int NT = T * T, NB = blockDim.x, A = T + W - 1;
  extern __shared__ __align__(16) unsigned char tsm_raw[];
  double *accs = reinterpret_cast<double *>(tsm_raw);        // 2 A^2
  int *pre = reinterpret_cast<int *>(accs + 2 * A * A);      // nbmax + 1
  int *offb = pre + (nbmax + 1);                             // nbmax
  int *pos = offb + nbmax;                                   // kRound
  int *ccnt = pos + kRound;                                  // kMaxTile^2
  int *wsum = ccnt + kMaxTile * kMaxTile;                    // 32
  unsigned short *rank = reinterpret_cast<unsigned short *>(wsum + 32);  // kRound
  unsigned short *sidx = rank + kRound;                      // kRound
  unsigned char *cell = reinterpret_cast<unsigned char *>(sidx + kRound);  // kRound
  __shared__ int total, bfirst;

  const int tid = threadIdx.x;
  const int tile = blockIdx.x / Q, part = blockIdx.x % Q;
  const int r0 = (tile / nt1) * T, c0 = (tile % nt1) * T;  // tile origin in start cells (0-based)
  for (int b = tid; b < nb; b += NB) {
    const int2 s = seg[(int64_t)tile * nbmax + b];
    pre[b] = s.y;
    offb[b] = s.x;
  }
  __syncthreads();
  block_exclusive_scan(pre, nb, &total, wsum);
  if (tid == 0) pre[nb] = total;
  __syncthreads();
  const int begin = (int)((int64_t)part * total / Q), end = (int)((int64_t)(part + 1) * total / Q);

  double a1[W][W], ay[W][W];
#pragma unroll
  for (int a = 0; a < W; ++a)
#pragma unroll
    for (int b = 0; b < W; ++b) a1[a][b] = ay[a][b] = 0.0;

  const int lane = tid & 31, warp = tid >> 5, nwarps = NB >> 5;
  const bool own = tid < NT;
  for (int rs = begin; rs < end; rs += kRound) {
    const int nr = min(kRound, end - rs);
    if (own) ccnt[tid] = 0;
    if (tid == 0) {  // last segment starting at or before rs
      int lo = 0, hi = nb;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (pre[mid] <= rs) lo = mid;
        else hi = mid;
      }
      bfirst = lo;
    }
    __syncthreads();
    // (1) global position of every record of the round
    for (int b = bfirst + warp; b < nb && pre[b] < rs + nr; b += nwarps) {
      const int lo = max(pre[b], rs), hi = min(pre[b + 1], rs + nr);
      const int basepos = b * kBinBatch + offb[b] - pre[b];
      for (int gi = lo + lane; gi < hi; gi += 32) pos[gi - rs] = basepos + gi;
    }
    __syncthreads();
    // (2) classify by start cell, kClassUnroll loads in flight per thread
    for (int j0 = tid; j0 < nr; j0 += NB * kClassUnroll) {
      double2 xx[kClassUnroll];
#pragma unroll
      for (int u = 0; u < kClassUnroll; ++u) {
        const int j = j0 + u * NB;
        if (j < nr) xx[u] = rec_x[pos[j]];
      }
#pragma unroll
      for (int u = 0; u < kClassUnroll; ++u) {
        const int j = j0 + u * NB;
        if (j < nr) {
          const int i1 = (int)ceil(h * xx[u].x * n1 - 0.5 * W) - s_lo - r0;
          const int i2 = (int)ceil(h * xx[u].y * n1 - 0.5 * W) - s_lo - c0;
          const int c = i1 * T + i2;
          cell[j] = (unsigned char)c;
          rank[j] = (unsigned short)atomicAdd(&ccnt[c], 1);
        }
      }
    }
    __syncthreads();
    // (3) counting sort by start cell
    const int mycnt = own ? ccnt[tid] : 0;
    block_exclusive_scan(ccnt, NT, &total, wsum);  // ccnt <- start offsets
    for (int j = tid; j < nr; j += NB) sidx[ccnt[cell[j]] + rank[j]] = (unsigned short)j;
    __syncthreads();
    // (4) accumulate this thread's start cell; the next record is prefetched from L2
    const int st = own ? ccnt[tid] : 0;
    if (mycnt > 0) {
      int p = pos[sidx[st]];
      double2 xv = rec_x[p];
      double yv = rec_y[p];
      for (int k = 0; k < mycnt; ++k) {
        double2 xn = xv;
        double yn = yv;
        if (k + 1 < mycnt) {
          const int pn = pos[sidx[st + k + 1]];
          xn = rec_x[pn];
          yn = rec_y[pn];
        }
        double w1[W], w2[W];
        es_weights<W>(h * xv.x * n1, P, w1);
        es_weights<W>(h * xv.y * n1, P, w2);
#pragma unroll
        for (int a = 0; a < W; ++a) {
          const double ca = w1[a], cy = yv * w1[a];
#pragma unroll
          for (int b2 = 0; b2 < W; ++b2) {
            a1[a][b2] = fma(ca, w2[b2], a1[a][b2]);
            ay[a][b2] = fma(cy, w2[b2], ay[a][b2]);
          }
        }
        xv = xn;
        yv = yn;
      }
    }
    __syncthreads();
  }
  // sum the windows in shared memory: W^2 conflict-free steps
  for (int i = tid; i < 2 * A * A; i += NB) accs[i] = 0.0;
  __syncthreads();
  const int my_r = tid / T, my_c = tid % T;
#pragma unroll
  for (int a = 0; a < W; ++a) {
#pragma unroll
    for (int b2 = 0; b2 < W; ++b2) {
      if (own) {
        const int idx = (my_r + a) * A + (my_c + b2);
        accs[idx] += a1[a][b2];
        accs[A * A + idx] += ay[a][b2];
      }
      __syncthreads();
    }
  }
  for (int i = tid; i < A * A; i += NB) {
    const double v1 = accs[i], vy = accs[A * A + i];
    if (v1 == 0.0 && vy == 0.0) continue;
    const int r = wrap_s(s_lo + r0 + i / A, n1), c = wrap_s(s_lo + c0 + i % A, n1);
    const int64_t gi = (int64_t)r * n1 + c;
    if (v1 != 0.0) atomicAdd(g1 + gi, v1);
    if (vy != 0.0) atomicAdd(gy + gi, vy);
  }
}

static size_t tiles_smem_bytes(int nbmax, int T, int W) {
  const int A = T + W - 1;
  size_t b = sizeof(double) * 2 * A * A;
  b += sizeof(int) * (size_t)(nbmax + 1 + nbmax + kRound + kMaxTile * kMaxTile + 32);
  b += sizeof(unsigned short) * 2 * kRound + kRound;
  return b;
}

// Tile side T, parts Q and chunk size: whole waves at 2 CTAs per SM, >= ~40 records per start cell
// per work item.
void sorted_geometry(Params &p, int num_sms) {
  p.s_lo = -(p.w / 2);
  const int hi0 = (int)std::ceil(p.h * p.n1 - 0.5 * p.w);
  p.s_count = hi0 - p.s_lo + 1;
  p.bin_batch = kBinBatch;
  p.chunk = int64_t(1) << 21;
  if (const char *e = std::getenv("EFGP_SORTED_CHUNK")) p.chunk = std::max<int64_t>(kBinBatch, std::atoll(e));
  const int nbmax = (int)((p.chunk + kBinBatch - 1) / kBinBatch);
  double best = -1.0;
  for (int T = 8; T <= kMaxTile; ++T) {
    const int nt1 = (p.s_count + T - 1) / T, ntiles = nt1 * nt1;
    // resident CTAs per SM: shared memory (227 KB) and registers (~170 per thread assumed)
    const int by_smem = (int)((227 * 1024) / tiles_smem_bytes(nbmax, T, p.w));
    const int by_regs = 65536 / (216 * ((T * T + 31) / 32) * 32);
    const int slots = std::max(1, std::min(by_smem, by_regs)) * num_sms;
    for (int Q = 1; Q <= 16; ++Q) {
      const int items = ntiles * Q;
      const double waves = std::ceil((double)items / slots);
      const double eff = (double)items / (waves * slots);
      const double per_thread = (double)p.chunk / ((double)items * T * T);
      const double score = eff * std::min(1.0, per_thread / 40.0) * (T * T >= 64 ? 1.0 : 0.5);
      if (score > best + 1e-9) {
        best = score;
        p.tile = T;
        p.ntile1 = nt1;
        p.tile_parts = Q;
      }
    }
  }
  // tuning overrides for experiments (tools/spread_sweep.py)
  if (const char *e = std::getenv("EFGP_SORTED_TILE")) {
    p.tile = std::max(4, std::min(kMaxTile, std::atoi(e)));
    p.ntile1 = (p.s_count + p.tile - 1) / p.tile;
  }
  if (const char *e = std::getenv("EFGP_SORTED_Q")) p.tile_parts = std::max(1, std::atoi(e));
}

template <int W>
static efgp_status run_sorted(efgp_plan *pl, const double *x, const double *y, int64_t N, cudaStream_t s) {
  const Params &P = pl->P;
  const int T = P.tile, nt1 = P.ntile1, ntiles = nt1 * nt1, Q = P.tile_parts;
  const int nbmax = (int)((P.chunk + kBinBatch - 1) / kBinBatch);
  const size_t bsm = sizeof(int) * (size_t)(ntiles + 1 + 32);
  const size_t tsm = tiles_smem_bytes(nbmax, T, W);
  EFGP_CUDA(cudaFuncSetAttribute(k_bin2<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
  EFGP_CUDA(cudaFuncSetAttribute(k_tiles2<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
  cudaStream_t sb = pl->bin_stream;
  EFGP_CUDA(cudaEventRecord(pl->ev_sp, s));
  EFGP_CUDA(cudaStreamWaitEvent(sb, pl->ev_sp, 0));
  int k = 0;
  for (int64_t c0 = 0; c0 < N; c0 += P.chunk, ++k) {
    const int buf = k & 1;
    const int64_t nc = std::min<int64_t>(P.chunk, N - c0);
    const int nb = (int)((nc + kBinBatch - 1) / kBinBatch);
    if (k >= 2) EFGP_CUDA(cudaStreamWaitEvent(sb, pl->ev_tiles[buf], 0));
    k_bin2<W><<<nb, kBinThreads, bsm, sb>>>(x + c0 * 2, y + c0, nc, P.h, (int)P.n1, P.s_lo, T, nt1, ntiles, nbmax,
                                            pl->rec_x[buf], pl->rec_y[buf], pl->seg[buf], pl->dflags);
    EFGP_CUDA(cudaEventRecord(pl->ev_bin[buf], sb));
    EFGP_CUDA(cudaStreamWaitEvent(s, pl->ev_bin[buf], 0));
    k_tiles2<W><<<ntiles * Q, (T * T + 31) / 32 * 32, tsm, s>>>(pl->rec_x[buf], pl->rec_y[buf], pl->seg[buf], nb, nbmax, T, nt1, Q,
                                               P.h, (int)P.n1, P.s_lo, P.poly, pl->g1, pl->g2);
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
