// NEXT-3: heteroskedastic noise sigma_n (reading G11).
//
// Weight space with S = diag(sigma_n^2):  (Phi^* S^-1 Phi + I) beta = Phi^* S^-1 y,  mu = phi(x*) beta.
// S breaks the Toeplitz structure of Phi^*Phi, so every CG product is applied "as in BBMM
// methods" with one NUFFT pair over the N points:
//
//   A p = D . F^*( S^-1 . F(D . p) ) + p
//       = K2_rhs( K1( x, K9( x, C2R(K8(p)) ) / sigma^2 ) ) + p
//
// K8 places D p / phi^2 on the type-2 box, cuFFT C2R gives the fine grid, K9 interpolates it at the
// data points and divides by sigma_n^2 (fused), K1 spreads those values (the same spreader as the
// fit; its strength-y grid is the one used), cuFFT R2C + k_het_modes deconvolve, multiply by D and
// add p.  The right-hand side is the same K1 -> R2C -> k_het_modes chain on y_n / sigma_n^2.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "efgp_internal.cuh"

namespace efgp {

// w_n = y_n * (1 / sigma_n^2); raise dflags[2] for sigma_n <= 0 or non-finite; min sigma_n into *minbits
// (for positive doubles the IEEE bit pattern is ordered like the value)
__global__ void k_het_prep(const double *__restrict__ y, const double *__restrict__ sd, int64_t N,
                           double *__restrict__ w, unsigned long long *__restrict__ minbits, int *__restrict__ err,
                           double *__restrict__ iv = nullptr) {
  unsigned long long lmin = ~0ull;
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const double s = sd[i];
    const bool ok = s > 0.0 && isfinite(s);
    bad |= !ok;
    // y_n * rcp(sigma_n^2): one IEEE reciprocal and a product — the roundings of the SORTED kernel's
    // pass 2, which forms the same two strengths from the raw (y_n, sigma_n)
    const double r = ok ? __drcp_rn(s * s) : 0.0;
    w[i] = ok ? y[i] * r : 0.0;
    if (iv) iv[i] = r;
    if (ok) {
      const unsigned long long b = (unsigned long long)__double_as_longlong(s);
      lmin = b < lmin ? b : lmin;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, lmin, o);
    lmin = t < lmin ? t : lmin;
  }
  if ((threadIdx.x & 31) == 0 && lmin != ~0ull) atomicMin(minbits, lmin);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err + 2, 1);
}

// out_q = D_q f_q + (p ? p_q : 0),  f_j = Delta^d G^(j) / prod phi(j_k) on the J_m half (type-1
// deconvolution of the strength-w grid, as K2)
template <int D>
__global__ void k_het_modes(const double2 *__restrict__ G, int64_t n, int m, const double *__restrict__ psi,
                            double sc, const double *__restrict__ Dh, const double2 *__restrict__ p,
                            double2 *__restrict__ out, int64_t Mh) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x) {
    int j[D];
    decode_half<D>(q, m, j);
    double den = 1.0;
#pragma unroll
    for (int k = 0; k < D; ++k) den *= psi[j[k] < 0 ? -j[k] : j[k]];
    const double2 g = G[box_index<D>(j, n)];
    const double f = Dh[q] * sc / den;
    double2 o = make_double2(f * g.x, f * g.y);
    if (p) {
      const double2 pp = p[q];
      o.x += pp.x;
      o.y += pp.y;
    }
    out[q] = o;
  }
}


// ---- sorted NUFFT-pair product (d <= 2): the points never move between CG iterations, so they are
// counting-sorted ONCE by their start cell on the type-2 grid n2 (structure of arrays: coordinates
// and 1/sigma_n^2).  Each iteration is then one streaming pass: a warp takes a run of one cell's
// points (lanes stride 32, coalesced), holds that cell's W^d grid window in registers, and per point
// evaluates the kernel weights once and uses them twice: u = sum g w (type-2 at the point),
// v = u / sigma_n^2, window += v w (type-1 of v).  The lanes' windows are reduced with shuffles and
// added to the output grid with W^d atomics per run.  Both transforms use the same grid, kernel and
// deconvolution, so the product is exactly Hermitian.
#ifndef EFGP_HET_RUN
#define EFGP_HET_RUN 2048
#endif
constexpr int kHetRun = EFGP_HET_RUN;  // points per warp work item (64 per lane)

struct HetItem {
  long long begin, end;
  int cell, pad_;
};

template <int D, int W>
__device__ __forceinline__ int het_cell_key(const double *__restrict__ x, int64_t i, double h, int n, int lo, int S) {
  int key = 0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const double t = __dmul_rn(__dmul_rn(h, __ldg(x + i * D + k)), (double)n);  // = K9's h x n
    int c = (int)ceil(__dsub_rn(t, 0.5 * W)) - lo;                             // es_weights' i0
    c = c < 0 ? 0 : (c >= S ? S - 1 : c);  // never taken: S covers x in [0,1] (validated before)
    key = key * S + c;
  }
  return key;
}

__device__ __forceinline__ void het_range(int64_t N, int64_t &a, int64_t &e) {
  const int64_t per = (N + gridDim.x - 1) / gridDim.x;
  a = (int64_t)blockIdx.x * per;
  e = a + per < N ? a + per : N;
}

template <int D, int W>
__global__ void k_het_count(const double *__restrict__ x, int64_t N, double h, int n, int lo, int S, int ncell,
                            unsigned *__restrict__ hist) {
  extern __shared__ unsigned hs[];
  for (int i = threadIdx.x; i < ncell; i += blockDim.x) hs[i] = 0;
  __syncthreads();
  int64_t a, e;
  het_range(N, a, e);
  for (int64_t i = a + threadIdx.x; i < e; i += blockDim.x) atomicAdd(&hs[het_cell_key<D, W>(x, i, h, n, lo, S)], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < ncell; i += blockDim.x) hist[(size_t)blockIdx.x * ncell + i] = hs[i];
}

// per cell: exclusive scan over the CTAs (in place) and the cell total
__global__ void k_het_colscan(unsigned *__restrict__ hist, int nblk, int ncell, long long *__restrict__ tot) {
  // hist[b][c] -> exclusive prefix over b (column scan), tot[c] = column total.  The loads of a
  // chunk of rows are issued before any store (no aliasing stall: r01 did one dependent load/store
  // pair per row, ~1 us per row of latency at 148 rows)
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncell) return;
  constexpr int kChunk = 16;
  long long run = 0;
  for (int b0 = 0; b0 < nblk; b0 += kChunk) {
    unsigned v[kChunk];
#pragma unroll
    for (int k = 0; k < kChunk; ++k) v[k] = b0 + k < nblk ? __ldcg(hist + (size_t)(b0 + k) * ncell + c) : 0u;
#pragma unroll
    for (int k = 0; k < kChunk; ++k) {
      if (b0 + k < nblk) hist[(size_t)(b0 + k) * ncell + c] = (unsigned)run;  // < 2^32 points per cell
      run += v[k];
    }
  }
  tot[c] = run;
}

// off[c] = sum_{c' < c} tot[c'], off[ncell] = N (one CTA of 1024 threads: each thread scans a
// contiguous slice serially, one block scan of the slice totals, then the slices are written)
__global__ void k_het_offsets(const long long *__restrict__ tot, int ncell, long long *__restrict__ off) {
  __shared__ long long wsum[32];
  const int t = threadIdx.x, nt = blockDim.x, lane = t & 31, wid = t >> 5;
  const int per = (ncell + nt - 1) / nt, a = t * per, e = min(ncell, a + per);
  long long s = 0;
  for (int c = a; c < e; ++c) s += tot[c];
  long long incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    long long w = lane < (nt >> 5) ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long v = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += v;
    }
    wsum[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  long long run = incl - s + (wid > 0 ? wsum[wid - 1] : 0);
  for (int c = a; c < e; ++c) {
    off[c] = run;
    run += tot[c];
  }
  if (t == nt - 1) off[ncell] = run;
}

template <int D, int W>
__global__ void k_het_scatter(const double *__restrict__ x, const double *__restrict__ sd, int64_t N, double h, int n,
                              int lo, int S, int ncell, const unsigned *__restrict__ hist,
                              const long long *__restrict__ off, double *__restrict__ xs, double *__restrict__ is2) {
  extern __shared__ unsigned long long cur[];
  for (int i = threadIdx.x; i < ncell; i += blockDim.x)
    cur[i] = (unsigned long long)(off[i] + hist[(size_t)blockIdx.x * ncell + i]);
  __syncthreads();
  int64_t a, e;
  het_range(N, a, e);
  for (int64_t i = a + threadIdx.x; i < e; i += blockDim.x) {
    const int key = het_cell_key<D, W>(x, i, h, n, lo, S);
    const long long pos = (long long)atomicAdd(&cur[key], 1ull);
#pragma unroll
    for (int k = 0; k < D; ++k) xs[(int64_t)k * N + pos] = __ldg(x + i * D + k);
    const double sn = __ldg(sd + i);
    is2[pos] = 1.0 / (sn * sn);
  }
}

__device__ __forceinline__ int het_wrap(int i, int n) {
  i %= n;
  return i < 0 ? i + n : i;
}

#ifndef EFGP_HET_GSM
#define EFGP_HET_GSM 1  // the warp's grid window in shared memory (broadcast reads) instead of registers
#endif
#ifndef EFGP_HET_PF
#define EFGP_HET_PF 1  // prefetch distance in points per lane (1: +17 %; 2-4 cost occupancy)
#endif
#ifndef EFGP_HET_THREADS
#define EFGP_HET_THREADS 128
#endif
// resident CTAs per SM the kernel is compiled for: 4 x 128 threads (<= 128 registers) for the 2D
// W <= 5 windows (+21 % over the unconstrained 154 registers on c5), else no constraint
template <int D, int W>
#ifndef EFGP_HET_MINB2
#define EFGP_HET_MINB2 4
#endif
constexpr int het_min_blocks() { return (D == 2 && W <= 5) ? EFGP_HET_MINB2 : 1; }
constexpr int kHetThreads = EFGP_HET_THREADS;

template <int D, int W>
__device__ __forceinline__ void het_point(double x0, double x1, double is, double h, int n, const EsPoly &P,
                                          const double *__restrict__ gw, double *__restrict__ acc) {
  double w0[W], w1[W];
  es_weights<W>(__dmul_rn(__dmul_rn(h, x0), (double)n), P, w0);
  if constexpr (D == 2) es_weights<W>(__dmul_rn(__dmul_rn(h, x1), (double)n), P, w1);
  double u = 0.0;
  if constexpr (D == 1) {
#pragma unroll
    for (int a = 0; a < W; ++a) u = fma(gw[a], w0[a], u);
    const double v = u * is;
#pragma unroll
    for (int a = 0; a < W; ++a) acc[a] = fma(v, w0[a], acc[a]);
  } else {
#pragma unroll
    for (int a = 0; a < W; ++a) {
      double ra = 0.0;
#pragma unroll
      for (int b = 0; b < W; ++b) ra = fma(gw[a * W + b], w1[b], ra);
      u = fma(ra, w0[a], u);
    }
    const double v = u * is;
#pragma unroll
    for (int a = 0; a < W; ++a) {
      const double va = v * w0[a];
#pragma unroll
      for (int b = 0; b < W; ++b) acc[a * W + b] = fma(va, w1[b], acc[a * W + b]);
    }
  }
}

template <int D, int W>
__global__ void __launch_bounds__(kHetThreads, het_min_blocks<D, W>()) k_het_apply_sorted(const HetItem *__restrict__ items, int64_t nitems,
                                                                  const double *__restrict__ xs,
                                                                  const double *__restrict__ is2, int64_t N,
                                                                  const double *__restrict__ g,
                                                                  double *__restrict__ out, double h, int n, int lo,
                                                                  int S, EsPoly P) {
  constexpr int WD = D == 1 ? W : W * W;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
#if EFGP_HET_GSM
  __shared__ double gsh[kHetThreads / 32][WD];
  double *gw = gsh[threadIdx.x >> 5];
#else
  double gw[WD];
#endif
  for (int64_t it = warp; it < nitems; it += nwarps) {
    const HetItem item = items[it];
    int c0, c1 = 0;
    if constexpr (D == 1) {
      c0 = item.cell + lo;
    } else {
      c0 = item.cell / S + lo;
      c1 = item.cell % S + lo;
    }
    double acc[WD];
#if EFGP_HET_GSM
    __syncwarp();
    for (int q = lane; q < WD; q += 32) {
      const int a = D == 1 ? q : q / W, b = D == 1 ? 0 : q % W;
      const int64_t gi = D == 1 ? het_wrap(c0 + a, n) : (int64_t)het_wrap(c0 + a, n) * n + het_wrap(c1 + b, n);
      gw[q] = __ldg(g + gi);
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < WD; ++q) acc[q] = 0.0;
#else
#pragma unroll
    for (int q = 0; q < WD; ++q) {
      const int a = D == 1 ? q : q / W, b = D == 1 ? 0 : q % W;
      const int64_t gi = D == 1 ? het_wrap(c0 + a, n) : (int64_t)het_wrap(c0 + a, n) * n + het_wrap(c1 + b, n);
      gw[q] = __ldg(g + gi);
      acc[q] = 0.0;
    }
#endif
    // the loads of the point PF positions ahead are in flight while this one is computed
    // (long-scoreboard stalls dominated without it)
    constexpr int PF = EFGP_HET_PF;
    double px0[PF], px1[PF], pis[PF];
    long long r = item.begin + lane;
#pragma unroll
    for (int k = 0; k < PF; ++k) {
      const long long rk = r + 32 * k;
      const bool ok = rk < item.end;
      px0[k] = ok ? __ldg(xs + rk) : 0.0;
      px1[k] = (D == 2 && ok) ? __ldg(xs + N + rk) : 0.0;
      pis[k] = ok ? __ldg(is2 + rk) : 0.0;
    }
    for (; r < item.end; r += 32) {
      const double x0 = px0[0], x1 = px1[0], is = pis[0];
#pragma unroll
      for (int k = 0; k + 1 < PF; ++k) {
        px0[k] = px0[k + 1];
        px1[k] = px1[k + 1];
        pis[k] = pis[k + 1];
      }
      const long long rn = r + 32 * PF;
      const bool ok = rn < item.end;
      px0[PF - 1] = ok ? __ldg(xs + rn) : 0.0;
      px1[PF - 1] = (D == 2 && ok) ? __ldg(xs + N + rn) : 0.0;
      pis[PF - 1] = ok ? __ldg(is2 + rn) : 0.0;
      het_point<D, W>(x0, x1, is, h, n, P, gw, acc);
    }
#pragma unroll
    for (int q = 0; q < WD; ++q) {
      double v = acc[q];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      acc[q] = v;
    }
#pragma unroll
    for (int q = 0; q < WD; ++q) {
      if (lane == (q & 31) && acc[q] != 0.0) {
        const int a = D == 1 ? q : q / W, b = D == 1 ? 0 : q % W;
        const int64_t gi = D == 1 ? het_wrap(c0 + a, n) : (int64_t)het_wrap(c0 + a, n) * n + het_wrap(c1 + b, n);
        atomicAdd(out + gi, acc[q]);
      }
    }
  }
}

namespace {

struct HetCtx {
  const double *x, *sd;
  double *w;
  int64_t N;
  int64_t n;           // fine grid of both transforms (n_rhs)
  const double *psi;   // its deconvolution table
  cufftHandle plan;    // its C2R plan
  double2 *box;
  double *grid;
};

unsigned grid_for(int64_t n, int sms) {
  int64_t b = (n + 255) / 256;
  const int64_t cap = (int64_t)sms * 8;
  return (unsigned)(b > cap ? cap : (b < 1 ? 1 : b));
}

// out = D . F^*(w) (+ p): spread the strengths w at x, R2C, deconvolve
efgp_status spread_to_modes(efgp_plan *pl, const double *x, const double *w, int64_t N, const double2 *p,
                            double2 *out, cudaStream_t s) {
  const Params &P = pl->P;
  EFGP_TRY(spread_begin(pl, s));
  EFGP_TRY(spread_points(pl, x, w, N, s));
  EFGP_CUFFT(cufftSetStream(pl->plan_g2, s));
  EFGP_CUFFT(cufftExecD2Z(pl->plan_g2, pl->g2, pl->G2h));
  const int64_t nr = P.n_rhs;
  const double *psir = (nr == P.n1) ? pl->psi1 : pl->psi2;
  const double sc = std::pow(2.0 * kPi / (double)nr, P.d);
  const unsigned g = grid_for(P.Mh, pl->num_sms);
  switch (P.d) {
    case 1: k_het_modes<1><<<g, 256, 0, s>>>(pl->G2h, nr, (int)P.m, psir, sc, pl->D_half, p, out, P.Mh); break;
    case 2: k_het_modes<2><<<g, 256, 0, s>>>(pl->G2h, nr, (int)P.m, psir, sc, pl->D_half, p, out, P.Mh); break;
    case 3: k_het_modes<3><<<g, 256, 0, s>>>(pl->G2h, nr, (int)P.m, psir, sc, pl->D_half, p, out, P.Mh); break;
  }
  EFGP_CUDA(cudaGetLastError());
  return EFGP_OK;
}

// A p = D F^*(S^-1 F(D p)) + p
efgp_status het_apply(efgp_plan *pl, const double2 *p, double2 *Ap, void *vctx) {
  const HetCtx *c = static_cast<const HetCtx *>(vctx);
  cudaStream_t s = pl->stream;
  EFGP_TRY(type2_grid_on(pl, p, c->n, c->psi, c->plan, c->box, c->grid, s));
  EFGP_TRY(interp_weighted(pl, c->grid, c->n, c->x, c->N, c->sd, c->w, s));
  return spread_to_modes(pl, c->x, c->w, c->N, p, Ap, s);
}


struct HetSorted {
  int lo = 0, S = 0, ncell = 0;
  double *xs = nullptr, *is2 = nullptr, *out = nullptr;
  HetItem *items = nullptr;
  int64_t nitems = 0;
  cufftHandle r2c = 0;
};

// d <= 2, register windows up to 8 x 8 (d = 2) or 16 (d = 1), scatter cursors in shared memory
bool het_sorted_geometry(const Params &P, HetSorted &H) {
  const char *e = getenv("EFGP_HETERO_SORTED");
  if (e && e[0] == '0') return false;
  if (P.d > 2 || (P.d == 2 && P.w > 8)) return false;
  H.lo = -(P.w / 2);  // ceil(-W/2)
  const int hi = (int)std::ceil(P.h * (double)P.n2 - 0.5 * P.w);
  H.S = hi - H.lo + 2;  // one spare row
  H.ncell = P.d == 1 ? H.S : H.S * H.S;
  return (size_t)H.ncell * 8 <= 200 * 1024;
}

template <int D, int W>
efgp_status het_sort_t(efgp_plan *pl, HetSorted &H, const double *x, const double *sd, int64_t N, cudaStream_t s) {
  const Params &P = pl->P;
  const int B = sort_ctas(pl->num_sms), T = 1024, n = (int)P.n2;
  unsigned *hist = nullptr;
  long long *tot = nullptr, *off = nullptr;
  EFGP_PALLOC(&hist, sizeof(unsigned) * B * H.ncell, s);
  EFGP_PALLOC(&tot, sizeof(long long) * H.ncell, s);
  EFGP_PALLOC(&off, sizeof(long long) * (H.ncell + 1), s);
  EFGP_PALLOC(&H.xs, sizeof(double) * N * D, s);
  EFGP_PALLOC(&H.is2, sizeof(double) * N, s);
  const size_t sm_count = sizeof(unsigned) * H.ncell, sm_scatter = sizeof(unsigned long long) * H.ncell;
  EFGP_CUDA(cudaFuncSetAttribute(k_het_count<D, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_count));
  EFGP_CUDA(cudaFuncSetAttribute(k_het_scatter<D, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_scatter));
  k_het_count<D, W><<<B, T, sm_count, s>>>(x, N, P.h, n, H.lo, H.S, H.ncell, hist);
  k_het_colscan<<<(H.ncell + 255) / 256, 256, 0, s>>>(hist, B, H.ncell, tot);
  k_het_offsets<<<1, 1024, 0, s>>>(tot, H.ncell, off);
  k_het_scatter<D, W><<<B, T, sm_scatter, s>>>(x, sd, N, P.h, n, H.lo, H.S, H.ncell, hist, off, H.xs, H.is2);
  EFGP_CUDA(cudaGetLastError());
  std::vector<long long> offh(H.ncell + 1);
  EFGP_CUDA(cudaMemcpyAsync(offh.data(), off, sizeof(long long) * (H.ncell + 1), cudaMemcpyDeviceToHost, s));
  EFGP_CUDA(cudaStreamSynchronize(s));
  cudaFreeAsync(hist, s);
  cudaFreeAsync(tot, s);
  cudaFreeAsync(off, s);
  if (offh[H.ncell] != N) {
    pl->err = "internal: hetero counting sort lost points";
    return EFGP_ERR_CUDA;
  }
  std::vector<HetItem> items;
  for (int c = 0; c < H.ncell; ++c)
    for (long long b = offh[c]; b < offh[c + 1]; b += kHetRun)
      items.push_back(HetItem{b, std::min<long long>(b + kHetRun, offh[c + 1]), c, 0});
  H.nitems = (int64_t)items.size();
  EFGP_PALLOC(&H.items, sizeof(HetItem) * std::max<size_t>(items.size(), 1), s);
  EFGP_CUDA(cudaMemcpyAsync(H.items, items.data(), sizeof(HetItem) * items.size(), cudaMemcpyHostToDevice, s));
  int64_t cells = 1;
  for (int k = 0; k < D; ++k) cells *= P.n2;
  EFGP_PALLOC(&H.out, sizeof(double) * cells, s);
  if (!pl->plan_het_r2c) {
    int dims[3] = {(int)P.n2, (int)P.n2, (int)P.n2};
    EFGP_CUFFT(cufftPlanMany(&pl->plan_het_r2c, D, dims, nullptr, 1, 0, nullptr, 1, 0, CUFFT_D2Z, 1));
  }
  H.r2c = pl->plan_het_r2c;
  EFGP_CUDA(cudaStreamSynchronize(s));  // items (host vector) uploaded before it goes out of scope
  return EFGP_OK;
}

void het_sorted_free(HetSorted &H, cudaStream_t s) {
  for (void *p : {(void *)H.xs, (void *)H.is2, (void *)H.out, (void *)H.items})
    if (p) cudaFreeAsync(p, s);
  H = HetSorted{};  // (the r2c plan belongs to the handle)
}

template <int D, int W>
efgp_status het_apply_sorted_t(efgp_plan *pl, const HetSorted &H, int64_t N, const double2 *p, double2 *Ap) {
  const Params &P = pl->P;
  cudaStream_t s = pl->stream;
  const int n = (int)P.n2;
  EFGP_TRY(type2_grid_on(pl, p, P.n2, pl->psi2, pl->plan_t2, pl->T2box, pl->t2grid, s));
  int64_t cells = 1, box = P.n2 / 2 + 1;
  for (int k = 0; k < D; ++k) cells *= P.n2;
  for (int k = 0; k < D - 1; ++k) box *= P.n2;
  EFGP_CUDA(cudaMemsetAsync(H.out, 0, sizeof(double) * cells, s));
  int per_sm = 1;
  EFGP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_het_apply_sorted<D, W>, kHetThreads, 0));
  int64_t blocks = std::min<int64_t>((int64_t)pl->num_sms * std::max(per_sm, 1),
                                     (H.nitems * 32 + kHetThreads - 1) / kHetThreads);
  if (blocks < 1) blocks = 1;
  if (H.nitems > 0)
    k_het_apply_sorted<D, W><<<(unsigned)blocks, kHetThreads, 0, s>>>(H.items, H.nitems, H.xs, H.is2, N, pl->t2grid, H.out,
                                                               P.h, n, H.lo, H.S, P.poly);
  EFGP_CUDA(cudaGetLastError());
  EFGP_CUFFT(cufftSetStream(H.r2c, s));
  EFGP_CUFFT(cufftExecD2Z(H.r2c, H.out, pl->T2box));  // the C2R input box is free again
  const double sc = std::pow(2.0 * kPi / (double)n, D);
  k_het_modes<D><<<grid_for(P.Mh, pl->num_sms), 256, 0, s>>>(pl->T2box, P.n2, (int)P.m, pl->psi2, sc, pl->D_half, p,
                                                             Ap, P.Mh);
  EFGP_CUDA(cudaGetLastError());
  return EFGP_OK;
}

#define EFGP_HET_W1(M) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10) M(11) M(12) M(13) M(14) M(15) M(16)
#define EFGP_HET_W2(M) M(2) M(3) M(4) M(5) M(6) M(7) M(8)

efgp_status het_sort(efgp_plan *pl, HetSorted &H, const double *x, const double *sd, int64_t N, cudaStream_t s) {
  const int W = pl->P.w;
  if (pl->P.d == 1) {
    switch (W) {
#define C1(WW) case WW: return het_sort_t<1, WW>(pl, H, x, sd, N, s);
      EFGP_HET_W1(C1)
#undef C1
    }
  } else {
    switch (W) {
#define C2(WW) case WW: return het_sort_t<2, WW>(pl, H, x, sd, N, s);
      EFGP_HET_W2(C2)
#undef C2
    }
  }
  pl->err = "internal: no sorted hetero kernel for this width";
  return EFGP_ERR_INVALID;
}

struct HetSortedCtx {
  HetSorted *H;
  int64_t N;
};

efgp_status het_apply_sorted(efgp_plan *pl, const double2 *p, double2 *Ap, void *vctx) {
  const HetSortedCtx *c = static_cast<const HetSortedCtx *>(vctx);
  const int W = pl->P.w;
  if (pl->P.d == 1) {
    switch (W) {
#define C1(WW) case WW: return het_apply_sorted_t<1, WW>(pl, *c->H, c->N, p, Ap);
      EFGP_HET_W1(C1)
#undef C1
    }
  } else {
    switch (W) {
#define C2(WW) case WW: return het_apply_sorted_t<2, WW>(pl, *c->H, c->N, p, Ap);
      EFGP_HET_W2(C2)
#undef C2
    }
  }
  return EFGP_ERR_INVALID;
}

float elapsed_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
    cudaGetLastError();
    return 0.f;
  }
  return ms;
}

}  // namespace

efgp_status fit_hetero_device(efgp_plan *pl, const double *x, const double *y, const double *sd, int64_t N) {
  const Params &P = pl->P;
  cudaStream_t s = pl->stream;
  pl->fitted = false;
  pl->op_valid = false;  // no Toeplitz operator: predict_var is refused after a heteroskedastic fit
  pl->t2_valid = false;  // the type-2 grid is rebuilt from beta by the next predict
  // G11b route: the weighted Toeplitz system, where the y spreading grid is the v grid (n_rhs = n1)
  const bool tz = P.hetero_method != EFGP_HETERO_NUFFT && P.n_rhs == P.n1;
  // SORTED one-pass route: the spreading kernel reads the raw (y_n, sigma_n), validates sigma_n, takes
  // min sigma_n and forms the strengths 1/sigma_n^2, y_n/sigma_n^2 in its balanced pass 2 — no prep
  // pass (32 B/point of HBM traffic) and no N-sized temporaries.  Every other route preps first.
  const bool raw = tz && P.spread_method == EFGP_SPREAD_SORTED;
  double *w = nullptr, *iv = nullptr;
  unsigned long long *minbits = reinterpret_cast<unsigned long long *>(pl->scal + 24);
  int flags[4] = {0, 0, 0, 0};
  unsigned long long mb = 0;
  EFGP_CUDA(cudaEventRecord(pl->ev[0], s));
  EFGP_CUDA(cudaMemsetAsync(minbits, 0xff, sizeof(unsigned long long), s));
  auto prep = [&]() -> efgp_status {  // w = y / sigma^2 (and iv = 1 / sigma^2), sigma_n checked, min sigma_n
    EFGP_PALLOC(&w, sizeof(double) * N, s);
    if (tz) EFGP_PALLOC(&iv, sizeof(double) * N, s);
    EFGP_CUDA(cudaMemsetAsync(minbits, 0xff, sizeof(unsigned long long), s));
    EFGP_CUDA(cudaMemsetAsync(pl->dflags + 2, 0, sizeof(int), s));
    k_het_prep<<<grid_for(N, pl->num_sms), 256, 0, s>>>(y, sd, N, w, minbits, pl->dflags, iv);
    EFGP_CUDA(cudaGetLastError());
    EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned, pl->dflags, sizeof(int) * 4, cudaMemcpyDeviceToHost, s));
    EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned + 8, minbits, sizeof(mb), cudaMemcpyDeviceToHost, s));
    EFGP_CUDA(cudaStreamSynchronize(s));
    std::memcpy(flags, pl->h_pinned, sizeof(flags));
    std::memcpy(&mb, pl->h_pinned + 8, sizeof(mb));
    if (flags[2]) {
      pl->err = "fit_hetero: every noise standard deviation must be finite and > 0";
      return EFGP_ERR_INVALID;
    }
    return EFGP_OK;
  };
  auto free_tmp = [&]() {
    if (w) cudaFreeAsync(w, s);
    if (iv) cudaFreeAsync(iv, s);
    w = iv = nullptr;
  };
  efgp_status st = raw ? EFGP_OK : prep();
  if (st == EFGP_OK && tz) {
    // v^w (J_2m) from strengths 1/sigma_n^2 and F^*(y/sigma^2) (J_m), both spread as the "y" strength
    // onto the v grid, then the homoskedastic Toeplitz machinery with sigma^2 -> 1 (reading G11b)
    double2 *vh = reinterpret_cast<double2 *>(pl->modes_sum), *fyh = vh + P.Kvh;
    bool one_pass = false;
    if (raw) {
      st = spread_begin(pl, s);  // clears dflags[0..3]
      if (st == EFGP_OK) st = spread_points(pl, x, y, N, s, sd, minbits);
      if (st == EFGP_OK) {
        one_pass = true;
        st = type1_modes(pl, pl->modes_sum, s);
        EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned, pl->dflags, sizeof(int) * 4, cudaMemcpyDeviceToHost, s));
        EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned + 8, minbits, sizeof(mb), cudaMemcpyDeviceToHost, s));
        EFGP_CUDA(cudaStreamSynchronize(s));
        std::memcpy(flags, pl->h_pinned, sizeof(flags));
        std::memcpy(&mb, pl->h_pinned + 8, sizeof(mb));
        if (st == EFGP_OK && flags[2]) {
          pl->err = "fit_hetero: every noise standard deviation must be finite and > 0";
          st = EFGP_ERR_INVALID;
        } else if (st == EFGP_OK && flags[0]) {
          pl->err = "fit_hetero: a coordinate is outside [0,1] or non-finite, or an observation is non-finite";
          st = EFGP_ERR_INVALID;
        }
      } else if (st == EFGP_ERR_RESOURCE) {
        // (unaligned inputs, no co-residency, 2^32 points and more in one call): prep, then the
        // two-pass route below
        pl->err.clear();
        st = prep();
      }
    } else if (P.spread_method == EFGP_SPREAD_CELLSORT) {
      // CELLSORT spreads both weighted strengths in one pass:
      // g1 = sum (1/sigma^2) phi (v^w), g2 = sum (y/sigma^2) phi, then the standard K2 for both
      st = spread_begin(pl, s);
      if (st == EFGP_OK) st = spread_points(pl, x, w, N, s, iv);
      if (st == EFGP_OK) {
        one_pass = true;
        st = type1_modes(pl, pl->modes_sum, s);
        EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned, pl->dflags, sizeof(int) * 4, cudaMemcpyDeviceToHost, s));
        EFGP_CUDA(cudaStreamSynchronize(s));
        std::memcpy(flags, pl->h_pinned, sizeof(flags));
        if (st == EFGP_OK && flags[0]) {
          pl->err = "fit_hetero: a coordinate is outside [0,1] or non-finite, or an observation is non-finite";
          st = EFGP_ERR_INVALID;
        }
      } else if (st == EFGP_ERR_RESOURCE) {
        st = EFGP_OK;  // (2^32 points and more in one call): the two-pass route below
        pl->err.clear();
      }
    }
    for (int pass = 0; pass < 2 && st == EFGP_OK && !one_pass; ++pass) {
      st = spread_begin(pl, s);
      if (st == EFGP_OK) st = spread_points(pl, x, pass == 0 ? iv : w, N, s);
      if (st != EFGP_OK) break;
      EFGP_CUFFT(cufftSetStream(pl->plan_g2, s));
      EFGP_CUFFT(cufftExecD2Z(pl->plan_g2, pl->g2, pl->G2h));
      if (pass == 0) st = type1_half(pl, pl->G2h, P.n1, (int)(2 * P.m), pl->psi1, vh, s);
      else st = type1_half(pl, pl->G2h, P.n1, (int)P.m, pl->psi1, fyh, s);
      EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned, pl->dflags, sizeof(int) * 4, cudaMemcpyDeviceToHost, s));
      EFGP_CUDA(cudaStreamSynchronize(s));
      std::memcpy(flags, pl->h_pinned, sizeof(flags));
      if (st == EFGP_OK && flags[0]) {
        pl->err = "fit_hetero: a coordinate is outside [0,1] or non-finite, or an observation is non-finite";
        st = EFGP_ERR_INVALID;
      }
    }
    EFGP_CUDA(cudaEventRecord(pl->ev[1], s));
    double smin = 0;
    std::memcpy(&smin, &mb, sizeof(smin));
    int64_t Ntot = N;
    if (pl->comm) {  // multi-GPU: v^w and F^*(y/sigma^2) are sums over the points
      // every rank takes part even after a local failure (failure flag reduced with the counts), so
      // no rank is left waiting in the collective; all ranks then return an error together
      const std::string local_err = pl->err;
      int fail = st != EFGP_OK;
      efgp_status cs = comm_sum(pl, pl->modes_sum, (size_t)2 * (P.Kvh + P.Mh));
      if (cs == EFGP_OK) cs = comm_count_min(pl, &Ntot, &smin, &fail);
      if (st != EFGP_OK) {
        pl->err = local_err;
      } else if (cs != EFGP_OK) {
        st = cs;
      } else if (fail) {
        pl->err = "fit_hetero: the spreading failed on another rank (invalid input there); no rank solved";
        st = EFGP_ERR_INVALID;
      }
    }
    if (st == EFGP_OK) {
      pl->sigma2_sys = 1.0;
      pl->cap_sigma = smin;
      st = toeplitz_setup(pl, pl->modes_sum, s);
      EFGP_CUDA(cudaEventRecord(pl->ev[2], s));
      if (st == EFGP_OK) {
        pl->op_valid = true;
        pl->pc_used = P.precond;
        if (P.precond) {
          st = precond_setup(pl, pl->modes_sum);
          if (st == EFGP_OK) st = pcg_solve(pl, Ntot);
        } else {
          st = cg_solve(pl, Ntot);
        }
      }
      pl->het_path = 2;
      EFGP_CUDA(cudaEventRecord(pl->ev[4], s));
      EFGP_CUDA(cudaEventSynchronize(pl->ev[4]));
      pl->t_spread = elapsed_ms(pl->ev[0], pl->ev[1]);
      pl->t_modes = elapsed_ms(pl->ev[1], pl->ev[2]);
      pl->t_solve = elapsed_ms(pl->ev[2], pl->ev[4]);
      if (st == EFGP_OK || st == EFGP_ERR_NOCONVERGE) {
        pl->fitted = true;
        pl->N_last = Ntot;
      }
      if (st == EFGP_ERR_NOCONVERGE) pl->err = "CG reached max_iter before the relative residual reached cg_tol";
    }
    free_tmp();
    EFGP_CUDA(cudaStreamSynchronize(s));
    return st;
  }
  if (st == EFGP_OK && pl->comm && pl->comm_size > 1) {
    pl->err = "fit_hetero: the NUFFT-pair solver is single-process (use hetero_method TOEPLITZ with a communicator)";
    st = EFGP_ERR_INVALID;
  }
  // b = D F^*(y / sigma^2); spread_begin clears the input flags, spread_points raises dflags[0]
  if (st == EFGP_OK) st = spread_to_modes(pl, x, w, N, nullptr, pl->b, s);
  if (st == EFGP_OK) {
    EFGP_CUDA(cudaEventRecord(pl->ev[1], s));
    EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned, pl->dflags, sizeof(int) * 4, cudaMemcpyDeviceToHost, s));
    EFGP_CUDA(cudaStreamSynchronize(s));
    std::memcpy(flags, pl->h_pinned, sizeof(flags));
    if (flags[0]) {
      pl->err = "fit_hetero: a coordinate is outside [0,1] or non-finite, or an observation is non-finite";
      st = EFGP_ERR_INVALID;
    }
  }
  if (st == EFGP_OK) {
    double smin = 0;
    std::memcpy(&smin, &mb, sizeof(smin));
    int64_t max_iter = P.max_iter_opt;
    if (max_iter <= 0) {  // P:1766 with sigma = min sigma_n (reading G11)
      max_iter = (int64_t)std::ceil(std::log(1.0 / P.cg_tol) * std::sqrt((double)N) / (2.0 * smin));
      if (max_iter < 10) max_iter = 10;
    }
    HetSorted H;
    if (het_sorted_geometry(P, H)) {
      st = het_sort(pl, H, x, sd, N, s);
      EFGP_CUDA(cudaEventRecord(pl->ev[2], s));
      HetSortedCtx sctx{&H, N};
      if (st == EFGP_OK) st = cg_solve_op(pl, max_iter, het_apply_sorted, &sctx);
      pl->het_path = 1;
      pl->pc_used = 0;
    } else {
      EFGP_CUDA(cudaEventRecord(pl->ev[2], s));
      // Both NUFFTs on the same fine grid n_rhs with the same kernel and deconvolution: the type-2 is
      // then the exact adjoint of the type-1, so the applied operator is exactly Hermitian (CG's
      // recurrences assume it; with the v grid n1 for the spread and n2 for the interpolation the
      // mismatch ~nufft_tol slowed parity-mode CG by ~30 %).
      HetCtx ctx{x, sd, w, N, P.n_rhs, nullptr, 0, nullptr, nullptr};
      if (P.n_rhs == P.n2) {
        ctx.psi = pl->psi2;
        ctx.plan = pl->plan_t2;
        ctx.box = pl->T2box;
        ctx.grid = pl->t2grid;
      } else {
        if (!pl->het_grid) {
          int64_t box = P.n_rhs / 2 + 1, cells = P.n_rhs;
          for (int k = 0; k < P.d - 1; ++k) {
            box *= P.n_rhs;
            cells *= P.n_rhs;
          }
          EFGP_CUDA(cudaMalloc((void **)&pl->het_box, sizeof(double2) * box));
          EFGP_CUDA(cudaMalloc((void **)&pl->het_grid, sizeof(double) * cells));
          int dims[3] = {(int)P.n_rhs, (int)P.n_rhs, (int)P.n_rhs};
          EFGP_CUFFT(cufftPlanMany(&pl->plan_het, P.d, dims, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2D, 1));
        }
        ctx.psi = pl->psi1;  // n_rhs == n1: psi1 covers k <= 2m
        ctx.plan = pl->plan_het;
        ctx.box = pl->het_box;
        ctx.grid = pl->het_grid;
      }
      st = cg_solve_op(pl, max_iter, het_apply, &ctx);
      pl->het_path = 0;
      pl->pc_used = 0;
    }
    het_sorted_free(H, s);
    EFGP_CUDA(cudaEventRecord(pl->ev[4], s));
    EFGP_CUDA(cudaEventSynchronize(pl->ev[4]));
    pl->t_spread = elapsed_ms(pl->ev[0], pl->ev[1]);  // right-hand side (prep + type-1)
    pl->t_modes = elapsed_ms(pl->ev[1], pl->ev[2]);   // sorted path: the one-time counting sort
    pl->t_solve = elapsed_ms(pl->ev[2], pl->ev[4]);
    if (st == EFGP_OK || st == EFGP_ERR_NOCONVERGE) {
      pl->fitted = true;
      pl->N_last = N;
    }
    if (st == EFGP_ERR_NOCONVERGE) pl->err = "CG reached max_iter before the relative residual reached cg_tol";
  }
  free_tmp();
  EFGP_CUDA(cudaStreamSynchronize(s));
  return st;
}

}  // namespace efgp
