// K9: type-2 interpolation mu(x*) = sum_{cells l near theta*} b_l prod_k phi((l_k - t_k) 2/W),
// t = h x* n2, b = C2R(c') the real type-2 fine grid (Alg a1 steps 5-6; eq "muws"
// P:557).  One thread per target.  SMEM variant: each CTA stages the occupied part of the grid
// (cells reachable from x* in [0,1]^d) in shared memory once, then gathers from it; GLOBAL
// variant gathers from L2.  Targets outside [0,1]^d or non-finite give mu = NaN and raise
// dflags[1].
#include <algorithm>
#include <cmath>
#include <cstring>

#include "efgp_internal.cuh"

namespace efgp {

#define EFGP_W_CASES2(MACRO) \
  MACRO(2) MACRO(3) MACRO(4) MACRO(5) MACRO(6) MACRO(7) MACRO(8) MACRO(9) MACRO(10) MACRO(11) MACRO(12) MACRO(13) MACRO(14) MACRO(15) MACRO(16)

struct Occ2 {
  int lo, A;
};
static inline Occ2 occupied2(double h, int n, int W) {
  const int lo = -(W / 2);
  const int hi0 = (int)std::ceil(h * n - 0.5 * W);
  return Occ2{lo, hi0 + W - 1 - lo + 1};
}

__device__ __forceinline__ int wrapn(int i, int n) {
  i %= n;
  return i < 0 ? i + n : i;
}

// threads per CTA the kernel is compiled for: 1024 where the weights fit in 64 registers
template <int D, int W>
constexpr int interp_max_threads() { return (D <= 2 && W <= 8) ? 1024 : 256; }

template <int D, int W, bool SMEM>
__global__ void __launch_bounds__(interp_max_threads<D, W>()) k_interp(const double *__restrict__ xt, int64_t q,
                                                const double *__restrict__ grid, int n, double h, EsPoly P,
                                                int lo, int A, const double *__restrict__ sd,
                                                double *__restrict__ mu, int *__restrict__ err) {
  extern __shared__ double sgrid[];
  if constexpr (SMEM) {
    int64_t cells = A;
    for (int k = 1; k < D; ++k) cells *= A;
    for (int64_t c = threadIdx.x; c < cells; c += blockDim.x) {
      int64_t rem = c, gi = 0;
      int idx[D];
#pragma unroll
      for (int k = D - 1; k >= 0; --k) {
        idx[k] = (int)(rem % A);
        rem /= A;
      }
#pragma unroll
      for (int k = 0; k < D; ++k) gi = gi * n + wrapn(idx[k] + lo, n);
      sgrid[c] = __ldg(grid + gi);
    }
    __syncthreads();
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < q; i += (int64_t)gridDim.x * blockDim.x) {
    double xc[D];
    bool ok = true;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      xc[k] = __ldg(xt + i * D + k);
      ok = ok && xc[k] >= 0.0 && xc[k] <= 1.0;
    }
    if (!ok) {
      mu[i] = __longlong_as_double(0x7ff8000000000000LL);
      atomicOr(err + 1, 1);
      continue;
    }
    int base[D];
    double wt[D][W];
#pragma unroll
    for (int k = 0; k < D; ++k) base[k] = es_weights<W>(h * xc[k] * (double)n, P, wt[k]);
    double acc = 0.0;
    if constexpr (D == 1) {
#pragma unroll
      for (int a = 0; a < W; ++a) {
        const double g = SMEM ? sgrid[base[0] + a - lo] : __ldg(grid + wrapn(base[0] + a, n));
        acc = fma(g, wt[0][a], acc);
      }
    } else if constexpr (D == 2) {
#pragma unroll
      for (int a = 0; a < W; ++a) {
        double ra = 0.0;
        if (SMEM) {
          const double *row = sgrid + (int64_t)(base[0] + a - lo) * A + (base[1] - lo);
#pragma unroll
          for (int b = 0; b < W; ++b) ra = fma(row[b], wt[1][b], ra);
        } else {
          const double *row = grid + (int64_t)wrapn(base[0] + a, n) * n;
#pragma unroll
          for (int b = 0; b < W; ++b) ra = fma(__ldg(row + wrapn(base[1] + b, n)), wt[1][b], ra);
        }
        acc = fma(ra, wt[0][a], acc);
      }
    } else {
#pragma unroll 1
      for (int a = 0; a < W; ++a) {
        double ra = 0.0;
#pragma unroll
        for (int b = 0; b < W; ++b) {
          double rb = 0.0;
          if (SMEM) {
            const double *row = sgrid + ((int64_t)(base[0] + a - lo) * A + (base[1] + b - lo)) * A + (base[2] - lo);
#pragma unroll
            for (int e = 0; e < W; ++e) rb = fma(row[e], wt[2][e], rb);
          } else {
            const double *row = grid + ((int64_t)wrapn(base[0] + a, n) * n + wrapn(base[1] + b, n)) * n;
#pragma unroll
            for (int e = 0; e < W; ++e) rb = fma(__ldg(row + wrapn(base[2] + e, n)), wt[2][e], rb);
          }
          ra = fma(rb, wt[1][b], ra);
        }
        acc = fma(ra, wt[0][a], acc);
      }
    }
    if (sd) {  // NEXT-3: w_n = (Phi p)_n / sigma_n^2 (reading G11)
      const double sn = __ldg(sd + i);
      acc /= sn * sn;
    }
    mu[i] = acc;
  }
}

// 2D, grid staged in shared memory, bank-aware order (the K9 variant for many random targets).
// Gathering a W x W window for 32 random targets is bound by shared-memory bank conflicts: a warp's
// LDS.64 of 32 random cells costs ~6.2 wavefronts instead of 2 (r01 ncu).  The bank of every cell
// of a target's window is (bank of its first cell + a A + b) mod 16 (8-byte banks of a half-warp
// phase), so if the 16 targets of each half-warp have pairwise different first-cell banks, all
// W^2 gathers are conflict-free.  Each CTA therefore takes batches of kIB targets, classifies them by
// first-cell bank (shared counters), and hands target rank k of bank class b to thread 16 k + b;
// the few targets beyond a class's quota fill the slots of the classes that ran short.  Same
// arithmetic per target as k_interp (bitwise-identical results), only the thread assignment changes.
#ifndef EFGP_KIB
#define EFGP_KIB 512
#endif
constexpr int kIB = EFGP_KIB;  // targets per batch = threads per CTA (1024 / kIB CTAs per SM overlap their barriers)

template <int W>
__global__ void __launch_bounds__(kIB, 1024 / kIB) k_interp2_banked(const double *__restrict__ xt, int64_t q,
                                                                    const double *__restrict__ grid, int n, double h,
                                                                    EsPoly P, int lo, int A, const double *__restrict__ sd,
                                                                    double *__restrict__ mu, int *__restrict__ err) {
  extern __shared__ __align__(16) double sgrid[];
  __shared__ double2 s_s[kIB];         // reduced coordinates (s0, s1) of the batch's targets (by batch
                                       // index): one 16-byte access in the permuted read
  __shared__ int s_cell[kIB];          // first-cell offset r A + c in the staged grid (-1: invalid / none)
  __shared__ short s_tbl[kIB];         // thread slot -> batch index
  __shared__ short s_ovf[kIB];         // targets beyond their class quota
  __shared__ int s_cnt[16], s_novf, s_take;
  const int tid = threadIdx.x;
  for (int c = tid; c < A * A; c += kIB) {
    const int r = c / A, cc = c % A;
    sgrid[c] = __ldg(grid + (int64_t)wrapn(r + lo, n) * n + wrapn(cc + lo, n));
  }
  const int64_t nb = (q + kIB - 1) / kIB;
  const double2 *x2 = reinterpret_cast<const double2 *>(xt);
  // targets are loaded one batch ahead (their HBM latency overlaps a batch of work)
  auto ld = [&](int64_t b) -> double2 {
    const int64_t ii = b * kIB + tid;
    return (b < nb && ii < q) ? __ldg(x2 + ii) : make_double2(0.0, 0.0);
  };
  double2 xn = ld(blockIdx.x);
  for (int64_t bt = blockIdx.x; bt < nb; bt += gridDim.x) {
    const double2 xc = xn;
    const int64_t i = bt * kIB + tid;
    xn = ld(bt + gridDim.x);
    __syncthreads();  // the previous batch is done with every table (and the grid is staged)
    if (tid < 16) s_cnt[tid] = 0;
    if (tid == 0) s_novf = s_take = 0;
    s_tbl[tid] = -1;
    __syncthreads();
    int cell = -1;
    if (i < q) {
      if (xc.x >= 0.0 && xc.x <= 1.0 && xc.y >= 0.0 && xc.y <= 1.0) {
        double s0, s1;
        const int b0 = es_reduce<W>(h * xc.x * (double)n, s0);
        const int b1 = es_reduce<W>(h * xc.y * (double)n, s1);
        s_s[tid] = make_double2(s0, s1);
        cell = (b0 - lo) * A + (b1 - lo);
      } else {
        mu[i] = __longlong_as_double(0x7ff8000000000000LL);
        atomicOr(err + 1, 1);
      }
    }
    s_cell[tid] = cell;
    if (cell >= 0) {
      const int b = cell & 15;
      const int k = atomicAdd(&s_cnt[b], 1);
      if (k < kIB / 16) s_tbl[16 * k + b] = (short)tid;
      else s_ovf[atomicAdd(&s_novf, 1)] = (short)tid;
    }
    __syncthreads();
    int j = s_tbl[tid];
    if (j < 0) {  // an empty slot takes an over-quota target, if any is left
      const int novf = s_novf;
      if (novf > 0) {
        const int t = atomicAdd(&s_take, 1);
        if (t < novf) j = s_ovf[t];
      }
    }
    if (j >= 0) {
      EFGP_DCHECK(j < kIB && s_cell[j] >= 0 && s_cell[j] + (W - 1) * (A + 1) < A * A);
      double wt[2][W];
      const double2 sj = s_s[j];
      es_weights_s<W>(sj.x, P, wt[0]);
      es_weights_s<W>(sj.y, P, wt[1]);
      const double *win = sgrid + s_cell[j];
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < W; ++a) {
        double ra = 0.0;
#pragma unroll
        for (int b = 0; b < W; ++b) ra = fma(win[a * A + b], wt[1][b], ra);
        acc = fma(ra, wt[0][a], acc);
      }
      const int64_t ij = bt * kIB + j;
      if (sd) {  // NEXT-3: w_n = (Phi p)_n / sigma_n^2 (reading G11)
        const double sn = __ldg(sd + ij);
        acc /= sn * sn;
      }
      mu[ij] = acc;
    }
  }
}

// 2D, C shifted copies of the staged grid, no bank-class overflow (r02b successor of k_interp2_banked).
// The banked kernel gives each of the 16 lanes of a half-warp one first-cell bank class; a class with
// more than its quota of a batch's targets spills them into other classes' slots, where every one of
// their W^2 gathers conflicts (~7 % of targets, ~1.2 extra wavefronts per target at c5, r02 ncu).
// Here the grid is staged C times, copy j at a shared offset = j R (mod 16) doubles (R = 16 / C), so a
// target whose first cell is in bank class b can be read through bank class b + j R: only its residue
// b mod R is fixed.  Target rank k of residue c goes to half-warp k / C, lane c + (k mod C) R, read from
// the copy that maps its class onto that lane — the per-residue quota (C HW) is far above the batch's
// mean count, so practically no target spills, and half-warps only run short at the tail.  The per
// batch tables are triple-buffered so one CTA barrier per batch suffices: a batch's classification
// (writes set it % 3, resets set (it + 1) % 3) overlaps the previous batch's gathers (reads set
// (it - 1) % 3).  Same arithmetic per target as k_interp (bitwise-identical results).
template <int W, int C, int T, int NT>
__global__ void __launch_bounds__(NT, (NT <= 512 ? 1024 / NT : 1)) k_interp2_copies(const double *__restrict__ xt, int64_t q,
                                                                  const double *__restrict__ grid, int n, double h,
                                                                  EsPoly P, int lo, int A, int Sg,
                                                                  const double *__restrict__ sd,
                                                                  double *__restrict__ mu, int *__restrict__ err) {
  constexpr int R = 16 / C;   // residue classes
  constexpr int QC = (NT / 16) * C;  // slots per residue class and batch
  static_assert(16 % C == 0 && T <= NT && T <= 32767, "k_interp2_copies shape");
  // dynamic shared memory: the C grid copies (copy j at j Sg doubles, Sg = R mod 16, Sg even), then
  // the triple-buffered tables
  extern __shared__ __align__(16) double sgrid[];
  auto s_s = reinterpret_cast<double2 (*)[T]>(sgrid + (size_t)C * Sg);  // reduced coordinates by batch index
  auto s_cell = reinterpret_cast<int (*)[T]>(s_s + 3);                   // first-cell offset in a copy
  auto s_tbl = reinterpret_cast<short (*)[NT]>(s_cell + 3);              // slot -> batch index (-1: empty)
  auto s_ovf = reinterpret_cast<short (*)[T]>(s_tbl + 3);                // targets beyond their residue's quota
  __shared__ int s_cnt[3][R], s_novf[3], s_take[3];
  const int tid = threadIdx.x;
  for (int c = tid; c < A * A; c += NT) {
    const int r = c / A, cc = c % A;
    const double g = __ldg(grid + (int64_t)wrapn(r + lo, n) * n + wrapn(cc + lo, n));
#pragma unroll
    for (int j = 0; j < C; ++j) sgrid[j * Sg + c] = g;
  }
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    s_tbl[p][tid] = -1;
    if (tid < R) s_cnt[p][tid] = 0;
    if (tid == 0) s_novf[p] = s_take[p] = 0;
  }
  __syncthreads();
  const int64_t nb = (q + T - 1) / T;
  const double2 *x2 = reinterpret_cast<const double2 *>(xt);
  auto ld = [&](int64_t b) -> double2 {
    const int64_t ii = b * T + tid;
    return (tid < T && b < nb && ii < q) ? __ldg(x2 + ii) : make_double2(0.0, 0.0);
  };
  double2 xn = ld(blockIdx.x);
  const int lane16 = tid & 15;
  int it = 0;
  for (int64_t bt = blockIdx.x; bt < nb; bt += gridDim.x, ++it) {
    const int p = it % 3, pn = (it + 1) % 3;
    const double2 xc = xn;
    const int64_t i = bt * T + tid;
    xn = ld(bt + gridDim.x);
    // classify into set p; set pn (last read two batches ago) is cleared for the next batch
    if (tid < R) s_cnt[pn][tid] = 0;
    if (tid == 0) s_novf[pn] = s_take[pn] = 0;
    if (tid < T && i < q) {
      if (xc.x >= 0.0 && xc.x <= 1.0 && xc.y >= 0.0 && xc.y <= 1.0) {
        double s0, s1;
        const int b0 = es_reduce<W>(h * xc.x * (double)n, s0);
        const int b1 = es_reduce<W>(h * xc.y * (double)n, s1);
        s_s[p][tid] = make_double2(s0, s1);
        const int cell = (b0 - lo) * A + (b1 - lo);
        s_cell[p][tid] = cell;
        const int c = cell & (R - 1);
        const int k = atomicAdd(&s_cnt[p][c], 1);
        if (k < QC) s_tbl[p][16 * (k / C) + c + (k % C) * R] = (short)tid;
        else s_ovf[p][atomicAdd(&s_novf[p], 1)] = (short)tid;
      } else {
        mu[i] = __longlong_as_double(0x7ff8000000000000LL);
        atomicOr(err + 1, 1);
      }
    }
    __syncthreads();
    // gathers from set p
    int j = s_tbl[p][tid];
    s_tbl[p][tid] = -1;  // (re-filled three batches on, after two more barriers)
    if (j < 0) {
      const int novf = s_novf[p];
      if (novf > 0) {
        const int t = atomicAdd(&s_take[p], 1);
        if (t < novf) j = s_ovf[p][t];
      }
    }
    if (j >= 0) {
      const int cell = s_cell[p][j];
      EFGP_DCHECK(j < T && cell >= 0 && cell + (W - 1) * (A + 1) < A * A);
      double wt[2][W];
      const double2 sj = s_s[p][j];
      es_weights_s<W>(sj.x, P, wt[0]);
      es_weights_s<W>(sj.y, P, wt[1]);
      // the copy whose shift maps this cell's bank class onto this lane (exact for in-quota targets)
      const int cp = ((lane16 - cell) & 15) / R;
      const double *win = sgrid + cp * Sg + cell;
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < W; ++a) {
        double ra = 0.0;
#pragma unroll
        for (int b = 0; b < W; ++b) ra = fma(win[a * A + b], wt[1][b], ra);
        acc = fma(ra, wt[0][a], acc);
      }
      const int64_t ij = bt * T + j;
      if (sd) {  // NEXT-3: w_n = (Phi p)_n / sigma_n^2 (reading G11)
        const double sn = __ldg(sd + ij);
        acc /= sn * sn;
      }
      mu[ij] = acc;
    }
  }
}

// dynamic shared bytes of the triple-buffered tables of k_interp2_copies<W, C, T, NT>
template <int C, int T, int NT>
constexpr size_t interp_copies_tables() {
  return 3 * ((size_t)T * (16 + 4 + 2) + (size_t)NT * 2);
}

template <int W, int C, int T, int NT>
static bool try_interp_copies(efgp_plan *pl, const double *grid, int n, const double *xt, int64_t q,
                              const double *sd, double *mu, int lo, int A, cudaStream_t s) {
  constexpr int R = 16 / C;
  const int Sg = ((A * A + 15) / 16) * 16 + R;  // copy stride = R (mod 16) doubles (R even: 16-byte tables)
  const size_t sb = (size_t)Sg * C * sizeof(double) + interp_copies_tables<C, T, NT>();
  const size_t per_cta = sb + 1024;
  const int ctas = NT <= 512 ? 1024 / NT : 1;
  if (per_cta * ctas > 227 * 1024) return false;
  if (cudaFuncSetAttribute(k_interp2_copies<W, C, T, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb) !=
      cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  const int64_t nbt = (q + T - 1) / T;
  const int64_t nblk = std::min<int64_t>(nbt, (int64_t)ctas * pl->num_sms);
  k_interp2_copies<W, C, T, NT><<<(unsigned)nblk, NT, sb, s>>>(xt, q, grid, n, pl->P.h, pl->P.poly, lo, A, Sg, sd,
                                                               mu, pl->dflags);
  return true;
}

template <int D, int W>
static efgp_status launch_interp(efgp_plan *pl, const double *grid, int n, const double *xt, int64_t q,
                                 const double *sd, double *mu, cudaStream_t s) {
  const Params &P = pl->P;
  const Occ2 o = occupied2(P.h, n, W);
  size_t cells = o.A;
  for (int k = 1; k < D; ++k) cells *= o.A;
  const size_t sb = cells * sizeof(double);
  int64_t blocks = (q + 255) / 256;
  if constexpr (D == 2) {
    // many targets: shifted grid copies (EFGP_K9 = banked | c2 | c4 selects the variant for A/B runs)
    const char *k9 = getenv("EFGP_K9");
    const bool aligned = (reinterpret_cast<uintptr_t>(xt) & 15) == 0 && !getenv("EFGP_INTERP_PLAIN");
    if (aligned && q >= (int64_t)pl->num_sms * 512 && !(k9 && !strcmp(k9, "banked"))) {
      // C = 4, 896 targets per batch (r02 A/B at q = 2e8: 2.69 ms against 2.79 for 768 and 2.84 for the
      // banked kernel; C = 2 with two CTAs per SM 2.89)
      const bool c2 = k9 && !strcmp(k9, "c2"), c4r = k9 && !strcmp(k9, "c4r");
      const bool ok = c2    ? try_interp_copies<W, 2, 384, 512>(pl, grid, n, xt, q, sd, mu, o.lo, o.A, s)
                      : c4r ? try_interp_copies<W, 4, 640, 768>(pl, grid, n, xt, q, sd, mu, o.lo, o.A, s)
                            : try_interp_copies<W, 4, 896, 1024>(pl, grid, n, xt, q, sd, mu, o.lo, o.A, s);
      if (ok) {
        EFGP_CUDA(cudaGetLastError());
        return EFGP_OK;
      }
    }
  }
  if (D == 2 && q >= (int64_t)pl->num_sms * kIB && sb <= 160 * 1024 && (reinterpret_cast<uintptr_t>(xt) & 15) == 0 &&
      !getenv("EFGP_INTERP_PLAIN")) {
    // many targets: bank-aware order (1024 / kIB CTAs of kIB threads per SM, persistent over batches)
    EFGP_CUDA(cudaFuncSetAttribute(k_interp2_banked<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
    const int64_t nbt = (q + kIB - 1) / kIB;
    const int64_t nblk = std::min<int64_t>(nbt, (int64_t)(1024 / kIB) * pl->num_sms);
    k_interp2_banked<W><<<(unsigned)nblk, kIB, sb, s>>>(xt, q, grid, n, P.h, P.poly, o.lo, o.A, sd, mu, pl->dflags);
    EFGP_CUDA(cudaGetLastError());
    return EFGP_OK;
  }
  if (sb <= 160 * 1024) {
    // one wave of persistent CTAs so the staged grid is reused across many targets; 1024 resident
    // threads per SM whatever the staged size (4 x 256, 2 x 512 or 1 x 1024)
    const int per_sm = sb <= 48 * 1024 ? 4 : (sb <= 100 * 1024 ? 2 : 1);
    const int threads = std::min(1024 / per_sm, interp_max_threads<D, W>());
    blocks = (q + threads - 1) / threads;
    const int64_t cap = (int64_t)pl->num_sms * per_sm;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    EFGP_CUDA(cudaFuncSetAttribute(k_interp<D, W, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
    k_interp<D, W, true><<<(unsigned)blocks, threads, sb, s>>>(xt, q, grid, n, P.h, P.poly, o.lo, o.A,
                                                               sd, mu, pl->dflags);
  } else {
    const int64_t cap = (int64_t)pl->num_sms * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    k_interp<D, W, false><<<(unsigned)blocks, 256, 0, s>>>(xt, q, grid, n, P.h, P.poly, o.lo, o.A,
                                                           sd, mu, pl->dflags);
  }
  EFGP_CUDA(cudaGetLastError());
  return EFGP_OK;
}

template <int D>
static efgp_status interp_d(efgp_plan *pl, const double *grid, int n, const double *xt, int64_t q,
                            const double *sd, double *mu, cudaStream_t s) {
  switch (pl->P.w) {
#define EFGP_CASE(WW) \
  case WW:            \
    return launch_interp<D, WW>(pl, grid, n, xt, q, sd, mu, s);
    EFGP_W_CASES2(EFGP_CASE)
#undef EFGP_CASE
  }
  return EFGP_ERR_INVALID;
}

efgp_status interp_targets(efgp_plan *pl, const double *xt, int64_t q, double *mu, cudaStream_t s) {
  return interp_weighted(pl, pl->t2grid, pl->P.n2, xt, q, nullptr, mu, s);
}

efgp_status interp_weighted(efgp_plan *pl, const double *grid, int64_t n, const double *xt, int64_t q,
                            const double *sd, double *out, cudaStream_t s) {
  if (q <= 0) return EFGP_OK;
  switch (pl->P.d) {
    case 1: return interp_d<1>(pl, grid, (int)n, xt, q, sd, out, s);
    case 2: return interp_d<2>(pl, grid, (int)n, xt, q, sd, out, s);
    case 3: return interp_d<3>(pl, grid, (int)n, xt, q, sd, out, s);
  }
  return EFGP_ERR_INVALID;
}

}  // namespace efgp
