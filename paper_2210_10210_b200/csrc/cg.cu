// K4-K7 + F2: conjugate gradients on (D F^*F D + sigma^2 I) beta = D F^*y (eq "be", P:570;
// Alg a1 step 4; stop at relative residual cg_tol), with the Toeplitz
// product of Alg a:FF done by real transforms:
//
//   A p = D . extract_{J_m}( R2C( C2R(pad_L(D . p)) * vhat ) ) + sigma^2 p,   vhat = C2R(v)/L^d (real)
//
// Vectors live on the Hermitian half j_d >= 0 (Mh entries); Hermitian inner products become
// sum_q w_q Re(conj(a_q) b_q) with w_q = 2 for j_d > 0 and 1 for j_d = 0.
// One iteration = C2R, k_mul, R2C, k_cg_apply, k_cg_xr, k_cg_p; a CUDA graph captures
// graph_iters iterations; the host polls a device-side "done" flag after each graph launch, so the
// reported iteration count is exact (kernels of iterations after convergence return at entry).
// Block reductions are deterministic (fixed order, no atomics).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <vector>

#include "efgp_internal.cuh"

namespace efgp {

struct CGState {
  double rr;        // current ||r||^2 (weighted)
  double rr_old;    // ||r||^2 of the previous iteration (for beta_cg)
  double bnorm;     // ||b||
  double tol;
  double sigma2;
  long long iter;
  long long max_iter;
  int done;         // 1: converged, 2: hit max_iter
  int pad_;
  double rz;        // PCG: (r, z) of the current residual (NEXT-4)
  double rrs[2];    // fused direct CG: ||r_j||^2 in slot j & 1 (written by k_cg_toep2f, read one iteration later)
};

constexpr int kCGThreads = 256;



__device__ __forceinline__ double block_sum(double v, double *sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  return t;  // valid in thread 0
}

// every block reduces the same partials in the same order -> identical value everywhere
__device__ __forceinline__ double reduce_partials(const double *__restrict__ part, int n, double *sh) {
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v += part[i];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) sh[32] = v;
  __syncthreads();
  return sh[32];
}

__global__ void k_cg_init(const double2 *__restrict__ b, double2 *__restrict__ x, double2 *__restrict__ r,
                          double2 *__restrict__ p, int64_t Mh, int m, double *__restrict__ part) {
  __shared__ double sh[40];
  double acc = 0.0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x) {
    const double2 bb = b[q];
    x[q] = make_double2(0.0, 0.0);
    r[q] = bb;
    p[q] = bb;
    const double wq = (q % (m + 1)) ? 2.0 : 1.0;
    acc += wq * (bb.x * bb.x + bb.y * bb.y);
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void k_cg_init2(CGState *st, const double *__restrict__ part, int nblk, double *hist) {
  __shared__ double sh[40];
  const double rr = reduce_partials(part, nblk, sh);
  if (threadIdx.x == 0) {
    st->rr = rr;
    st->rr_old = rr;
    st->rrs[0] = rr;
    st->bnorm = sqrt(rr);
    st->iter = 0;
    st->done = (rr == 0.0) ? 1 : 0;
    hist[0] = rr == 0.0 ? 0.0 : 1.0;
  }
}

// pad: Xbox = D . p at the J_m bins of the L-box, 0 elsewhere (the C2R input; cuFFT may overwrite
// it, so it is rewritten in full every iteration)
template <int D>
__device__ __forceinline__ void pad_box(const double2 *__restrict__ p, const double *__restrict__ Dh, int m,
                                        int64_t L, double2 *__restrict__ X, int64_t box) {
  const int64_t nh = L / 2 + 1;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < box;
       idx += (int64_t)gridDim.x * blockDim.x) {
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

template <int D>
__global__ void k_cg_pad0(const double2 *__restrict__ p, const double *__restrict__ Dh, int m, int64_t L,
                          double2 *__restrict__ X, int64_t box) {
  pad_box<D>(p, Dh, m, L, X, box);
}

__global__ void k_mul(double *__restrict__ Y, const double *__restrict__ vhat, int64_t n, const CGState *st) {
  if (st->done) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    Y[i] *= vhat[i];
}

// Ap = D . Z[J_m] + sigma^2 p ; partial <p, Ap>
template <int D>
__global__ void k_cg_apply(const double2 *__restrict__ Z, const double2 *__restrict__ p, const double *__restrict__ Dh,
                           double2 *__restrict__ Ap, int64_t Mh, int m, int64_t L, const CGState *st,
                           double *__restrict__ part) {
  __shared__ double sh[40];
  pdl_trigger();
  if (st->done) return;
  const double s2 = st->sigma2;
  double acc = 0.0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = q;
    const int64_t jd = rem % (m + 1);
    rem /= (m + 1);
    int64_t zi = jd, stride = L / 2 + 1;
#pragma unroll
    for (int k = D - 2; k >= 0; --k) {
      int64_t j = rem % (2 * m + 1) - m;
      rem /= (2 * m + 1);
      zi += (j < 0 ? j + L : j) * stride;
      stride *= L;
    }
    const double2 z = Z[zi], pp = p[q];
    const double dq = Dh[q];
    const double2 a = make_double2(dq * z.x + s2 * pp.x, dq * z.y + s2 * pp.y);
    Ap[q] = a;
    const double wq = jd ? 2.0 : 1.0;
    acc += wq * (pp.x * a.x + pp.y * a.y);
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// alpha = rr / <p,Ap>; x += alpha p; r -= alpha Ap; partial ||r||^2
__global__ void k_cg_xr(double2 *__restrict__ x, double2 *__restrict__ r, const double2 *__restrict__ p,
                        const double2 *__restrict__ Ap, int64_t Mh, int m, CGState *st,
                        const double *__restrict__ part_pAp, double *__restrict__ part_rr, int nblk,
                        const double *__restrict__ part_rz = nullptr) {
  __shared__ double sh[40];
  pdl_wait();
  pdl_trigger();
  if (st->done) return;
  const double pAp = reduce_partials(part_pAp, nblk, sh);
  // CG: alpha = (r,r)/(p,Ap); PCG: alpha = (r,z)/(p,Ap), (r,z) reduced from its partials
  const double rr = part_rz ? reduce_partials(part_rz, nblk, sh) : st->rr;
  if (part_rz && blockIdx.x == 0 && threadIdx.x == 0) st->rz = rr;
  const double alpha = rr / pAp;
  double acc = 0.0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x) {
    const double2 pp = p[q], a = Ap[q];
    double2 xx = x[q], rq = r[q];
    xx.x += alpha * pp.x;
    xx.y += alpha * pp.y;
    rq.x -= alpha * a.x;
    rq.y -= alpha * a.y;
    x[q] = xx;
    r[q] = rq;
    const double wq = (q % (m + 1)) ? 2.0 : 1.0;
    acc += wq * (rq.x * rq.x + rq.y * rq.y);
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) {
    part_rr[blockIdx.x] = acc;
    if (blockIdx.x == 0 && !part_rz) st->rr_old = rr;
  }
}

// beta_cg = rr_new / rr_old; p = r + beta_cg p; pad; bookkeeping (block 0)
template <int D>
__global__ void k_cg_p(const double2 *__restrict__ r, double2 *__restrict__ p, const double *__restrict__ Dh,
                       int64_t Mh, int m, int64_t L, double2 *__restrict__ X, int64_t box, CGState *st,
                       const double *__restrict__ part_rr, int nblk, double *__restrict__ hist) {
  __shared__ double sh[40];
  pdl_wait();
  pdl_trigger();
  if (st->done) return;
  const double rr_new = reduce_partials(part_rr, nblk, sh);
  const double bcg = rr_new / st->rr_old;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x) {
    const double2 rq = r[q], pp = p[q];
    const double2 pn = make_double2(rq.x + bcg * pp.x, rq.y + bcg * pp.y);
    p[q] = pn;
    if (X) {  // partial-transform product (toeplitz_pt): scatter D p into its slab (X = pt_P, box = L^(d-1))
      int j[D];
      decode_half<D>(q, m, j);
      int64_t o = 0;
#pragma unroll
      for (int k = 0; k < D - 1; ++k) o = o * L + (j[k] < 0 ? j[k] + L : j[k]);
      const double dq = Dh[q];
      X[(int64_t)j[D - 1] * box + o] = make_double2(dq * pn.x, dq * pn.y);
    }
  }
  // grid-wide dependency: the padded-FFT path's pad reads p written by other blocks -> separate kernel
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->rr = rr_new;
    const long long it = st->iter + 1;
    st->iter = it;
    const double rel = sqrt(rr_new) / st->bnorm;
    hist[it] = rel;
    if (rel <= st->tol) st->done = 1;
    else if (it >= st->max_iter) st->done = 2;
  }
}

template <int D>
__global__ void k_cg_pad(const double2 *__restrict__ p, const double *__restrict__ Dh, int m, int64_t L,
                         double2 *__restrict__ X, int64_t box, const CGState *st) {
  // runs even when done was just set: harmless (the next C2R input is never used)
  pdl_wait();
  pad_box<D>(p, Dh, m, L, X, box);
}

// ---- Toeplitz product by partial transforms (toeplitz_pt: d >= 2, m too large for the direct one)
// out_j = sum_{k in J_m} v_{j-k} u_k (u = D p, j in J_m; eq "223") split as j = (j', j_d):
//   T[k_d][x]  = sum_{k'} u_{k', k_d} e^{+2 pi i k'.x/L}                 (x in the L^(d-1) plane; cuFFT)
//   W[j_d][x]  = sum_{k_d = -m}^{m} Vt[j_d - k_d][x] T[k_d][x]           (direct 1D convolution per line)
//   out_{j', j_d} = sum_x e^{-2 pi i j'.x/L} W[j_d][x]                    (cuFFT)
// with Vt[delta_d][x] = L^(1-d) sum_{delta'} v_{delta', delta_d} e^{+2 pi i delta'.x/L}, delta_d in
// [-m, 2m].  Exact for L >= 4m+1 (the circulant embedding of Alg a:FF, on the first d-1
// axes only); T[-k_d][x] = conj T[k_d][x] because u is Hermitian, so only the m+1 half slabs are
// transformed.  Against the padded real-FFT product: 2 (d-1)-dim transforms of (m+1)/(L/2+1) of the
// box instead of two d-dim ones, no L^d real intermediate, and the last axis is pruned exactly
// (2m+1 inputs, m+1 outputs).  Layout: slab-major, [slab][x], x = bins row-major over the first d-1 axes.

static int64_t ipow_(int64_t b, int e) {
  int64_t r = 1;
  while (e-- > 0) r *= b;
  return r;
}
static unsigned nblocks_pt(int64_t n, int sms) {
  const int64_t b = std::min<int64_t>((n + kCGThreads - 1) / kCGThreads, (int64_t)sms * 4);
  return (unsigned)(b < 1 ? 1 : b);
}

// plane offset of the bins of j' (first d-1 coordinates of j) in an L^(d-1) plane
template <int D>
__device__ __forceinline__ int64_t pt_plane(const int (&j)[D], int64_t L) {
  int64_t o = 0;
#pragma unroll
  for (int k = 0; k < D - 1; ++k) o = o * L + (j[k] < 0 ? j[k] + L : j[k]);
  return o;
}

// P[j_d][bins(j')] = D_j p_j for every half mode (the other entries stay zero from setup)
template <int D>
__global__ void k_pt_pad(const double2 *__restrict__ p, const double *__restrict__ Dh, int64_t Mh, int m, int64_t L,
                         int64_t Lp, double2 *__restrict__ Pb) {
  pdl_wait();
  pdl_trigger();
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x) {
    int j[D];
    decode_half<D>(q, m, j);
    const double2 pp = p[q];
    const double dq = Dh[q];
    Pb[(int64_t)j[D - 1] * Lp + pt_plane<D>(j, L)] = make_double2(dq * pp.x, dq * pp.y);
  }
}

// Vt before its transform: slab s = delta_d + m, plane bins -> delta' (|delta'_k| <= 2m, else 0)
template <int D>
__global__ void k_pt_place_v(const double2 *__restrict__ vh, int m, int64_t L, int64_t Lp, double scale,
                             double2 *__restrict__ V) {
  const int64_t n = (int64_t)(3 * m + 1) * Lp;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t x = i % Lp;
    int j[D];
    j[D - 1] = (int)(i / Lp) - m;
    bool ok = true;
#pragma unroll
    for (int k = D - 2; k >= 0; --k) {
      const int64_t b = x % L;
      x /= L;
      const int64_t dl = b <= L / 2 ? b : b - L;
      ok = ok && dl >= -2 * m && dl <= 2 * m;
      j[k] = (int)dl;
    }
    double2 val = make_double2(0.0, 0.0);
    if (ok) {
      const bool neg = j[D - 1] < 0;
      if (neg)
#pragma unroll
        for (int k = 0; k < D; ++k) j[k] = -j[k];
      const double2 v = vh[encode_half<D>(j, 2 * m)];
      val = make_double2(scale * v.x, scale * (neg ? -v.y : v.y));
    }
    V[i] = val;
  }
}

// W[j][x] = sum_{k=-m}^{m} Vt[j - k][x] T[k][x] for j in [j0, j0 + G).  CTA = 32 consecutive lines x
// (lane) x ngroups warps (warp g: outputs [g G, g G + G)).  The CTA first stages its lines' T (m+1
// slabs) and Vt (3m+1 slabs) in shared memory with coalesced 512-byte rows (one pass over HBM/L2 for
// both arrays), then each thread slides a G-register window of Vt down one slab per step k, so
// every step costs two conflict-free shared loads for G complex MACs (slot of window element r is r
// mod G; the steps are unrolled in blocks of G so every slot index is static).
// Shared-memory geometry of k_pt_conv: KS warps split the 2m+1 steps of each output group (SS steps
// each, a multiple of G), the staged Vt is padded with zero slabs below (vlo) and above, T with zero
// slabs above m, so the inner loop has no bounds checks.
struct PtConvGeom {
  int ng, SS, vlo, nV, nT;
  __host__ __device__ PtConvGeom(int m, int G, int KS) {
    ng = (m + 1 + G - 1) / G;
    SS = ((2 * m + 1 + KS - 1) / KS + G - 1) / G * G;
    vlo = KS * SS - 1 - 2 * m > 0 ? KS * SS - 1 - 2 * m : 0;
    const int vhi = ng * G - 1 - m > 0 ? ng * G - 1 - m : 0;
    nV = vlo + 3 * m + 1 + vhi;
    const int tmax = KS * SS - 1 - m > m ? KS * SS - 1 - m : m;
    nT = tmax + 1;
  }
  __host__ __device__ size_t smem() const { return sizeof(double2) * 32 * (size_t)(nT + nV); }
};
constexpr int kPtKS = 2;

// W[j][x] = sum_{k=-m}^{m} Vt[j - k][x] T[k][x] for j in [j0, j0 + G).  CTA = 32 consecutive lines x
// (lane) x ng output groups x KS step splits (warp w: group w % ng, steps of split w / ng; the KS
// partial sums are added through shared memory at the end).  The CTA first stages its lines' T (m+1
// slabs) and Vt (3m+1 slabs) in shared memory by bulk async copies of 512-byte rows (one pass over
// HBM/L2 for both), then each thread slides a G-register window of Vt down one slab per step k, so
// every step costs two conflict-free shared loads for G complex MACs (slot of window element r is r
// mod G; steps are unrolled in blocks of G so every slot index is static).
template <int G>
__global__ void __launch_bounds__(512) k_pt_conv(const double2 *__restrict__ T, const double2 *__restrict__ Vt,
                                                 double2 *__restrict__ W, int m, int64_t Lp, const CGState *st) {
  extern __shared__ __align__(16) double2 pt_sm[];
  __shared__ __align__(8) uint64_t bar;
  pdl_wait();
  pdl_trigger();
  if (st && st->done) return;
  const PtConvGeom geo(m, G, kPtKS);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, grp = w % geo.ng, ks = w / geo.ng;
  const int64_t x0 = (int64_t)blockIdx.x * 32;
  const int nl = Lp - x0 < 32 ? (int)(Lp - x0) : 32;
  double2 *sT = pt_sm, *sV = pt_sm + 32 * geo.nT;
  // zero the padding slabs, then one bulk async copy (TMA engine) of nl x 16 bytes per slab row
  for (int i = threadIdx.x; i < 32 * geo.nT; i += blockDim.x)
    if (i >= 32 * (m + 1)) sT[i] = make_double2(0.0, 0.0);
  for (int i = threadIdx.x; i < 32 * geo.nV; i += blockDim.x) {
    const int sl = i >> 5;
    if (sl < geo.vlo || sl >= geo.vlo + 3 * m + 1) sV[i] = make_double2(0.0, 0.0);
  }
  const uint32_t sbar = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nrow = m + 1 + 3 * m + 1;
  if (w == 0) {
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"((uint32_t)(nrow * nl * 16))
                   : "memory");
    __syncwarp();
    for (int sl = lane; sl < nrow; sl += 32) {
      const bool isT = sl < m + 1;
      const double2 *src = isT ? T + (int64_t)sl * Lp + x0 : Vt + (int64_t)(sl - m - 1) * Lp + x0;
      double2 *dst = isT ? sT + 32 * sl : sV + 32 * (geo.vlo + sl - m - 1);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(dst)),
                   "l"(src), "r"((uint32_t)(nl * 16)), "r"(sbar)
                   : "memory");
    }
  }
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}" ::"r"(sbar)
      : "memory");
  const int j0 = grp * G, s0 = ks * geo.SS;
  // window element r (output g = r + s at step s) lives in slot r mod G; its slab is j0 + r + 2m
  const double2 *vl = sV + 32 * (geo.vlo + j0 + 2 * m) + lane;
  double2 acc[G], win[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    acc[g] = make_double2(0.0, 0.0);
    win[g] = vl[32 * (g - s0)];  // r = g - s0 (slot g, since s0 = 0 mod G)
  }
  const double2 *tl = sT + lane;
  for (int sb = s0; sb < s0 + geo.SS; sb += G) {
#pragma unroll
    for (int u = 0; u < G; ++u) {
      const int s = sb + u;
      if (u > 0 || sb > s0) win[(G - u) % G] = vl[-32 * s];  // element r = -s enters slot (-s) mod G
      const int k = s - m;
      double2 t = tl[32 * (k >= 0 ? k : -k)];
      t.y = k >= 0 ? t.y : -t.y;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const double2 wv = win[((g - u) % G + G) % G];
        acc[g].x = fma(wv.x, t.x, fma(-wv.y, t.y, acc[g].x));
        acc[g].y = fma(wv.x, t.y, fma(wv.y, t.x, acc[g].y));
      }
    }
  }
  // split partial sums: warps of split ks > 0 park theirs in shared memory, split 0 adds and stores
  __syncthreads();
  double2 *red = pt_sm + (size_t)(w - geo.ng) * 32 * G;  // (ks >= 1) slot of warp w
  if (ks > 0)
#pragma unroll
    for (int g = 0; g < G; ++g) red[g * 32 + lane] = acc[g];
  __syncthreads();
  if (ks == 0 && lane < nl) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      double2 a = acc[g];
      for (int q = 1; q < kPtKS; ++q) {
        const double2 b = pt_sm[(size_t)((q - 1) * geo.ng + grp) * 32 * G + g * 32 + lane];
        a.x += b.x;
        a.y += b.y;
      }
      if (j0 + g <= m) W[(int64_t)(j0 + g) * Lp + x0 + lane] = a;
    }
  }
}

template <int G>
static size_t pt_conv_smem(int m) { return PtConvGeom(m, G, kPtKS).smem(); }

// Ap = D . out[J_m] + sigma^2 p ; partial <p, Ap> (out = forward transform of W, slab-major)
template <int D>
__global__ void k_pt_apply(const double2 *__restrict__ Z, const double2 *__restrict__ p, const double *__restrict__ Dh,
                           double2 *__restrict__ Ap, int64_t Mh, int m, int64_t L, int64_t Lp, const CGState *st,
                           double *__restrict__ part) {
  __shared__ double sh[40];
  pdl_trigger();
  if (st->done) return;
  const double s2 = st->sigma2;
  double acc = 0.0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x) {
    int j[D];
    decode_half<D>(q, m, j);
    // exactly Hermitian in the j_d = 0 plane (as the R2C of the padded-FFT product is): out_{-j'} =
    // conj out_{j'}, read from the canonical j' (first nonzero coordinate positive); without this the
    // roundoff of the two independent sums breaks the half-space CG (iterates leave the Hermitian set)
    bool neg = false, zero = false;
    if (j[D - 1] == 0) {
      int sgn = 0;
#pragma unroll
      for (int k = 0; k < D - 1; ++k)
        if (sgn == 0 && j[k] != 0) sgn = j[k] > 0 ? 1 : -1;
      neg = sgn < 0;
      zero = sgn == 0;
      if (neg)
#pragma unroll
        for (int k = 0; k < D - 1; ++k) j[k] = -j[k];
    }
    double2 z = Z[(int64_t)j[D - 1] * Lp + pt_plane<D>(j, L)];
    if (neg) z.y = -z.y;
    if (zero) z.y = 0.0;  // j = 0: real
    const double2 pp = p[q];
    const double dq = Dh[q];
    const double2 a = make_double2(dq * z.x + s2 * pp.x, dq * z.y + s2 * pp.y);
    Ap[q] = a;
    acc += (j[D - 1] ? 2.0 : 1.0) * (pp.x * a.x + pp.y * a.y);
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

static int pt_group() {  // outputs per thread of k_pt_conv (EFGP_PT_G overrides: 4, 8, 10, 13)
  const char *e = getenv("EFGP_PT_G");
  return e ? atoi(e) : 0;
}

template <int G>
static cudaError_t pt_conv_launch(efgp_plan *pl, const CGState *st, cudaStream_t s) {
  const Params &P = pl->P;
  const int64_t Lp = ipow_(P.L, P.d - 1);
  const int ng = (int)((P.m + 1 + G - 1) / G);
  return launch_pdl_smem(k_pt_conv<G>, (unsigned)((Lp + 31) / 32), 32 * ng * kPtKS, pt_conv_smem<G>((int)P.m), s,
                         (const double2 *)pl->pt_T, (const double2 *)pl->pt_V, pl->pt_W, (int)P.m, Lp, st);
}

// out = T(D p) into pt_T (slab-major), the three launches between the pad and the apply
static efgp_status pt_product(efgp_plan *pl, const CGState *st, cudaStream_t s) {
  const Params &P = pl->P;
  EFGP_CUFFT(cufftExecZ2Z(pl->plan_pt, pl->pt_P, pl->pt_T, CUFFT_INVERSE));
  int G = pt_group();
  const int64_t Lp = ipow_(P.L, P.d - 1);
  if (G == 0) G = 10;
  cudaError_t e;
  switch (G) {
    case 4: e = pt_conv_launch<4>(pl, st, s); break;
    case 8: e = pt_conv_launch<8>(pl, st, s); break;
    case 10: e = pt_conv_launch<10>(pl, st, s); break;
    default: e = pt_conv_launch<13>(pl, st, s); break;
  }
  EFGP_CUDA(e);
  EFGP_CUFFT(cufftExecZ2Z(pl->plan_pt, pl->pt_W, pl->pt_T, CUFFT_FORWARD));
  return EFGP_OK;
}

template <int D>
static efgp_status pt_pad(efgp_plan *pl, const double2 *p, cudaStream_t s) {
  const Params &P = pl->P;
  EFGP_CUDA(launch_pdl(k_pt_pad<D>, nblocks_pt(P.Mh, pl->num_sms), kCGThreads, s, p, (const double *)pl->D_half, P.Mh,
                       (int)P.m, (int64_t)P.L, ipow_(P.L, D - 1), pl->pt_P));
  return EFGP_OK;
}

efgp_status pt_setup(efgp_plan *pl, const double2 *vh, cudaStream_t s) {
  const Params &P = pl->P;
  const int d = P.d;
  const int64_t Lp = ipow_(P.L, d - 1), ns = P.m + 1;
  if (!pl->pt_P) {
    EFGP_CUDA(cudaMalloc((void **)&pl->pt_P, sizeof(double2) * ns * Lp));
    EFGP_CUDA(cudaMalloc((void **)&pl->pt_T, sizeof(double2) * ns * Lp));
    EFGP_CUDA(cudaMalloc((void **)&pl->pt_W, sizeof(double2) * ns * Lp));
    EFGP_CUDA(cudaMalloc((void **)&pl->pt_V, sizeof(double2) * (3 * P.m + 1) * Lp));
    EFGP_CUDA(cudaMemsetAsync(pl->pt_P, 0, sizeof(double2) * ns * Lp, s));
    int dims[2] = {(int)P.L, (int)P.L};
    EFGP_CUFFT(cufftPlanMany(&pl->plan_pt, d - 1, dims, nullptr, 1, (int)Lp, nullptr, 1, (int)Lp, CUFFT_Z2Z, (int)ns));
    EFGP_CUFFT(cufftPlanMany(&pl->plan_ptv, d - 1, dims, nullptr, 1, (int)Lp, nullptr, 1, (int)Lp, CUFFT_Z2Z,
                             (int)(3 * P.m + 1)));
  }
  const int64_t n = (3 * P.m + 1) * Lp;
  const unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)pl->num_sms * 8);
  EFGP_CUDA(cudaFuncSetAttribute(k_pt_conv<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pt_conv_smem<4>((int)P.m)));
  EFGP_CUDA(cudaFuncSetAttribute(k_pt_conv<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pt_conv_smem<8>((int)P.m)));
  EFGP_CUDA(cudaFuncSetAttribute(k_pt_conv<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pt_conv_smem<10>((int)P.m)));
  EFGP_CUDA(cudaFuncSetAttribute(k_pt_conv<13>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pt_conv_smem<13>((int)P.m)));
  if (d == 2) k_pt_place_v<2><<<g, 256, 0, s>>>(vh, (int)P.m, P.L, Lp, 1.0 / (double)Lp, pl->pt_V);
  else k_pt_place_v<3><<<g, 256, 0, s>>>(vh, (int)P.m, P.L, Lp, 1.0 / (double)Lp, pl->pt_V);
  EFGP_CUDA(cudaGetLastError());
  EFGP_CUFFT(cufftSetStream(pl->plan_ptv, s));
  EFGP_CUFFT(cufftExecZ2Z(pl->plan_ptv, pl->pt_V, pl->pt_V, CUFFT_INVERSE));
  return EFGP_OK;
}


// Toeplitz product by direct convolution (2D, small m; toeplitz_direct): CTA = output row j1.
//   out_j = sum_{k in J_m} v_{j-k} u_k,  u = D p (Hermitian completion of the half),  j = (j1, 0..m)
//   Ap_j = D_j out_j + sigma^2 p_j,  partial <p, Ap>
// Replaces pad + C2R + multiply + R2C + apply of the FFT path; the same operator (the FFT path's
// circulant embedding is exact for |j - k| <= 2m), summed directly.  c3 / c5: 25-28 -> 20-21 us per
// CG iteration (1024 threads; 256 threads gave 23-24 us, a thread per output 27 us).
constexpr int kToepThreads = 1024;
__global__ void __launch_bounds__(kToepThreads) k_cg_toep2(const double2 *__restrict__ vfull,
                                                           const double2 *__restrict__ p,
                                                           const double *__restrict__ Dh, double2 *__restrict__ Ap,
                                                           int m, const CGState *st, double *__restrict__ part) {
  extern __shared__ double2 tsm[];
  __shared__ double sh[40];
  pdl_trigger();
  if (st->done) return;
  const int n = 2 * m + 1, nv = 4 * m + 1, j1 = (int)blockIdx.x - m;
  double2 *u = tsm;                // n x n: u[(k1+m) n + (k2+m)]
  double2 *vr = tsm + n * n;       // n rows x nv: vr[(k1+m) nv + (s+2m)] = v_{j1-k1, s}
  double2 *red = vr + n * nv;      // partial sums [slices][m+1]
  // u from the canonical half (k2 > 0, or k2 = 0 and k1 >= 0): the redundant (k1 < 0, 0) entries of the
  // stored half are not read, so the product is exactly Hermitian (the FFT path's C2R projects the
  // same way); without this the CG stalls on the c3 systems (roundoff in the j2 = 0 plane)
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    int k1 = idx / n - m, k2 = idx % n - m;
    const bool neg = k2 < 0 || (k2 == 0 && k1 < 0);
    if (neg) {
      k1 = -k1;
      k2 = -k2;
    }
    const int64_t q = (int64_t)(k1 + m) * (m + 1) + k2;
    const double2 pp = p[q];
    const double dq = Dh[q];
    u[idx] = make_double2(dq * pp.x, neg ? -dq * pp.y : dq * pp.y);
  }
  for (int idx = threadIdx.x; idx < n * nv; idx += blockDim.x) {
    const int k1 = idx / nv - m, sc = idx % nv;
    vr[idx] = vfull[(int64_t)(j1 - k1 + 2 * m) * nv + sc];
  }
  __syncthreads();
  // each thread: 4 consecutive outputs j2 .. j2+3 over a slice of the k1 rows; along k2 the four
  // v_{j1-k1, j2+o-k2} form a sliding window (one new shared load per step): 2 loads per 4 MACs
  const int nout = m + 1, ngrp = (nout + 3) / 4, slices = blockDim.x / ngrp;
  const int t = threadIdx.x, g4 = t % ngrp, sl = t / ngrp, j2b = 4 * g4;
  if (sl < slices) {
    double re[4] = {0.0, 0.0, 0.0, 0.0}, im[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k1 = sl; k1 < n; k1 += slices) {  // k1 + m
      const double2 *ur = u + k1 * n;
      // v index of (j2b + o) - k2 at k2 = -m: j2b + o + m + 2m
      const double2 *vrow = vr + k1 * nv + (j2b + 3 * m);
      double2 w[4];
#pragma unroll
      for (int o = 0; o < 4; ++o) w[o] = (j2b + o <= m) ? vrow[o] : make_double2(0.0, 0.0);
      for (int k2 = 0; k2 < n; ++k2) {  // k2 + m; the window moves down by one cell per step
        const double2 b = ur[k2];
#pragma unroll
        for (int o = 0; o < 4; ++o) {
          re[o] = fma(w[o].x, b.x, fma(-w[o].y, b.y, re[o]));
          im[o] = fma(w[o].x, b.y, fma(w[o].y, b.x, im[o]));
        }
#pragma unroll
        for (int o = 3; o > 0; --o) w[o] = w[o - 1];
        const int nxt = j2b + 3 * m - (k2 + 1);  // v index of output j2b at the next k2
        w[0] = (k2 + 1 < n) ? vr[k1 * nv + nxt] : make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int o = 0; o < 4; ++o)
      if (j2b + o <= m) red[sl * nout + j2b + o] = make_double2(re[o], im[o]);
  }
  __syncthreads();
  double acc = 0.0;
  if (t < nout && !(t == 0 && j1 < 0)) {  // (j1 < 0, 0) is written by row -j1 as the conjugate
    double2 o = make_double2(0.0, 0.0);
    for (int k = 0; k < slices; ++k) {
      o.x += red[k * nout + t].x;
      o.y += red[k * nout + t].y;
    }
    const int64_t q = (int64_t)(j1 + m) * (m + 1) + t;
    const double2 pp = p[q];
    const double dq = Dh[q], s2 = st->sigma2;
    double2 a = make_double2(dq * o.x + s2 * pp.x, dq * o.y + s2 * pp.y);
    if (t == 0 && j1 == 0) a.y = s2 * pp.y;  // j = 0: (T u)_0 is real
    Ap[q] = a;
    acc = (t ? 2.0 : 1.0) * (pp.x * a.x + pp.y * a.y);
    if (t == 0 && j1 > 0) {  // the mirrored entry (-j1, 0) = conj, with the canonical p
      Ap[(int64_t)(m - j1) * (m + 1)] = make_double2(a.x, -a.y);
      acc *= 2.0;
    }
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// The same product split over the k1 rows so that all SMs work (k_cg_toep2 runs 2m+1 = 51 CTAs on
// 148 SMs, FP64 pipe ~22 %, r01 ncu): CTA (row j1, split s) sums k1 in its range, every thread 4
// consecutive outputs j2 over one k1 row and a chunk of the k2 range (sliding window as above); the
// CTA's partial row goes to part[row][s]; the last CTA of a row (counter) adds the kToepSplits partials
// in fixed order (deterministic), applies D and sigma^2 and writes the row's <p, Ap> partial.
constexpr int kToepSplits = kToepSplitsHost, kToepSThreads = 256;
__host__ __device__ constexpr int toeps_rows_per_split(int n) { return (n + kToepSplits - 1) / kToepSplits; }

__global__ void __launch_bounds__(kToepSThreads) k_cg_toep2s(const double2 *__restrict__ vfull,
                                                             const double2 *__restrict__ p,
                                                             const double *__restrict__ Dh, double2 *__restrict__ Ap,
                                                             int m, const CGState *st, double2 *__restrict__ tpart,
                                                             unsigned *__restrict__ tcnt, double *__restrict__ part) {
  extern __shared__ double2 tsm[];
  __shared__ double sh[40];
  __shared__ bool last_s;
  pdl_trigger();
  if (st->done) return;
  const int n = 2 * m + 1, nv = 4 * m + 1, nout = m + 1, ngrp = (nout + 3) / 4;
  const int row = (int)blockIdx.x % n, spl = (int)blockIdx.x / n, j1 = row - m;
  const int nk = toeps_rows_per_split(n), k1a = spl * nk, k1b = min(n, k1a + nk), nkr = k1b - k1a;
  const int nc = kToepSThreads / (ngrp * nk), clen = (n + nc - 1) / nc;  // k2 chunks
  double2 *u = tsm;              // nk x n: u[(k1 - k1a) n + (k2 + m)]
  double2 *vr = u + nk * n;      // nk x nv: v_{j1 - k1, .}
  double2 *red = vr + nk * nv;   // [nk * nc][nout] partial sums
  for (int idx = threadIdx.x; idx < nkr * n; idx += blockDim.x) {
    int k1 = k1a + idx / n - m, k2 = idx % n - m;
    const bool neg = k2 < 0 || (k2 == 0 && k1 < 0);  // canonical half (exactly Hermitian, see above)
    if (neg) {
      k1 = -k1;
      k2 = -k2;
    }
    const int64_t q = (int64_t)(k1 + m) * (m + 1) + k2;
    const double2 pp = p[q];
    const double dq = Dh[q];
    u[idx] = make_double2(dq * pp.x, neg ? -dq * pp.y : dq * pp.y);
  }
  for (int idx = threadIdx.x; idx < nkr * nv; idx += blockDim.x) {
    const int k1 = k1a + idx / nv - m, sc = idx % nv;
    vr[idx] = vfull[(int64_t)(j1 - k1 + 2 * m) * nv + sc];
  }
  for (int idx = threadIdx.x; idx < nk * nc * nout; idx += blockDim.x) red[idx] = make_double2(0.0, 0.0);
  __syncthreads();
  const int t = threadIdx.x, g4 = t % ngrp, kk = (t / ngrp) % nk, c = t / (ngrp * nk), j2b = 4 * g4;
  if (c < nc && kk < nkr) {
    const int c2a = c * clen, c2b = min(n, c2a + clen);
    double re[4] = {0.0, 0.0, 0.0, 0.0}, im[4] = {0.0, 0.0, 0.0, 0.0};
    const double2 *ur = u + kk * n, *vrow = vr + kk * nv;
    double2 w[4];  // v_{j1-k1, j2b+o - k2} at k2 = c2a - m: index j2b + o - c2a + 3m
#pragma unroll
    for (int o = 0; o < 4; ++o) w[o] = (j2b + o <= m && c2a < c2b) ? vrow[j2b + o - c2a + 3 * m] : make_double2(0.0, 0.0);
    for (int c2 = c2a; c2 < c2b; ++c2) {
      const double2 b = ur[c2];
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        re[o] = fma(w[o].x, b.x, fma(-w[o].y, b.y, re[o]));
        im[o] = fma(w[o].x, b.y, fma(w[o].y, b.x, im[o]));
      }
#pragma unroll
      for (int o = 3; o > 0; --o) w[o] = w[o - 1];
      w[0] = (c2 + 1 < c2b) ? vrow[j2b - (c2 + 1) + 3 * m] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int o = 0; o < 4; ++o)
      if (j2b + o <= m) red[(kk * nc + c) * nout + j2b + o] = make_double2(re[o], im[o]);
  }
  __syncthreads();
  if (t < nout) {
    double2 o = make_double2(0.0, 0.0);
    for (int k = 0; k < nk * nc; ++k) {
      o.x += red[k * nout + t].x;
      o.y += red[k * nout + t].y;
    }
    tpart[((int64_t)row * kToepSplits + spl) * nout + t] = o;
  }
  __threadfence();
  __syncthreads();
  if (t == 0) last_s = atomicAdd(tcnt + row, 1u) == kToepSplits - 1;
  __syncthreads();
  if (!last_s) return;
  __threadfence();  // the other splits' partials of this row are visible
  double acc = 0.0;
  if (t < nout && !(t == 0 && j1 < 0)) {  // (j1 < 0, 0) is written by row -j1 as the conjugate
    double2 o = make_double2(0.0, 0.0);
    for (int k = 0; k < kToepSplits; ++k) {
      const double2 v = __ldcg(tpart + ((int64_t)row * kToepSplits + k) * nout + t);
      o.x += v.x;
      o.y += v.y;
    }
    const int64_t q = (int64_t)(j1 + m) * (m + 1) + t;
    const double2 pp = p[q];
    const double dq = Dh[q], s2 = st->sigma2;
    double2 a = make_double2(dq * o.x + s2 * pp.x, dq * o.y + s2 * pp.y);
    if (t == 0 && j1 == 0) a.y = s2 * pp.y;  // j = 0: (T u)_0 is real
    Ap[q] = a;
    acc = (t ? 2.0 : 1.0) * (pp.x * a.x + pp.y * a.y);
    if (t == 0 && j1 > 0) {  // the mirrored entry (-j1, 0) = conj, with the canonical p
      Ap[(int64_t)(m - j1) * (m + 1)] = make_double2(a.x, -a.y);
      acc *= 2.0;
    }
  }
  acc = block_sum(acc, sh);
  if (t == 0) {
    part[row] = acc;
    tcnt[row] = 0;  // for the next product
  }
}

static size_t toep2s_smem(int m) {
  const int n = 2 * m + 1, nv = 4 * m + 1, nout = m + 1, ngrp = (nout + 3) / 4, nk = toeps_rows_per_split(n);
  const int nc = kToepSThreads / (ngrp * nk);
  return sizeof(double2) * ((size_t)nk * n + (size_t)nk * nv + (size_t)nk * nc * nout);
}
static bool toep_split() {
  const char *e = getenv("EFGP_TOEP_SPLIT");
  return !(e && e[0] == '0');
}


// ---- fused direct CG (2D, small m): two kernels per iteration instead of three -----------------
// Iteration j (slot q = j & 1; the graph captures an even number of iterations, so the slot of a
// captured iteration is fixed):
//   k_cg_toep2f: rr_j = ||r_j||^2 from the previous k_cg_xr2's partials (redundantly in every CTA, same
//                order), stop test (hist, done), beta = rr_j / rr_{j-1}, p_j = r_j + beta p_{j-1} formed on
//                the fly from (r, p slot 1-q) and written to p slot q, then A p_j as k_cg_toep2s;
//   k_cg_xr2   : alpha = rr_j / <p_j, A p_j>, x += alpha p_j, r -= alpha A p_j, ||r_{j+1}||^2 partials.
// Same recurrences and stopping rule as k_cg_xr + k_cg_p (reading G6); one launch (~4-5 us of
// dependency latency) fewer per iteration.
__global__ void __launch_bounds__(kToepSThreads) k_cg_toep2f(
    const double2 *__restrict__ vfull, const double2 *__restrict__ r, const double2 *__restrict__ p_old,
    double2 *__restrict__ p_new, const double *__restrict__ Dh, double2 *__restrict__ Ap, int m, CGState *st,
    double2 *__restrict__ tpart, unsigned *__restrict__ tcnt, double *__restrict__ part_pAp,
    const double *__restrict__ part_rr, int nblk, double *__restrict__ hist, int q) {
  extern __shared__ double2 tsm[];
  __shared__ double sh[40];
  __shared__ bool last_s;
  pdl_wait();
  pdl_trigger();
  if (st->done) return;
  const long long it = st->iter;
  double beta = 0.0;
  if (it > 0) {
    const double rr = reduce_partials(part_rr, nblk, sh);
    beta = rr / st->rrs[q ^ 1];
    const double rel = sqrt(rr) / st->bnorm;
    const int stop = rel <= st->tol ? 1 : (it >= st->max_iter ? 2 : 0);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->rrs[q] = rr;
      st->rr = rr;
      hist[it] = rel;
      if (stop) st->done = stop;
    }
    if (stop) return;
  }
  const int n = 2 * m + 1, nv = 4 * m + 1, nout = m + 1, ngrp = (nout + 3) / 4;
  const int row = (int)blockIdx.x % n, spl = (int)blockIdx.x / n, j1 = row - m;
  const int nk = toeps_rows_per_split(n), k1a = spl * nk, k1b = min(n, k1a + nk), nkr = k1b - k1a;
  const int nc = kToepSThreads / (ngrp * nk), clen = (n + nc - 1) / nc;
  double2 *u = tsm, *vr = u + nk * n, *red = vr + nk * nv;
  for (int idx = threadIdx.x; idx < nkr * n; idx += blockDim.x) {
    int k1 = k1a + idx / n - m, k2 = idx % n - m;
    const bool neg = k2 < 0 || (k2 == 0 && k1 < 0);
    if (neg) {
      k1 = -k1;
      k2 = -k2;
    }
    const int64_t qq = (int64_t)(k1 + m) * (m + 1) + k2;
    const double2 rq = r[qq], po = p_old[qq];
    const double2 pp = make_double2(rq.x + beta * po.x, rq.y + beta * po.y);
    const double dq = Dh[qq];
    u[idx] = make_double2(dq * pp.x, neg ? -dq * pp.y : dq * pp.y);
  }
  if (row == 0)  // p_j of this split's stored rows (every stored entry exactly once over the splits)
    for (int idx = threadIdx.x; idx < nkr * (m + 1); idx += blockDim.x) {
      const int64_t qq = (int64_t)k1a * (m + 1) + idx;
      const double2 rq = r[qq], po = p_old[qq];
      p_new[qq] = make_double2(rq.x + beta * po.x, rq.y + beta * po.y);
    }
  for (int idx = threadIdx.x; idx < nkr * nv; idx += blockDim.x) {
    const int k1 = k1a + idx / nv - m, sc = idx % nv;
    vr[idx] = vfull[(int64_t)(j1 - k1 + 2 * m) * nv + sc];
  }
  for (int idx = threadIdx.x; idx < nk * nc * nout; idx += blockDim.x) red[idx] = make_double2(0.0, 0.0);
  __syncthreads();
  const int t = threadIdx.x, g4 = t % ngrp, kk = (t / ngrp) % nk, c = t / (ngrp * nk), j2b = 4 * g4;
  if (c < nc && kk < nkr) {
    const int c2a = c * clen, c2b = min(n, c2a + clen);
    double re[4] = {0.0, 0.0, 0.0, 0.0}, im[4] = {0.0, 0.0, 0.0, 0.0};
    const double2 *ur = u + kk * n, *vrow = vr + kk * nv;
    double2 w[4];
#pragma unroll
    for (int o = 0; o < 4; ++o) w[o] = (j2b + o <= m && c2a < c2b) ? vrow[j2b + o - c2a + 3 * m] : make_double2(0.0, 0.0);
    for (int c2 = c2a; c2 < c2b; ++c2) {
      const double2 b = ur[c2];
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        re[o] = fma(w[o].x, b.x, fma(-w[o].y, b.y, re[o]));
        im[o] = fma(w[o].x, b.y, fma(w[o].y, b.x, im[o]));
      }
#pragma unroll
      for (int o = 3; o > 0; --o) w[o] = w[o - 1];
      w[0] = (c2 + 1 < c2b) ? vrow[j2b - (c2 + 1) + 3 * m] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int o = 0; o < 4; ++o)
      if (j2b + o <= m) red[(kk * nc + c) * nout + j2b + o] = make_double2(re[o], im[o]);
  }
  __syncthreads();
  if (t < nout) {
    double2 o = make_double2(0.0, 0.0);
    for (int k = 0; k < nk * nc; ++k) {
      o.x += red[k * nout + t].x;
      o.y += red[k * nout + t].y;
    }
    tpart[((int64_t)row * kToepSplits + spl) * nout + t] = o;
  }
  __threadfence();
  __syncthreads();
  if (t == 0) last_s = atomicAdd(tcnt + row, 1u) == kToepSplits - 1;
  __syncthreads();
  if (!last_s) return;
  __threadfence();
  double acc = 0.0;
  if (t < nout && !(t == 0 && j1 < 0)) {
    double2 o = make_double2(0.0, 0.0);
    for (int k = 0; k < kToepSplits; ++k) {
      const double2 v = __ldcg(tpart + ((int64_t)row * kToepSplits + k) * nout + t);
      o.x += v.x;
      o.y += v.y;
    }
    const int64_t qq = (int64_t)(j1 + m) * (m + 1) + t;
    const double2 rq = r[qq], po = p_old[qq];
    const double2 pp = make_double2(rq.x + beta * po.x, rq.y + beta * po.y);
    const double dq = Dh[qq], s2 = st->sigma2;
    double2 a = make_double2(dq * o.x + s2 * pp.x, dq * o.y + s2 * pp.y);
    if (t == 0 && j1 == 0) a.y = s2 * pp.y;
    Ap[qq] = a;
    acc = (t ? 2.0 : 1.0) * (pp.x * a.x + pp.y * a.y);
    if (t == 0 && j1 > 0) {
      Ap[(int64_t)(m - j1) * (m + 1)] = make_double2(a.x, -a.y);
      acc *= 2.0;
    }
  }
  acc = block_sum(acc, sh);
  if (t == 0) {
    part_pAp[row] = acc;
    tcnt[row] = 0;
  }
}

__global__ void k_cg_xr2(double2 *__restrict__ x, double2 *__restrict__ r, const double2 *__restrict__ p,
                         const double2 *__restrict__ Ap, int64_t Mh, int m, CGState *st,
                         const double *__restrict__ part_pAp, int nrow, double *__restrict__ part_rr, int q) {
  __shared__ double sh[40];
  pdl_wait();
  pdl_trigger();
  if (st->done) return;
  const double alpha = st->rrs[q] / reduce_partials(part_pAp, nrow, sh);
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < Mh; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 pp = p[i], a = Ap[i];
    double2 xx = x[i], rq = r[i];
    xx.x += alpha * pp.x;
    xx.y += alpha * pp.y;
    rq.x -= alpha * a.x;
    rq.y -= alpha * a.y;
    x[i] = xx;
    r[i] = rq;
    acc += ((i % (m + 1)) ? 2.0 : 1.0) * (rq.x * rq.x + rq.y * rq.y);
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) {
    part_rr[blockIdx.x] = acc;
    if (blockIdx.x == 0) st->iter = st->iter + 1;
  }
}

// ---- persistent direct CG (2D, small m: c3, c5) ------------------------------------------------
// The whole CG loop of the direct path (same recurrences and stopping rule as k_cg_xr + k_cg_p,
// reading G6) as ONE cooperative kernel with ONE grid barrier per iteration:
//   phase 1: p_j = r_j + beta_j p_{j-1}, then the split direct product A p_j (CTA (row, split); the
//            last CTA of a row adds the row's splits in fixed order, applies D and sigma^2 and writes
//            the row's <p, Ap> partial);
//   grid barrier;
//   phase 2: alpha = rr_j / <p_j, A p_j>, r_{j+1} = r_j - alpha A p_j and ||r_{j+1}||^2, beta_{j+1},
//            the stop test.
// The M_h-entry vectors r and p are small (21 KB each for c5), so EVERY CTA keeps its own copy in
// shared memory and updates all of it in phase 2 from the exchanged A p_j: the sums of phase 2 are
// formed in the same fixed order in every CTA, so all CTAs hold bitwise-equal r, p, rr and take the
// same stop decision, and the second grid-wide reduction of the launched path (||r||^2 before
// beta) needs no barrier.  Only A p_j and the <p, Ap> row partials cross CTAs; they are
// double-buffered by iteration parity (a CTA can be at most one phase ahead of the slowest: the
// barrier of iteration j+1 waits for everyone's phase 2 of iteration j).  x is updated by the CTA
// that owns each entry.  The v rows a CTA convolves with are staged once for all iterations.
// Data written by other CTAs is read with ld.global.cg (L2), never through the non-coherent paths.
__device__ __forceinline__ unsigned ld_acq_gpu(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct PersistGeom {  // CTA (row, split) of the persistent direct CG; nsplit is a launch parameter
  int n, nv, nout, ngrp, nk, nc, Mh;
  __host__ __device__ PersistGeom(int m, int nsplit, int threads) {
    n = 2 * m + 1;
    nv = 4 * m + 1;
    nout = m + 1;
    ngrp = (nout + 3) / 4;
    nk = (n + nsplit - 1) / nsplit;
    nc = threads / (ngrp * nk);
    Mh = n * nout;
  }
  __host__ __device__ bool ok() const { return nc >= 1; }  // every (output group, k1 row) has a thread
  __host__ __device__ size_t smem() const {
    return sizeof(double2) * ((size_t)nk * n + (size_t)nk * nv + (size_t)nk * nc * nout + 2 * (size_t)Mh);
  }
};
constexpr int kPersistThreads = 256;
constexpr int kPersistPer = 9;  // M_h entries per thread in phase 2: M_h <= 9 x 256 covers m <= 32
constexpr int kPersistU = 3;    // u entries per thread (nk (2m+1) <= 3 x 256: checked at launch)

__global__ void __launch_bounds__(kPersistThreads, 2) k_cg_toep2_persist(
    const double2 *__restrict__ vfull, const double *__restrict__ Dh, double2 *x, double2 *r, double2 *p0,
    double2 *ap0, double2 *ap1, int m, int nsplit, CGState *st, double2 *tpart, unsigned *tcnt, double *part_pAp,
    double *hist, unsigned *gbar, long long *trace, const double2 *vh0) {
  // vh0 != nullptr: Jacobi PCG (reading G12b, NEXT-4): z = r / (D^2 v_0 + sigma^2), p = z + beta p with
  // beta = (r, z)_new / (r, z), alpha = (r, z) / (p, Ap); the stop test stays on ||r|| (as pcg_solve)
  extern __shared__ double2 tsm[];
  __shared__ double sh[40];
  __shared__ bool last_s;
  // optional phase timing (EFGP_CG_TRACE): clock64 cycles per phase, thread 0, summed over iterations
  long long tr_acc[6] = {0, 0, 0, 0, 0, 0}, tr_t = clock64();
#define TR(i)                       \
  if (trace && threadIdx.x == 0) {  \
    const long long t_ = clock64(); \
    tr_acc[(i)] += t_ - tr_t;       \
    tr_t = t_;                      \
  }
  const PersistGeom G(m, nsplit, kPersistThreads);
  const int n = G.n, nv = G.nv, nout = G.nout, ngrp = G.ngrp, nk = G.nk, nc = G.nc, Mh = G.Mh;
  const int row = (int)blockIdx.x % n, spl = (int)blockIdx.x / n, j1 = row - m;
  const int k1a = min(n, spl * nk), k1b = min(n, k1a + nk), nkr = k1b - k1a;
  const int clen = (n + nc - 1) / nc;
  double2 *u = tsm, *vr = u + nk * n, *red = vr + nk * nv, *rs = red + nk * nc * nout, *ps = rs + Mh;
  for (int idx = threadIdx.x; idx < nkr * nv; idx += blockDim.x) {  // once for all iterations
    const int k1 = k1a + idx / nv - m, sc = idx % nv;
    vr[idx] = vfull[(int64_t)(j1 - k1 + 2 * m) * nv + sc];
  }
  for (int i = threadIdx.x; i < Mh; i += blockDim.x) rs[i] = ps[i] = r[i];  // r_0 = b (k_cg_init)
  const int t = threadIdx.x, g4 = t % ngrp, kk = (t / ngrp) % nk, c = t / (ngrp * nk), j2b = 4 * g4;
  const double tol = st->tol, bnorm = st->bnorm, s2 = st->sigma2;
  const long long max_iter = st->max_iter;
  long long it = st->iter;
  if (st->done) return;  // (rr = 0: decided by k_cg_init2, the same in every CTA)
  double rr = st->rrs[0], beta = 0.0;
  unsigned target = 0;
  const int own_lo = (int)blockIdx.x * kPersistThreads, own_hi = min(Mh, own_lo + kPersistThreads);
  const bool jac = vh0 != nullptr;
  const double v0 = jac ? vh0->x : 0.0;
  auto inv_diag = [&](int i) { const double d = Dh[i]; return 1.0 / (d * d * v0 + s2); };
  double rz = 0.0;  // Jacobi: (r, z), the same fixed-order sum in every CTA
  if (jac) {
    double a = 0.0;
    for (int i = threadIdx.x; i < Mh; i += blockDim.x) {
      const double2 rq = rs[i];
      a += ((i % (m + 1)) ? 2.0 : 1.0) * (rq.x * rq.x + rq.y * rq.y) * inv_diag(i);
    }
    a = block_sum(a, sh);
    if (threadIdx.x == 0) sh[34] = a;
    __syncthreads();
    rz = sh[34];
  }
  // this thread's entries of u = D p on the split's k1 rows, fixed for all iterations: the stored
  // (canonical-half) index << 1 | conjugate flag, and D (-1: no entry)
  int uq[kPersistU];
  double ud[kPersistU];
#pragma unroll
  for (int k = 0; k < kPersistU; ++k) {
    const int idx = threadIdx.x + k * kPersistThreads;
    uq[k] = -1;
    ud[k] = 0.0;
    if (idx < nkr * n) {
      int k1 = k1a + idx / n - m, k2 = idx % n - m;
      const bool neg = k2 < 0 || (k2 == 0 && k1 < 0);
      if (neg) {
        k1 = -k1;
        k2 = -k2;
      }
      const int qq = (k1 + m) * (m + 1) + k2;
      uq[k] = qq << 1 | (neg ? 1 : 0);
      ud[k] = Dh[qq];
    }
  }
  __shared__ double2 xs[kPersistThreads];
  xs[t] = own_lo + t < own_hi ? x[own_lo + t] : make_double2(0.0, 0.0);
  __syncthreads();
  for (;;) {
    const int q = (int)(it & 1);
    double2 *Ap = q ? ap1 : ap0;
    double *pAp = part_pAp + q * n;
    // phase 1: p_j (all entries, every CTA), u = D p_j on this split's k1 rows (canonical half:
    // exactly Hermitian, see k_cg_toep2), the product
    for (int i = threadIdx.x; i < Mh; i += blockDim.x) {
      double2 rq = rs[i];
      if (jac) {
        const double w = inv_diag(i);
        rq = make_double2(rq.x * w, rq.y * w);  // z = M^-1 r
      }
      const double2 po = ps[i];
      ps[i] = make_double2(rq.x + beta * po.x, rq.y + beta * po.y);
    }
    for (int idx = threadIdx.x; idx < nk * nc * nout; idx += blockDim.x) red[idx] = make_double2(0.0, 0.0);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPersistU; ++k)
      if (uq[k] >= 0) {
        const int idx = threadIdx.x + k * kPersistThreads;
        const double2 pp = ps[uq[k] >> 1];
        u[idx] = make_double2(ud[k] * pp.x, (uq[k] & 1) ? -ud[k] * pp.y : ud[k] * pp.y);
      }
    __syncthreads();
    TR(0);
    if (c < nc && kk < nkr) {
      const int c2a = c * clen, c2b = min(n, c2a + clen);
      double re[4] = {0.0, 0.0, 0.0, 0.0}, im[4] = {0.0, 0.0, 0.0, 0.0};
      const double2 *ur = u + kk * n, *vrow = vr + kk * nv;
      double2 w[4];
#pragma unroll
      for (int o = 0; o < 4; ++o)
        w[o] = (j2b + o <= m && c2a < c2b) ? vrow[j2b + o - c2a + 3 * m] : make_double2(0.0, 0.0);
      for (int c2 = c2a; c2 < c2b; ++c2) {
        const double2 b = ur[c2];
#pragma unroll
        for (int o = 0; o < 4; ++o) {
          re[o] = fma(w[o].x, b.x, fma(-w[o].y, b.y, re[o]));
          im[o] = fma(w[o].x, b.y, fma(w[o].y, b.x, im[o]));
        }
#pragma unroll
        for (int o = 3; o > 0; --o) w[o] = w[o - 1];
        w[0] = (c2 + 1 < c2b) ? vrow[j2b - (c2 + 1) + 3 * m] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int o = 0; o < 4; ++o)
        if (j2b + o <= m) red[(kk * nc + c) * nout + j2b + o] = make_double2(re[o], im[o]);
    }
    __syncthreads();
    {  // the nk nc partial rows of this CTA, in two fixed-order stages (u is free: it holds them)
      const int spl2 = min(kPersistThreads / nout, nk * n / nout), np = nk * nc;
      if (t < spl2 * nout) {
        const int o = t % nout, g = t / nout;
        double2 a = make_double2(0.0, 0.0);
        for (int k = g; k < np; k += spl2) {
          a.x += red[k * nout + o].x;
          a.y += red[k * nout + o].y;
        }
        u[g * nout + o] = a;
      }
      __syncthreads();
      if (t < nout) {
        double2 o = make_double2(0.0, 0.0);
        for (int g = 0; g < spl2; ++g) {
          o.x += u[g * nout + t].x;
          o.y += u[g * nout + t].y;
        }
        tpart[((int64_t)row * nsplit + spl) * nout + t] = o;
      }
    }
    TR(1);
    __threadfence();
    __syncthreads();
    if (t == 0) last_s = atomicAdd(tcnt + row, 1u) == (unsigned)nsplit - 1;
    __syncthreads();
    TR(2);
    if (last_s) {
      __threadfence();
      double acc = 0.0;
      if (t < nout && !(t == 0 && j1 < 0)) {  // (j1 < 0, 0) is written by row -j1 as the conjugate
        double2 tv[kToepSplitsHost];  // all loads first, then the fixed-order sum
#pragma unroll
        for (int k = 0; k < kToepSplitsHost; ++k)
          tv[k] = k < nsplit ? __ldcg(tpart + ((int64_t)row * nsplit + k) * nout + t) : make_double2(0.0, 0.0);
        double2 o = make_double2(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < kToepSplitsHost; ++k) {
          o.x += tv[k].x;
          o.y += tv[k].y;
        }
        const int qq = (j1 + m) * (m + 1) + t;
        const double2 pp = ps[qq];
        const double dq = Dh[qq];
        double2 a = make_double2(dq * o.x + s2 * pp.x, dq * o.y + s2 * pp.y);
        if (t == 0 && j1 == 0) a.y = s2 * pp.y;  // j = 0: (T u)_0 is real
        Ap[qq] = a;
        acc = (t ? 2.0 : 1.0) * (pp.x * a.x + pp.y * a.y);
        if (t == 0 && j1 > 0) {  // the mirrored entry (-j1, 0) = conj, with the canonical p
          Ap[(m - j1) * (m + 1)] = make_double2(a.x, -a.y);
          acc *= 2.0;
        }
      }
      acc = block_sum(acc, sh);
      if (t == 0) {
        pAp[row] = acc;
        tcnt[row] = 0;  // for the next product
        __threadfence();
        atomicAdd(gbar, 1u);  // the row is complete (arrivals: one per row, 2m+1 per iteration)
      }
    }
    TR(3);
    // grid barrier: every row's A p_j and <p, Ap> partial are written
    target += n;
    if (t == 0)
      while (ld_acq_gpu(gbar) < target) {
      }
    __syncthreads();
    TR(4);
    // phase 2 (every CTA, the same fixed order): alpha, x (owned entries), r and ||r||^2, beta, stop.
    // Every load of the phase is issued before the first use (A p_j entries in registers)
    double2 av[kPersistPer];
#pragma unroll
    for (int k = 0; k < kPersistPer; ++k) {
      const int i = t + k * kPersistThreads;
      av[k] = i < Mh ? __ldcg(Ap + i) : make_double2(0.0, 0.0);
    }
    double v = t < n ? __ldcg(pAp + t) : 0.0;
    v = block_sum(v, sh);
    if (threadIdx.x == 0) sh[32] = v;
    __syncthreads();
    const double alpha = (jac ? rz : rr) / sh[32];
    double acc = 0.0, accz = 0.0;
#pragma unroll
    for (int k = 0; k < kPersistPer; ++k) {
      const int i = t + k * kPersistThreads;
      if (i < Mh) {
        const double2 a = av[k], pp = ps[i];
        double2 rq = rs[i];
        rq.x -= alpha * a.x;
        rq.y -= alpha * a.y;
        rs[i] = rq;
        const double e = ((i % (m + 1)) ? 2.0 : 1.0) * (rq.x * rq.x + rq.y * rq.y);
        acc += e;
        if (jac) accz += e * inv_diag(i);
        if (i >= own_lo && i < own_hi) {  // x of the owned entries lives in shared memory until the end
          xs[t].x += alpha * pp.x;
          xs[t].y += alpha * pp.y;
        }
      }
    }
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) sh[33] = acc;
    __syncthreads();
    const double rr_new = sh[33];
    if (jac) {
      accz = block_sum(accz, sh);
      if (threadIdx.x == 0) sh[35] = accz;
      __syncthreads();
      const double rz_new = sh[35];
      beta = rz_new / rz;
      rz = rz_new;
    }
    TR(5);
    ++it;
    if (!jac) beta = rr_new / rr;
    const double rr_prev = rr;
    rr = rr_new;
    const double rel = sqrt(rr_new) / bnorm;
    const int stop = rel <= tol ? 1 : (it >= max_iter ? 2 : 0);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->rr = rr_new;
      st->rr_old = rr_prev;
      st->rrs[it & 1] = rr_new;
      st->iter = it;
      hist[it] = rel;
      if (stop) st->done = stop;
    }
    if (stop) {  // x (owned entries), r and p to global memory
      if (trace && t == 0)
        for (int k = 0; k < 6; ++k) trace[(size_t)blockIdx.x * 8 + k] = tr_acc[k];
      if (trace && t == 0) trace[(size_t)blockIdx.x * 8 + 6] = last_s ? 1 : 0;
      if (own_lo + t < own_hi) {
        const int i = own_lo + t;
        x[i] = xs[t];
        r[i] = rs[i];
        p0[i] = ps[i];
      }
      return;
    }
    __syncthreads();  // sh[32], sh[33] reusable
  }
}
#undef TR

// ---- persistent DFT CG (2D beyond the direct product: c2, m = 49) ------------------------------
// The Toeplitz product out_j = sum_k v_{j-k} u_k (u = D p, j, k in J_m^2) with a DFT of length L
// (>= 4m+1, the Toeplitz box) along the second axis and a direct convolution along the first:
//   T[k1][x2]  = sum_{k2} u_{k1,k2} w^(-k2 x2)                                   (w = e^(2 pi i / L))
//   W[j1][x2]  = sum_{k1} Vt[j1-k1][x2] T[k1][x2],   Vt[d1][x2] = sum_{d2} v_{d1,d2} w^(-d2 x2)
//   out_{j1,j2} = (1/L) sum_{x2} w^(j2 x2) W[j1][x2]                                 (j2 = 0..m)
// exact because |j2 - k2 - d2| < L for every term that survives (L >= 4m+1): (1/L) sum_x2 Vt[d1][x2]
// w^((j2-k2) x2) = v_{d1, j2-k2}.  4.9e6 complex MACs per product for c2 against 4.9e7 for the direct
// sum and four cuFFT launches for the padded real FFTs (Alg a:FF).
// One cooperative kernel runs the whole CG (recurrences and stopping rule of k_cg_xr + k_cg_p,
// reading G6), two grid barriers per iteration:
//   phase 1 (CTA c owns the columns x2 in [c L / G, (c+1) L / G)): p_j = r_j + beta p_{j-1} (all
//            entries), T and W of its columns, W to global memory; barrier;
//   phase 2 (CTA c < 2m+1 owns row j1 = c - m): out of its row from W, A p_j = D out + sigma^2 p_j
//            (exactly Hermitian in the j2 = 0 column, as k_cg_toep2), its <p, Ap> partial; barrier;
//   phase 3 (every CTA, the same fixed order): alpha, r_{j+1} and ||r_{j+1}||^2 for ALL entries
//            (r, p, D in every CTA's shared memory), beta, the stop test; x of the owned entries.
// W, A p and the partials need no double buffer: a CTA passes the barrier of a phase only after
// every CTA has finished the phase that reads what it is about to overwrite.
constexpr int kDftThreads = 256, kDftCols = 2;  // columns per CTA: L <= kDftCols x grid
constexpr int kDftPer = kDft2MaxMh / kDftThreads + 1;  // A p entries per thread in phase 3
struct DftGeom {
  int n, nv, nout, Mh, L, G;
  __host__ __device__ DftGeom(int m, int L_, int G_) : n(2 * m + 1), nv(4 * m + 1), nout(m + 1), Mh(n * (m + 1)), L(L_), G(G_) {}
  __host__ __device__ size_t smem() const {
    const size_t opn = 8 * (size_t)nout > 2 * (size_t)n * kDftCols ? 8 * (size_t)nout : 2 * (size_t)n * kDftCols;
    return sizeof(double2) * (2 * (size_t)Mh + (size_t)kDftCols * nv + (size_t)kDftCols * n + L + L + opn) +
           sizeof(double) * (size_t)Mh;
  }
};

__global__ void __launch_bounds__(kDftThreads, 1) k_cg_dft2_persist(
    const double2 *__restrict__ Vt, const double2 *__restrict__ roots, const double *__restrict__ Dh, double2 *x,
    double2 *r, double2 *p0, double2 *Ap, double2 *Wg, int m, int L, CGState *st, double *part_pAp, double *hist,
    unsigned *gbar, long long *trace, const double2 *vh0) {
  // vh0 != nullptr: Jacobi PCG (reading G12b), as k_cg_toep2_persist
  extern __shared__ __align__(16) double2 dsm[];
  __shared__ double sh[40];
  // optional phase timing (EFGP_CG_TRACE), thread 0, cycles summed over iterations: 0 p + T, 2 W,
  // 1 barrier 1, 4 phase 2, 5 barrier 2, 3 fence after W + phase 3
  long long tr_acc[6] = {0, 0, 0, 0, 0, 0}, tr_t = clock64();
#define TRD(i)                      \
  if (trace && threadIdx.x == 0) {  \
    const long long t_ = clock64(); \
    tr_acc[(i)] += t_ - tr_t;       \
    tr_t = t_;                      \
  }
  const DftGeom Gm(m, L, (int)gridDim.x);
  const int n = Gm.n, nv = Gm.nv, nout = Gm.nout, Mh = Gm.Mh, t = threadIdx.x;
  // r, p and D live in shared memory in k2-major order s(k1, k2) = k2 n + (k1 + m) (the global
  // half is row-major g(k1, k2) = (k1 + m)(m + 1) + k2): the T sums read p and D of consecutive k1 in
  // consecutive lanes (row-major: a 800-byte lane stride, 8-way bank conflicts, the kernel's limit)
  double2 *rs = dsm, *ps = rs + Mh, *vs = ps + Mh, *ts = vs + kDftCols * nv, *wr = ts + kDftCols * n,
          *rt = wr + L, *op = rt + L;
  double *ds = reinterpret_cast<double *>(op + (8 * nout > 2 * n * kDftCols ? 8 * nout : 2 * n * kDftCols));
  auto gidx = [&](int si) { return (si % n) * nout + si / n; };
  const int c0 = (int)((int64_t)blockIdx.x * L / gridDim.x), c1 = (int)((int64_t)(blockIdx.x + 1) * L / gridDim.x);
  const int nx = c1 - c0;  // <= kDftCols (checked at launch)
  for (int i = t; i < Mh; i += kDftThreads) {
    const int g = gidx(i);
    rs[i] = ps[i] = r[g];  // r_0 = b (k_cg_init)
    ds[i] = Dh[g];
  }
  for (int i = t; i < nx * nv; i += kDftThreads) vs[i] = Vt[(int64_t)(i % nv) * L + c0 + i / nv];  // [col][d1 + 2m]
  for (int i = t; i < L; i += kDftThreads) rt[i] = roots[i];
  const int own_lo = (int)((int64_t)blockIdx.x * Mh / gridDim.x), own_hi = (int)((int64_t)(blockIdx.x + 1) * Mh / gridDim.x);
  __shared__ double2 xs[kDftThreads];
  if (own_lo + t < own_hi) xs[t] = x[gidx(own_lo + t)];
  const double tol = st->tol, bnorm = st->bnorm, s2 = st->sigma2;
  const long long max_iter = st->max_iter;
  long long it = st->iter;
  if (st->done) return;
  double rr = st->rrs[0], beta = 0.0;
  unsigned target = 0;
  const double invL = 1.0 / (double)L;
  __syncthreads();
  const bool jac = vh0 != nullptr;
  const double v0 = jac ? vh0->x : 0.0;
  auto inv_diag = [&](int i) { const double d = ds[i]; return 1.0 / (d * d * v0 + s2); };
  double rz = 0.0;  // Jacobi: (r, z) in one fixed order (k2-major), the same in every CTA
  if (jac) {
    double a = 0.0;
    for (int i = t; i < Mh; i += kDftThreads) {
      const double2 rq = rs[i];
      a += (i >= n ? 2.0 : 1.0) * (rq.x * rq.x + rq.y * rq.y) * inv_diag(i);
    }
    a = block_sum(a, sh);
    if (t == 0) sh[34] = a;
    __syncthreads();
    rz = sh[34];
  }
  for (;;) {
    // ---- phase 1: p_j; T and W of this CTA's columns
    for (int i = t; i < Mh; i += kDftThreads) {
      double2 rq = rs[i];
      if (jac) {
        const double w = inv_diag(i);
        rq = make_double2(rq.x * w, rq.y * w);  // z = M^-1 r
      }
      const double2 po = ps[i];
      ps[i] = make_double2(rq.x + beta * po.x, rq.y + beta * po.y);
    }
    __syncthreads();
    // T[k1][x2] = u_{k1,0} + sum_{k2 = 1..m} (u_{k1,k2} w^(-k2 x2) + conj(u_{-k1,k2}) w^(k2 x2)); the
    // (k1 < 0, 0) entry is read as conj(u_{-k1,0}) (canonical half: the product is exactly Hermitian).
    // Thread (k1, half h): k2 in half h of 1..m for BOTH columns of the CTA (the p and D loads serve
    // two independent accumulator chains), the halves added in fixed order below
    const int kh = (m + 1) / 2;  // k2 = 1..kh | kh+1..m
    for (int item = t; item < 2 * n; item += kDftThreads) {
      const int k1 = item % n - m, hf = item / n;
      const int ka = hf ? kh + 1 : 1, kb = hf ? m : kh;
      double tx[kDftCols] = {}, ty[kDftCols] = {};
      int e[kDftCols];
#pragma unroll
      for (int xi = 0; xi < kDftCols; ++xi) e[xi] = ((ka - 1) * (c0 + xi)) % L;
      for (int k2 = ka; k2 <= kb; ++k2) {
        const int sa = k2 * n + k1 + m, sb = k2 * n - k1 + m;
        const double2 a = ps[sa], b = ps[sb];
        const double da = ds[sa], db = ds[sb];
        const double2 ua = make_double2(da * a.x, da * a.y), ub = make_double2(db * b.x, db * b.y);
        const double c1x = ua.x + ub.x, c1y = ua.y + ub.y, c2x = ua.y - ub.y, c2y = ub.x - ua.x;
#pragma unroll
        for (int xi = 0; xi < kDftCols; ++xi) {
          e[xi] += c0 + xi;
          if (e[xi] >= L) e[xi] -= L;
          const double2 w = rt[e[xi]];  // w^(k2 x2), the same for every lane (broadcast)
          // ua w^-1 + conj(ub) w
          tx[xi] = fma(c1x, w.x, fma(c1y, w.y, tx[xi]));
          ty[xi] = fma(c2x, w.x, fma(c2y, w.y, ty[xi]));
        }
      }
#pragma unroll
      for (int xi = 0; xi < kDftCols; ++xi) op[(hf * n + k1 + m) * kDftCols + xi] = make_double2(tx[xi], ty[xi]);
    }
    __syncthreads();
    for (int item = t; item < n * nx; item += kDftThreads) {
      const int k1 = item / nx - m, xi = item % nx;
      const int q0 = k1 >= 0 ? k1 + m : -k1 + m;  // s(|k1|, 0)
      double2 u0 = make_double2(ds[q0] * ps[q0].x, ds[q0] * ps[q0].y);
      if (k1 < 0) u0.y = -u0.y;
      const double2 h0 = op[(k1 + m) * kDftCols + xi], h1 = op[(n + k1 + m) * kDftCols + xi];
      ts[(k1 + m) * kDftCols + xi] = make_double2(u0.x + h0.x + h1.x, u0.y + h0.y + h1.y);
    }
    __syncthreads();
    TRD(0);
    // W[j1][x2] = sum_{k1} Vt[j1 - k1][x2] T[k1][x2]: thread (j1, half of the k1 range), both columns
    const int k1h = -m + n / 2;  // k1 = -m..k1h-1 | k1h..m
    for (int item = t; item < 2 * n; item += kDftThreads) {
      const int j1 = item % n - m, hf = item / n;
      const int ka = hf ? k1h : -m, kb = hf ? m + 1 : k1h;
      double wx[kDftCols] = {}, wy[kDftCols] = {};
      for (int k1 = ka; k1 < kb; ++k1) {
#pragma unroll
        for (int xi = 0; xi < kDftCols; ++xi) {
          if (xi < nx) {
            const double2 a = vs[xi * nv + j1 - k1 + 2 * m], b = ts[(k1 + m) * kDftCols + xi];
            wx[xi] = fma(a.x, b.x, fma(-a.y, b.y, wx[xi]));
            wy[xi] = fma(a.x, b.y, fma(a.y, b.x, wy[xi]));
          }
        }
      }
#pragma unroll
      for (int xi = 0; xi < kDftCols; ++xi) op[(hf * n + j1 + m) * kDftCols + xi] = make_double2(wx[xi], wy[xi]);
    }
    __syncthreads();
    for (int item = t; item < n * nx; item += kDftThreads) {
      const int j1 = item / nx - m, xi = item % nx;
      const double2 h0 = op[(j1 + m) * kDftCols + xi], h1 = op[(n + j1 + m) * kDftCols + xi];
      Wg[(int64_t)(j1 + m) * L + c0 + xi] = make_double2(h0.x + h1.x, h0.y + h1.y);
    }
    __syncthreads();
    TRD(2);
    __threadfence();
    __syncthreads();
    TRD(3);
    target += gridDim.x;
    if (t == 0) {
      atomicAdd(gbar, 1u);
      while (ld_acq_gpu(gbar) < target) {
      }
    }
    __syncthreads();
    TRD(1);
    // ---- phase 2: row j1 = blockIdx - m
    if ((int)blockIdx.x < n) {
      const int j1 = (int)blockIdx.x - m;
      for (int i = t; i < L; i += kDftThreads) wr[i] = __ldcg(Wg + (int64_t)(j1 + m) * L + i);
      __syncthreads();
      // out[j2] = (1/L) sum_x2 w^(j2 x2) W[x2]: 8 x2-slices per j2, partials summed in fixed order;
      // the twiddle by recurrence (w^(j2 (x2+1)) = w^(j2 x2) w^j2, at most L/8 steps from a table entry)
      for (int item = t; item < 8 * nout; item += kDftThreads) {
        const int j2 = item % nout, sl = item / nout;
        const int xa = (int)((int64_t)sl * L / 8), xb = (int)((int64_t)(sl + 1) * L / 8);
        double ox = 0.0, oy = 0.0;
        double2 w = rt[(j2 * xa) % L];
        const double2 st1 = rt[j2];
        for (int x2 = xa; x2 < xb; ++x2) {
          const double2 a = wr[x2];
          ox = fma(a.x, w.x, fma(-a.y, w.y, ox));
          oy = fma(a.x, w.y, fma(a.y, w.x, oy));
          w = make_double2(w.x * st1.x - w.y * st1.y, w.x * st1.y + w.y * st1.x);
        }
        op[sl * nout + j2] = make_double2(ox, oy);
      }
      __syncthreads();
      double acc = 0.0;
      if (t < nout && !(t == 0 && j1 < 0)) {  // (j1 < 0, 0) is written by row -j1 as the conjugate
        double ox = 0.0, oy = 0.0;
#pragma unroll
        for (int sl = 0; sl < 8; ++sl) {
          ox += op[sl * nout + t].x;
          oy += op[sl * nout + t].y;
        }
        const int sq = t * n + j1 + m;
        const double2 pp = ps[sq];
        const double dq = ds[sq];
        double2 a = make_double2(dq * ox * invL + s2 * pp.x, dq * oy * invL + s2 * pp.y);
        if (t == 0 && j1 == 0) a.y = s2 * pp.y;  // j = 0: (T u)_0 is real
        Ap[sq] = a;  // (A p is exchanged in the k2-major order of the shared copies)
        acc = (t ? 2.0 : 1.0) * (pp.x * a.x + pp.y * a.y);
        if (t == 0 && j1 > 0) {  // the mirrored entry (-j1, 0) = conj, with the canonical p
          Ap[m - j1] = make_double2(a.x, -a.y);
          acc *= 2.0;
        }
      }
      acc = block_sum(acc, sh);
      if (t == 0) {
        part_pAp[blockIdx.x] = acc;
        __threadfence();
        atomicAdd(gbar, 1u);
      }
    }
    TRD(4);
    target += n;
    if (t == 0)
      while (ld_acq_gpu(gbar) < target) {
      }
    __syncthreads();
    TRD(5);
    // ---- phase 3 (every CTA): alpha, r and ||r||^2 (all entries, k2-major order), x (owned entries);
    // all of its L2 loads are issued before the first use (M_h <= kDftPer x 256)
    double acc = 0.0, accz = 0.0;
    double alpha;
    {
      double2 av[kDftPer];
#pragma unroll
      for (int k = 0; k < kDftPer; ++k) {
        const int i = t + k * kDftThreads;
        av[k] = i < Mh ? __ldcg(Ap + i) : make_double2(0.0, 0.0);
      }
      double v = t < n ? __ldcg(part_pAp + t) : 0.0;
      v = block_sum(v, sh);
      if (t == 0) sh[32] = v;
      __syncthreads();
      alpha = (jac ? rz : rr) / sh[32];
#pragma unroll
      for (int k = 0; k < kDftPer; ++k) {
        const int i = t + k * kDftThreads;
        if (i < Mh) {
          double2 rq = rs[i];
          rq.x -= alpha * av[k].x;
          rq.y -= alpha * av[k].y;
          rs[i] = rq;
          const double e = (i >= n ? 2.0 : 1.0) * (rq.x * rq.x + rq.y * rq.y);  // k2 = i / n > 0 weighs 2
          acc += e;
          if (jac) accz += e * inv_diag(i);
          if (i >= own_lo && i < own_hi) {
            xs[i - own_lo].x += alpha * ps[i].x;
            xs[i - own_lo].y += alpha * ps[i].y;
          }
        }
      }
    }
    acc = block_sum(acc, sh);
    if (t == 0) sh[33] = acc;
    __syncthreads();
    const double rr_new = sh[33];
    if (jac) {
      accz = block_sum(accz, sh);
      if (t == 0) sh[35] = accz;
      __syncthreads();
      const double rz_new = sh[35];
      beta = rz_new / rz;
      rz = rz_new;
    }
    TRD(3);
    ++it;
    if (!jac) beta = rr_new / rr;
    const double rr_prev = rr;
    rr = rr_new;
    const double rel = sqrt(rr_new) / bnorm;
    const int stop = rel <= tol ? 1 : (it >= max_iter ? 2 : 0);
    if (blockIdx.x == 0 && t == 0) {
      st->rr = rr_new;
      st->rr_old = rr_prev;
      st->rrs[it & 1] = rr_new;
      st->iter = it;
      hist[it] = rel;
      if (stop) st->done = stop;
    }
    if (stop) {
      for (int i = t; i < Mh; i += kDftThreads) {  // r and p back to global memory (every CTA holds them)
        if (blockIdx.x == 0) {
          r[gidx(i)] = rs[i];
          p0[gidx(i)] = ps[i];
        }
      }
      if (own_lo + t < own_hi) x[gidx(own_lo + t)] = xs[t];
      if (trace && t == 0)
        for (int k = 0; k < 6; ++k) trace[(size_t)blockIdx.x * 8 + k] = tr_acc[k];
      return;
    }
    __syncthreads();
  }
#undef TRD
}

// Vt[d1][x2] = sum_{d2 = -2m..2m} v_{d1,d2} w^(-d2 x2) (once per fit; v full over J_2m, row-major)
__global__ void k_dft2_vt(const double2 *__restrict__ vfull, const double2 *__restrict__ roots, int m, int L,
                          double2 *__restrict__ Vt) {
  const int nv = 4 * m + 1;
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)nv * L) return;
  const int d1 = (int)(id / L), x2 = (int)(id % L);
  double sx = 0.0, sy = 0.0;
  for (int d2 = -2 * m; d2 <= 2 * m; ++d2) {
    int e = (int)((((int64_t)-d2 * x2) % L + L) % L);
    const double2 w = roots[e], a = vfull[(int64_t)d1 * nv + d2 + 2 * m];
    sx = fma(a.x, w.x, fma(-a.y, w.y, sx));
    sy = fma(a.x, w.y, fma(a.y, w.x, sy));
  }
  Vt[id] = make_double2(sx, sy);
}

efgp_status dft2_setup(efgp_plan *pl, cudaStream_t s) {
  const Params &P = pl->P;
  const int m = (int)P.m, L = (int)P.L, nv = 4 * m + 1, n = 2 * m + 1;
  if (!pl->dft_V) {
    EFGP_CUDA(cudaMalloc((void **)&pl->dft_V, sizeof(double2) * (size_t)nv * L));
    EFGP_CUDA(cudaMalloc((void **)&pl->dft_roots, sizeof(double2) * (size_t)L));
    EFGP_CUDA(cudaMalloc((void **)&pl->dft_W, sizeof(double2) * (size_t)n * L));
    std::vector<double2> w(L);
    for (int t = 0; t < L; ++t) {  // w^t = e^(2 pi i t / L), sincospi for exact angles at t/L = k/4
      double sn, cs;
      sincospi(2.0 * t / (double)L, &sn, &cs);
      w[t] = make_double2(cs, sn);
    }
    EFGP_CUDA(cudaMemcpyAsync(pl->dft_roots, w.data(), sizeof(double2) * L, cudaMemcpyHostToDevice, s));
    EFGP_CUDA(cudaStreamSynchronize(s));  // (the host table goes out of scope)
  }
  const int64_t tot = (int64_t)nv * L;
  k_dft2_vt<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(pl->vfull, pl->dft_roots, m, L, pl->dft_V);
  EFGP_CUDA(cudaGetLastError());
  return EFGP_OK;
}

static cudaError_t launch_dft2_cg(efgp_plan *pl, CGState *st, cudaStream_t s, const double2 *vh0 = nullptr) {
  const Params &P = pl->P;
  const int m = (int)P.m, n = 2 * m + 1, L = (int)P.L;
  int dev = 0, coop = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  // as few CTAs as give every CTA kDftCols columns and every row an owner (c2: 100), so phase 1 is
  // balanced (148 CTAs: 52 with two columns, 96 with one, and every CTA waits for the two-column ones)
  const int G = std::min(pl->num_sms, std::max(n, (L + kDftCols - 1) / kDftCols));
  const DftGeom Gm(m, L, G);
  const size_t smem = Gm.smem();
  if (!coop || !pl->dft_V || G < n || (L + G - 1) / G > kDftCols || smem > 220 * 1024 || n > kDftThreads ||
      n > pl->cg_blocks)
    return cudaErrorNotSupported;
  cudaError_t e = cudaFuncSetAttribute(k_cg_dft2_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cg_dft2_persist, kDftThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorNotSupported;
  if (!pl->cg_gbar) {
    e = cudaMalloc((void **)&pl->cg_gbar, sizeof(unsigned));
    if (e != cudaSuccess) return e;
  }
  e = cudaMemsetAsync(pl->cg_gbar, 0, sizeof(unsigned), s);
  if (e != cudaSuccess) return e;
  const double2 *Vt = pl->dft_V, *roots = pl->dft_roots;
  const double *Dh = pl->D_half;
  double2 *x = pl->x, *r = pl->r, *p0 = pl->p, *Ap = pl->Ap, *Wg = pl->dft_W;
  double *part = pl->partials, *hist = pl->hist;
  unsigned *gbar = pl->cg_gbar;
  int mm = m, LL = L;
  long long *trace = nullptr;
  const bool want_trace = getenv("EFGP_CG_TRACE") != nullptr;
  if (want_trace) {
    e = cudaMallocAsync((void **)&trace, sizeof(long long) * 8 * G, s);
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(trace, 0, sizeof(long long) * 8 * G, s);
  }
  void *args[] = {(void *)&Vt, (void *)&roots, (void *)&Dh, (void *)&x, (void *)&r, (void *)&p0, (void *)&Ap,
                  (void *)&Wg, (void *)&mm, (void *)&LL, (void *)&st, (void *)&part, (void *)&hist, (void *)&gbar,
                  (void *)&trace, (void *)&vh0};
  e = cudaLaunchCooperativeKernel((const void *)k_cg_dft2_persist, dim3((unsigned)G), dim3(kDftThreads), args, smem, s);
  if (want_trace && e == cudaSuccess) {
    std::vector<long long> h((size_t)8 * G);
    cudaMemcpyAsync(h.data(), trace, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    CGState hs{};
    cudaMemcpy(&hs, st, sizeof(CGState), cudaMemcpyDeviceToHost);
    double mean[6] = {0, 0, 0, 0, 0, 0};
    for (int b = 0; b < G; ++b)
      for (int k = 0; k < 6; ++k) mean[k] += (double)h[(size_t)b * 8 + k] / G;
    const double it = hs.iter > 0 ? (double)hs.iter : 1.0;
    fprintf(stderr, "cg dft2 trace (cycles/iteration, mean over %d CTAs, %lld iterations): p + T %.0f, W + store %.0f, "
            "barrier 1 %.0f, phase 2 %.0f, barrier 2 %.0f, fence after W + phase 3 %.0f\n", G, hs.iter, mean[0] / it,
            mean[2] / it, mean[1] / it, mean[4] / it, mean[5] / it, mean[3] / it);
    cudaFreeAsync(trace, s);
  }
  return e;
}

// ---- 1D CG in one CTA (c1: m = 15) -------------------------------------------------------------
// In 1D the system is tiny (M_h = m + 1 entries; c1: 16), and the launched loop (pad, C2R, multiply,
// R2C, apply, x/r, p: 7 launches per iteration, ~17 us) is all dependent-launch latency.  One CTA runs
// the whole CG with every vector in shared memory and the Toeplitz product by its direct sum
// out_j = sum_{k=-m}^{m} v_{j-k} u_k (u = D p, u_{-k} = conj u_k; out_0 forced real, as the FFT
// path's C2R projects), the recurrences and stopping rule of k_cg_xr + k_cg_p (reading G6).
constexpr int kCg1Threads = 256, kCg1MaxM = 256;
__device__ __forceinline__ double cg1_sum(double v, double *sh) {  // block sum, valid in every thread
  v = block_sum(v, sh);
  if (threadIdx.x == 0) sh[32] = v;
  __syncthreads();
  const double r = sh[32];
  __syncthreads();
  return r;
}
__global__ void __launch_bounds__(kCg1Threads) k_cg_1d(const double2 *__restrict__ vh, const double *__restrict__ Dh,
                                                       double2 *x, double2 *r, double2 *p0, int m, CGState *st,
                                                       double *hist) {
  extern __shared__ __align__(16) double2 c1sm[];
  __shared__ double sh[40];
  const int Mh = m + 1, t = threadIdx.x;
  double2 *vs = c1sm, *us = vs + 4 * m + 1, *rs = us + 2 * m + 1, *ps = rs + Mh, *xs = ps + Mh;
  double *ds = reinterpret_cast<double *>(xs + Mh);
  for (int d = t; d <= 4 * m; d += kCg1Threads) {  // v over J_2m: v_{-d} = conj v_d
    const int dl = d - 2 * m;
    const double2 v = vh[dl >= 0 ? dl : -dl];
    vs[d] = dl >= 0 ? v : make_double2(v.x, -v.y);
  }
  for (int i = t; i < Mh; i += kCg1Threads) {
    rs[i] = ps[i] = r[i];  // r_0 = b (k_cg_init)
    xs[i] = x[i];
    ds[i] = Dh[i];
  }
  const double tol = st->tol, bnorm = st->bnorm, s2 = st->sigma2;
  const long long max_iter = st->max_iter;
  long long it = st->iter;
  if (st->done) return;
  double rr = st->rrs[0], beta = 0.0;
  __syncthreads();
  for (;;) {
    for (int i = t; i < Mh; i += kCg1Threads) {
      const double2 rq = rs[i], po = ps[i];
      ps[i] = make_double2(rq.x + beta * po.x, rq.y + beta * po.y);
    }
    __syncthreads();
    for (int k = t; k <= 2 * m; k += kCg1Threads) {
      const int kk = k - m, a = kk >= 0 ? kk : -kk;
      const double2 pp = ps[a];
      us[k] = make_double2(ds[a] * pp.x, kk >= 0 ? ds[a] * pp.y : -ds[a] * pp.y);
    }
    __syncthreads();
    double acc = 0.0;
    double2 apv[(kCg1MaxM + kCg1Threads) / kCg1Threads];
#pragma unroll
    for (int q = 0; q < (kCg1MaxM + kCg1Threads) / kCg1Threads; ++q) {
      const int j = t + q * kCg1Threads;
      if (j < Mh) {
        double ox = 0.0, oy = 0.0;
        for (int k = 0; k <= 2 * m; ++k) {  // v_{j-k} u_k, k = -m..m
          const double2 v = vs[j - (k - m) + 2 * m], u = us[k];
          ox = fma(v.x, u.x, fma(-v.y, u.y, ox));
          oy = fma(v.x, u.y, fma(v.y, u.x, oy));
        }
        const double2 pp = ps[j];
        double2 a = make_double2(ds[j] * ox + s2 * pp.x, ds[j] * oy + s2 * pp.y);
        if (j == 0) a.y = s2 * pp.y;  // j = 0: (T u)_0 is real
        apv[q] = a;
        acc += (j ? 2.0 : 1.0) * (pp.x * a.x + pp.y * a.y);
      }
    }
    const double alpha = rr / cg1_sum(acc, sh);
    double racc = 0.0;
#pragma unroll
    for (int q = 0; q < (kCg1MaxM + kCg1Threads) / kCg1Threads; ++q) {
      const int j = t + q * kCg1Threads;
      if (j < Mh) {
        const double2 pp = ps[j];
        double2 rq = rs[j], xq = xs[j];
        xq.x += alpha * pp.x;
        xq.y += alpha * pp.y;
        rq.x -= alpha * apv[q].x;
        rq.y -= alpha * apv[q].y;
        xs[j] = xq;
        rs[j] = rq;
        racc += (j ? 2.0 : 1.0) * (rq.x * rq.x + rq.y * rq.y);
      }
    }
    const double rr_new = cg1_sum(racc, sh);
    ++it;
    beta = rr_new / rr;
    const double rr_prev = rr;
    rr = rr_new;
    const double rel = sqrt(rr_new) / bnorm;
    const int stop = rel <= tol ? 1 : (it >= max_iter ? 2 : 0);
    if (t == 0) {
      st->rr = rr_new;
      st->rr_old = rr_prev;
      st->rrs[it & 1] = rr_new;
      st->iter = it;
      hist[it] = rel;
      if (stop) st->done = stop;
    }
    if (stop) {
      for (int i = t; i < Mh; i += kCg1Threads) {
        x[i] = xs[i];
        r[i] = rs[i];
        p0[i] = ps[i];
      }
      return;
    }
  }
}

static int persist_split_env() {
  const char *e = getenv("EFGP_CG_PSPLIT");
  return (e && atoi(e) > 0) ? atoi(e) : 0;
}
static bool cg_persist() {
  const char *e = getenv("EFGP_CG_PERSIST");
  return !(e && e[0] == '0');
}

// One cooperative launch runs the whole CG (returns cudaErrorNotSupported when the grid cannot be
// co-resident: the caller then takes the launched path).
static cudaError_t launch_persist_cg(efgp_plan *pl, CGState *st, cudaStream_t s, const double2 *vh0 = nullptr) {
  const Params &P = pl->P;
  const int m = (int)P.m, n = 2 * m + 1;
  int dev = 0, coop = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop) return cudaErrorNotSupported;
  int nsplit = persist_split_env() ? persist_split_env() : kToepSplitsHost;
  for (; nsplit >= 1; --nsplit) {
    const PersistGeom G(m, nsplit, kPersistThreads);
    const size_t smem = G.smem();
    if (!G.ok() || smem > 200 * 1024 || 2 * n > pl->cg_blocks || G.Mh > kPersistPer * kPersistThreads ||
        n > kPersistThreads || G.nk * n > kPersistU * kPersistThreads)
      continue;
    cudaError_t e = cudaFuncSetAttribute(k_cg_toep2_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cg_toep2_persist, kPersistThreads, smem);
    if (e != cudaSuccess) return e;
    if ((int64_t)per_sm * pl->num_sms < (int64_t)n * nsplit || nsplit > kToepSplitsHost) continue;
    if (!pl->cg_gbar) {
      e = cudaMalloc((void **)&pl->cg_gbar, sizeof(unsigned));
      if (e != cudaSuccess) return e;
    }
    e = cudaMemsetAsync(pl->cg_gbar, 0, sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    double *part_pAp = pl->partials;  // two slots of 2m+1 row partials (cg_blocks >= 2 (2m+1))
    const double2 *vfull = pl->vfull;
    const double *Dh = pl->D_half;
    double2 *x = pl->x, *r = pl->r, *p0 = pl->p, *ap0 = pl->Ap, *ap1 = pl->p2, *tpart = pl->toep_part;
    unsigned *tcnt = pl->toep_cnt, *gbar = pl->cg_gbar;
    double *hist = pl->hist;
    long long *trace = nullptr;
    const bool want_trace = getenv("EFGP_CG_TRACE") != nullptr;
    if (want_trace) {
      e = cudaMallocAsync((void **)&trace, sizeof(long long) * 8 * n * nsplit, s);
      if (e != cudaSuccess) return e;
      cudaMemsetAsync(trace, 0, sizeof(long long) * 8 * n * nsplit, s);
    }
    void *args[] = {(void *)&vfull, (void *)&Dh, (void *)&x, (void *)&r, (void *)&p0, (void *)&ap0, (void *)&ap1,
                    (void *)&m, (void *)&nsplit, (void *)&st, (void *)&tpart, (void *)&tcnt, (void *)&part_pAp,
                    (void *)&hist, (void *)&gbar, (void *)&trace, (void *)&vh0};
    pl->cg_persist_split = nsplit;
    e = cudaLaunchCooperativeKernel((const void *)k_cg_toep2_persist, dim3((unsigned)(n * nsplit)),
                                    dim3(kPersistThreads), args, smem, s);
    if (want_trace && e == cudaSuccess) {  // diagnostics: mean cycles per phase over CTAs (stderr)
      std::vector<long long> h((size_t)8 * n * nsplit);
      cudaMemcpyAsync(h.data(), trace, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      CGState hs{};
      cudaMemcpy(&hs, st, sizeof(CGState), cudaMemcpyDeviceToHost);
      double mean[6] = {0, 0, 0, 0, 0, 0};
      for (int b = 0; b < n * nsplit; ++b)
        for (int k = 0; k < 6; ++k) mean[k] += (double)h[(size_t)b * 8 + k] / (n * nsplit);
      const double it = hs.iter > 0 ? (double)hs.iter : 1.0;
      fprintf(stderr, "cg persist trace (cycles/iteration, mean over %d CTAs, %lld iterations): p-update+u %.0f, "
              "product+partials %.0f, fence+row atomic %.0f, last-CTA row %.0f, barrier wait %.0f, phase 2 %.0f\n",
              n * nsplit, hs.iter, mean[0] / it, mean[1] / it, mean[2] / it, mean[3] / it, mean[4] / it, mean[5] / it);
      cudaFreeAsync(trace, s);
    }
    return e;
  }
  return cudaErrorNotSupported;
}

static bool cg_fused() {
  const char *e = getenv("EFGP_CG_FUSED");
  return !(e && e[0] == '0');
}

static size_t toep2_smem(int m) {
  const int n = 2 * m + 1, nv = 4 * m + 1;
  const int nout = m + 1, slices = kToepThreads / ((nout + 3) / 4);
  return sizeof(double2) * ((size_t)n * n + (size_t)n * nv + (size_t)slices * nout);
}

static efgp_status ensure_hist(efgp_plan *pl, int64_t max_iter) {
  if (max_iter + 1 > pl->hist_cap) {
    for (cudaGraphExec_t *e : {&pl->cg_exec, &pl->pcg_exec})  // captured graphs hold the old pointer
      if (*e) {
        cudaGraphExecDestroy(*e);
        *e = nullptr;
      }
    if (pl->hist) cudaFree(pl->hist);
    pl->hist = nullptr;
    pl->hist_cap = 0;
    EFGP_CUDA(cudaMalloc(&pl->hist, sizeof(double) * (max_iter + 1)));
    pl->hist_cap = max_iter + 1;
  }
  return EFGP_OK;
}

static unsigned nblocks(int64_t n, int sms) {
  int64_t b = (n + kCGThreads - 1) / kCGThreads;
  const int64_t cap = (int64_t)sms * 4;
  if (b > cap) b = cap;
  return (unsigned)(b < 1 ? 1 : b);
}

template <int D>
static efgp_status enqueue_iteration(efgp_plan *pl, cudaStream_t s, CGState *st, int64_t box, int64_t Ld,
                                     unsigned nb, unsigned nbox, int slot) {
  const Params &P = pl->P;
  double *part_pAp = pl->partials, *part_rr = pl->partials + pl->cg_blocks;
  const bool direct = D == 2 && toeplitz_direct(P);
  const bool pt = D >= 2 && toeplitz_pt(P);
  if (direct && pl->p2 && pl->toep_part && cg_fused() && toep_split()) {  // fused direct CG: two kernels per iteration
    const int nrow = (int)(2 * P.m + 1);
    double2 *pq = slot ? pl->p2 : pl->p, *pold = slot ? pl->p : pl->p2;
    EFGP_CUDA(launch_pdl_smem(k_cg_toep2f, nrow * kToepSplits, kToepSThreads, toep2s_smem((int)P.m), s, pl->vfull,
                              (const double2 *)pl->r, (const double2 *)pold, pq, (const double *)pl->D_half, pl->Ap,
                              (int)P.m, st, pl->toep_part, pl->toep_cnt, part_pAp, (const double *)part_rr, (int)nb,
                              pl->hist, slot));
    EFGP_CUDA(launch_pdl(k_cg_xr2, nb, kCGThreads, s, pl->x, pl->r, (const double2 *)pq, (const double2 *)pl->Ap, P.Mh,
                         (int)P.m, st, (const double *)part_pAp, nrow, part_rr, slot));
    return EFGP_OK;
  }
  if (direct) {  // the partials come from 2m+1 CTAs
    const int nrow = (int)(2 * P.m + 1);
    if (toep_split() && pl->toep_part)
      k_cg_toep2s<<<nrow * kToepSplits, kToepSThreads, toep2s_smem((int)P.m), s>>>(
          pl->vfull, pl->p, pl->D_half, pl->Ap, (int)P.m, st, pl->toep_part, pl->toep_cnt, part_pAp);
    else
      k_cg_toep2<<<nrow, kToepThreads, toep2_smem((int)P.m), s>>>(pl->vfull, pl->p, pl->D_half, pl->Ap, (int)P.m, st,
                                                                  part_pAp);
    EFGP_CUDA(launch_pdl(k_cg_xr, nb, kCGThreads, s, pl->x, pl->r, pl->p, pl->Ap, P.Mh, (int)P.m, st, part_pAp,
                         part_rr, nrow, (const double *)nullptr));
  } else if (pt) {  // partial-transform product (c2, c4)
    EFGP_TRY(pt_product(pl, st, s));
    k_pt_apply<D><<<nb, kCGThreads, 0, s>>>(pl->pt_T, pl->p, pl->D_half, pl->Ap, P.Mh, (int)P.m, P.L, ipow_(P.L, D - 1),
                                            st, part_pAp);
    EFGP_CUDA(launch_pdl(k_cg_xr, nb, kCGThreads, s, pl->x, pl->r, pl->p, pl->Ap, P.Mh, (int)P.m, st, part_pAp,
                         part_rr, (int)nb, (const double *)nullptr));
  } else {
  EFGP_CUFFT(cufftExecZ2D(pl->plan_c2r_L, pl->Xbox, pl->Yr));
  k_mul<<<nblocks(Ld, pl->num_sms), kCGThreads, 0, s>>>(pl->Yr, pl->vhat, Ld, st);
  EFGP_CUFFT(cufftExecD2Z(pl->plan_r2c_L, pl->Yr, pl->Zbox));
  k_cg_apply<D><<<nb, kCGThreads, 0, s>>>(pl->Zbox, pl->p, pl->D_half, pl->Ap, P.Mh, (int)P.m, P.L, st, part_pAp);
  EFGP_CUDA(launch_pdl(k_cg_xr, nb, kCGThreads, s, pl->x, pl->r, pl->p, pl->Ap, P.Mh, (int)P.m, st, part_pAp,
                       part_rr, (int)nb, (const double *)nullptr));
  }
  EFGP_CUDA(launch_pdl(k_cg_p<D>, nb, kCGThreads, s, pl->r, pl->p, pl->D_half, P.Mh, (int)P.m, P.L,
                       pt ? pl->pt_P : (double2 *)nullptr, pt ? ipow_(P.L, D - 1) : (int64_t)0, st, part_rr, (int)nb,
                       pl->hist));
  if (!direct && !pt)
    EFGP_CUDA(launch_pdl(k_cg_pad<D>, nbox, kCGThreads, s, pl->p, pl->D_half, (int)P.m, P.L, pl->Xbox, box,
                         (const CGState *)st));
  EFGP_CUDA(cudaGetLastError());
  return EFGP_OK;
}

template <int D>
static efgp_status cg_solve_d(efgp_plan *pl, int64_t N_total) {
  const Params &P = pl->P;
  cudaStream_t s = pl->stream;
  int64_t box = P.L / 2 + 1, Ld = P.L;
  for (int k = 0; k < D - 1; ++k) {
    box *= P.L;
    Ld *= P.L;
  }
  const unsigned nb = nblocks(P.Mh, pl->num_sms);
  const unsigned nbox = nblocks(box, pl->num_sms);
  if ((int)nb > pl->cg_blocks) {
    pl->err = "internal: cg partials too small";
    return EFGP_ERR_INVALID;
  }
  int64_t max_iter = P.max_iter_opt;
  if (max_iter <= 0) {
    const double Nd = (double)(N_total > 0 ? N_total : 1);
    max_iter = (int64_t)std::ceil(std::log(1.0 / P.cg_tol) * std::sqrt(Nd) / (2.0 * pl->cap_sigma));
    if (max_iter < 10) max_iter = 10;
  }
  pl->max_iter_used = max_iter;
  EFGP_TRY(ensure_hist(pl, max_iter));
  CGState *st = reinterpret_cast<CGState *>(pl->scal);
  CGState init{};
  init.tol = P.cg_tol;
  init.sigma2 = pl->sigma2_sys;
  init.max_iter = max_iter;
  EFGP_CUDA(cudaMemcpyAsync(st, &init, sizeof(CGState), cudaMemcpyHostToDevice, s));
  k_cg_init<<<nb, kCGThreads, 0, s>>>(pl->b, pl->x, pl->r, pl->p, P.Mh, (int)P.m, pl->partials);
  k_cg_init2<<<1, kCGThreads, 0, s>>>(st, pl->partials, (int)nb, pl->hist);
  if (D >= 2 && toeplitz_pt(P)) {
    EFGP_TRY(pt_pad<D>(pl, pl->p, s));
    EFGP_CUFFT(cufftSetStream(pl->plan_pt, s));
  } else {
    k_cg_pad0<D><<<nbox, kCGThreads, 0, s>>>(pl->p, pl->D_half, (int)P.m, P.L, pl->Xbox, box);
  }
  EFGP_CUDA(cudaGetLastError());
  EFGP_CUFFT(cufftSetStream(pl->plan_c2r_L, s));
  EFGP_CUFFT(cufftSetStream(pl->plan_r2c_L, s));
  if (D == 2 && toeplitz_direct(P))
    EFGP_CUDA(cudaFuncSetAttribute(k_cg_toep2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)toep2_smem((int)P.m)));

  int G = P.graph_iters;
  const bool fused = D == 2 && toeplitz_direct(P) && pl->p2 && pl->toep_part && cg_fused() && toep_split();
  pl->cg_persist_split = 0;
  pl->cg_dft2 = 0;
  if (D == 1 && P.m <= kCg1MaxM && cg_persist()) {  // 1D: the whole CG in one CTA
    const int m = (int)P.m;
    const size_t smem = sizeof(double2) * ((4 * (size_t)m + 1) + (2 * (size_t)m + 1) + 3 * ((size_t)m + 1)) +
                        sizeof(double) * ((size_t)m + 1);
    EFGP_CUDA(cudaFuncSetAttribute(k_cg_1d, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_cg_1d<<<1, kCg1Threads, smem, s>>>(reinterpret_cast<const double2 *>(pl->modes_sum), pl->D_half, pl->x, pl->r,
                                         pl->p, m, st, pl->hist);
    EFGP_CUDA(cudaGetLastError());
    pl->cg_dft2 = 2;  // (info: 2 = the one-CTA 1D kernel)
    CGState host{};
    EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned, st, sizeof(CGState), cudaMemcpyDeviceToHost, s));
    EFGP_CUDA(cudaStreamSynchronize(s));
    std::memcpy(&host, pl->h_pinned, sizeof(CGState));
    pl->iters = host.iter;
    pl->rel_resid = host.bnorm > 0 ? std::sqrt(host.rr) / host.bnorm : 0.0;
    return host.done == 2 ? EFGP_ERR_NOCONVERGE : EFGP_OK;
  }
  if (D == 2 && toeplitz_dft2(P) && cg_persist()) {  // 2D beyond the direct product: persistent DFT CG
    const cudaError_t e = launch_dft2_cg(pl, st, s);
    if (e == cudaSuccess) {
      pl->cg_dft2 = 1;
      CGState host{};
      EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned, st, sizeof(CGState), cudaMemcpyDeviceToHost, s));
      EFGP_CUDA(cudaStreamSynchronize(s));
      std::memcpy(&host, pl->h_pinned, sizeof(CGState));
      pl->iters = host.iter;
      pl->rel_resid = host.bnorm > 0 ? std::sqrt(host.rr) / host.bnorm : 0.0;
      return host.done == 2 ? EFGP_ERR_NOCONVERGE : EFGP_OK;
    }
    if (e != cudaErrorNotSupported && e != cudaErrorCooperativeLaunchTooLarge) {
      pl->err = "persistent DFT CG launch failed";
      return EFGP_ERR_CUDA;
    }
    cudaGetLastError();
  }
  if (fused && cg_persist()) {  // the whole loop in one cooperative kernel
    const cudaError_t e = launch_persist_cg(pl, st, s);
    if (e == cudaSuccess) {
      CGState host{};
      EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned, st, sizeof(CGState), cudaMemcpyDeviceToHost, s));
      EFGP_CUDA(cudaStreamSynchronize(s));
      std::memcpy(&host, pl->h_pinned, sizeof(CGState));
      pl->iters = host.iter;
      pl->rel_resid = host.bnorm > 0 ? std::sqrt(host.rr) / host.bnorm : 0.0;
      return host.done == 2 ? EFGP_ERR_NOCONVERGE : EFGP_OK;
    }
    pl->cg_persist_split = 0;
    if (e != cudaErrorNotSupported && e != cudaErrorCooperativeLaunchTooLarge) {
      pl->err = "persistent CG launch failed";
      return EFGP_ERR_CUDA;
    }
    cudaGetLastError();  // not co-resident: the launched path below
  }
  if (fused) G += G & 1;  // the fused iterations alternate two p slots: an even count per graph
  if (!pl->cg_exec || pl->cg_exec_iters != G) {
    if (pl->cg_exec) cudaGraphExecDestroy(pl->cg_exec);
    pl->cg_exec = nullptr;
    cudaGraph_t graph;
    EFGP_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int it = 0; it < G; ++it) {
      efgp_status e = enqueue_iteration<D>(pl, s, st, box, Ld, nb, nbox, it & 1);
      if (e != EFGP_OK) {
        cudaStreamEndCapture(s, &graph);
        return e;
      }
    }
    EFGP_CUDA(cudaStreamEndCapture(s, &graph));
    EFGP_CUDA(cudaGraphInstantiate(&pl->cg_exec, graph, 0));
    cudaGraphDestroy(graph);
    pl->cg_exec_iters = G;
  }
  CGState host{};
  for (;;) {
    EFGP_CUDA(cudaGraphLaunch(pl->cg_exec, s));
    EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned, st, sizeof(CGState), cudaMemcpyDeviceToHost, s));
    EFGP_CUDA(cudaStreamSynchronize(s));
    std::memcpy(&host, pl->h_pinned, sizeof(CGState));
    if (host.done) break;
  }
  pl->iters = host.iter;
  pl->rel_resid = host.bnorm > 0 ? std::sqrt(host.rr) / host.bnorm : 0.0;
  return host.done == 2 ? EFGP_ERR_NOCONVERGE : EFGP_OK;
}

// ---- CG with a caller-applied operator (NEXT-3: the product is a type-2 + type-1 NUFFT pair, not a
// Toeplitz product).  Same recurrences and stopping rule (reading G6); host-driven, one small
// device->host read of the state per iteration (each iteration is O(N) work).
__global__ void k_dot_pAp(const double2 *__restrict__ p, const double2 *__restrict__ Ap, int64_t Mh, int m,
                          double *__restrict__ part) {
  __shared__ double sh[40];
  double acc = 0.0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x) {
    const double2 pp = p[q], a = Ap[q];
    const double wq = (q % (m + 1)) ? 2.0 : 1.0;
    acc += wq * (pp.x * a.x + pp.y * a.y);
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

template <int D>
static efgp_status cg_solve_op_d(efgp_plan *pl, int64_t max_iter, CGOp op, void *ctx) {
  const Params &P = pl->P;
  cudaStream_t s = pl->stream;
  const unsigned nb = nblocks(P.Mh, pl->num_sms);
  pl->max_iter_used = max_iter;
  EFGP_TRY(ensure_hist(pl, max_iter));
  CGState *st = reinterpret_cast<CGState *>(pl->scal);
  CGState init{};
  init.tol = P.cg_tol;
  init.max_iter = max_iter;
  double *part_pAp = pl->partials, *part_rr = pl->partials + pl->cg_blocks;
  EFGP_CUDA(cudaMemcpyAsync(st, &init, sizeof(CGState), cudaMemcpyHostToDevice, s));
  k_cg_init<<<nb, kCGThreads, 0, s>>>(pl->b, pl->x, pl->r, pl->p, P.Mh, (int)P.m, pl->partials);
  k_cg_init2<<<1, kCGThreads, 0, s>>>(st, pl->partials, (int)nb, pl->hist);
  EFGP_CUDA(cudaGetLastError());
  CGState host{};
  for (;;) {
    EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned, st, sizeof(CGState), cudaMemcpyDeviceToHost, s));
    EFGP_CUDA(cudaStreamSynchronize(s));
    std::memcpy(&host, pl->h_pinned, sizeof(CGState));
    if (host.done) break;
    EFGP_TRY(op(pl, pl->p, pl->Ap, ctx));
    k_dot_pAp<<<nb, kCGThreads, 0, s>>>(pl->p, pl->Ap, P.Mh, (int)P.m, part_pAp);
    k_cg_xr<<<nb, kCGThreads, 0, s>>>(pl->x, pl->r, pl->p, pl->Ap, P.Mh, (int)P.m, st, part_pAp, part_rr, (int)nb);
    k_cg_p<D><<<nb, kCGThreads, 0, s>>>(pl->r, pl->p, pl->D_half, P.Mh, (int)P.m, P.L, nullptr, 0, st, part_rr,
                                        (int)nb, pl->hist);
    EFGP_CUDA(cudaGetLastError());
  }
  pl->iters = host.iter;
  pl->rel_resid = host.bnorm > 0 ? std::sqrt(host.rr) / host.bnorm : 0.0;
  return host.done == 2 ? EFGP_ERR_NOCONVERGE : EFGP_OK;
}

efgp_status cg_solve_op(efgp_plan *pl, int64_t max_iter, CGOp op, void *ctx) {
  switch (pl->P.d) {
    case 1: return cg_solve_op_d<1>(pl, max_iter, op, ctx);
    case 2: return cg_solve_op_d<2>(pl, max_iter, op, ctx);
    case 3: return cg_solve_op_d<3>(pl, max_iter, op, ctx);
  }
  return EFGP_ERR_INVALID;
}

// PCG x/r update after the direct Toeplitz product: (p, Ap) partials come from its nrow CTAs, (r, z)
// partials from the previous dot over nb CTAs
__global__ void k_cg_xr_pc_direct(double2 *__restrict__ x, double2 *__restrict__ r, const double2 *__restrict__ p,
                                  const double2 *__restrict__ Ap, int64_t Mh, int m, CGState *st,
                                  const double *__restrict__ part_pAp, int npAp, double *__restrict__ part_rr,
                                  const double *__restrict__ part_rz, int nblk) {
  __shared__ double sh[40];
  pdl_wait();
  pdl_trigger();
  if (st->done) return;
  const double pAp = reduce_partials(part_pAp, npAp, sh);
  const double rz = reduce_partials(part_rz, nblk, sh);
  if (blockIdx.x == 0 && threadIdx.x == 0) st->rz = rz;
  const double alpha = rz / pAp;
  double acc = 0.0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x) {
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
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part_rr[blockIdx.x] = acc;
}

// ---- NEXT-4: preconditioned CG with the Kronecker preconditioner of precond.cu (reading G12).
// Standard PCG recurrences; the stopping rule and history are those of CG (||r_k|| / ||b||, G6).
__global__ void k_pcg_check(CGState *st, const double *__restrict__ part_rr, int nblk, double *__restrict__ hist) {
  __shared__ double sh[40];
  pdl_wait();
  pdl_trigger();
  if (st->done) return;
  const double rr = reduce_partials(part_rr, nblk, sh);
  if (threadIdx.x == 0) {
    st->rr = rr;
    const long long it = st->iter + 1;
    st->iter = it;
    const double rel = sqrt(rr) / st->bnorm;
    hist[it] = rel;
    if (rel <= st->tol) st->done = 1;
    else if (it >= st->max_iter) st->done = 2;
  }
}

__global__ void k_pcg_dot(const double2 *__restrict__ r, const double2 *__restrict__ z, int64_t Mh, int m,
                          const CGState *st, double *__restrict__ part) {
  __shared__ double sh[40];
  pdl_wait();
  pdl_trigger();
  if (st->done) return;
  double acc = 0.0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x) {
    const double2 a = r[q], b = z[q];
    const double wq = (q % (m + 1)) ? 2.0 : 1.0;
    acc += wq * (a.x * b.x + a.y * b.y);
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// p = z + (rz_new / rz) p   (first == true: p = z)
__global__ void k_pcg_p(const double2 *__restrict__ z, double2 *__restrict__ p, int64_t Mh, const CGState *st,
                        const double *__restrict__ part_rz, int nblk, int first) {
  __shared__ double sh[40];
  pdl_wait();
  pdl_trigger();
  if (st->done) return;
  const double bcg = first ? 0.0 : reduce_partials(part_rz, nblk, sh) / st->rz;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Mh; q += (int64_t)gridDim.x * blockDim.x) {
    const double2 zq = z[q], pp = p[q];
    p[q] = make_double2(zq.x + bcg * pp.x, zq.y + bcg * pp.y);
  }
}

template <int D>
static efgp_status enqueue_pcg_iteration(efgp_plan *pl, cudaStream_t s, CGState *st, int64_t box, int64_t Ld,
                                         unsigned nb, unsigned nbox) {
  const Params &P = pl->P;
  double *part_pAp = pl->partials, *part_rr = pl->partials + pl->cg_blocks, *part_rz = pl->partials + 2 * pl->cg_blocks;
  const bool direct = D == 2 && toeplitz_direct(P);
  const bool pt = D >= 2 && toeplitz_pt(P);
  if (direct) {
    const int nrow = (int)(2 * P.m + 1);
    if (toep_split() && pl->toep_part)
      k_cg_toep2s<<<nrow * kToepSplits, kToepSThreads, toep2s_smem((int)P.m), s>>>(
          pl->vfull, pl->p, pl->D_half, pl->Ap, (int)P.m, st, pl->toep_part, pl->toep_cnt, part_pAp);
    else
      k_cg_toep2<<<nrow, kToepThreads, toep2_smem((int)P.m), s>>>(pl->vfull, pl->p, pl->D_half, pl->Ap, (int)P.m, st,
                                                                  part_pAp);
    // (x, r update: alpha from the toep2 partials, (r, z) from the previous dot's partials)
    EFGP_CUDA(launch_pdl(k_cg_xr_pc_direct, nb, kCGThreads, s, pl->x, pl->r, pl->p, (const double2 *)pl->Ap, P.Mh,
                         (int)P.m, st, (const double *)part_pAp, nrow, part_rr, (const double *)part_rz, (int)nb));
  } else {
  if (pt) {
    EFGP_TRY(pt_product(pl, st, s));
    k_pt_apply<D><<<nb, kCGThreads, 0, s>>>(pl->pt_T, pl->p, pl->D_half, pl->Ap, P.Mh, (int)P.m, P.L, ipow_(P.L, D - 1),
                                            st, part_pAp);
  } else {
  EFGP_CUFFT(cufftExecZ2D(pl->plan_c2r_L, pl->Xbox, pl->Yr));
  k_mul<<<nblocks(Ld, pl->num_sms), kCGThreads, 0, s>>>(pl->Yr, pl->vhat, Ld, st);
  EFGP_CUFFT(cufftExecD2Z(pl->plan_r2c_L, pl->Yr, pl->Zbox));
  k_cg_apply<D><<<nb, kCGThreads, 0, s>>>(pl->Zbox, pl->p, pl->D_half, pl->Ap, P.Mh, (int)P.m, P.L, st, part_pAp);
  }
  k_cg_xr<<<nb, kCGThreads, 0, s>>>(pl->x, pl->r, pl->p, pl->Ap, P.Mh, (int)P.m, st, part_pAp, part_rr, (int)nb,
                                    part_rz);
  }
  EFGP_CUDA(launch_pdl(k_pcg_check, 1, kCGThreads, s, st, (const double *)part_rr, (int)nb, pl->hist));
  EFGP_TRY(precond_apply(pl, pl->r, pl->z, &st->done, s, true));
  EFGP_CUDA(launch_pdl(k_pcg_dot, nb, kCGThreads, s, (const double2 *)pl->r, (const double2 *)pl->z, P.Mh, (int)P.m,
                       (const CGState *)st, part_rz));
  EFGP_CUDA(launch_pdl(k_pcg_p, nb, kCGThreads, s, (const double2 *)pl->z, pl->p, P.Mh, (const CGState *)st,
                       (const double *)part_rz, (int)nb, 0));
  if (pt) EFGP_TRY(pt_pad<D>(pl, pl->p, s));
  else if (!direct) k_cg_pad<D><<<nbox, kCGThreads, 0, s>>>(pl->p, pl->D_half, (int)P.m, P.L, pl->Xbox, box, st);
  EFGP_CUDA(cudaGetLastError());
  return EFGP_OK;
}

template <int D>
static efgp_status pcg_solve_d(efgp_plan *pl, int64_t N_total) {
  const Params &P = pl->P;
  cudaStream_t s = pl->stream;
  int64_t box = P.L / 2 + 1, Ld = P.L;
  for (int k = 0; k < D - 1; ++k) {
    box *= P.L;
    Ld *= P.L;
  }
  const unsigned nb = nblocks(P.Mh, pl->num_sms);
  const unsigned nbox = nblocks(box, pl->num_sms);
  int64_t max_iter = P.max_iter_opt;
  if (max_iter <= 0) {
    const double Nd = (double)(N_total > 0 ? N_total : 1);
    max_iter = (int64_t)std::ceil(std::log(1.0 / P.cg_tol) * std::sqrt(Nd) / (2.0 * pl->cap_sigma));
    if (max_iter < 10) max_iter = 10;
  }
  pl->max_iter_used = max_iter;
  EFGP_TRY(ensure_hist(pl, max_iter));
  CGState *st = reinterpret_cast<CGState *>(pl->scal);
  CGState init{};
  init.tol = P.cg_tol;
  init.sigma2 = pl->sigma2_sys;
  init.max_iter = max_iter;
  double *part_rz = pl->partials + 2 * pl->cg_blocks;
  EFGP_CUDA(cudaMemcpyAsync(st, &init, sizeof(CGState), cudaMemcpyHostToDevice, s));
  k_cg_init<<<nb, kCGThreads, 0, s>>>(pl->b, pl->x, pl->r, pl->p, P.Mh, (int)P.m, pl->partials);
  k_cg_init2<<<1, kCGThreads, 0, s>>>(st, pl->partials, (int)nb, pl->hist);
  pl->cg_persist_split = 0;
  pl->cg_dft2 = 0;
  if (D == 2 && P.precond == EFGP_PRECOND_JACOBI && cg_persist()) {
    // Jacobi PCG in the persistent 2D kernels (z = r / (D^2 v_0 + sigma^2) formed in place)
    const double2 *vh0 = reinterpret_cast<const double2 *>(pl->modes_sum) + (int64_t)(2 * P.m) * (2 * P.m + 1);
    cudaError_t e = cudaErrorNotSupported;
    if (toeplitz_direct(P) && pl->p2 && pl->toep_part) {
      e = launch_persist_cg(pl, st, s, vh0);
    } else if (toeplitz_dft2(P)) {
      e = launch_dft2_cg(pl, st, s, vh0);
      if (e == cudaSuccess) pl->cg_dft2 = 1;
    }
    if (e == cudaSuccess) {
      CGState host{};
      EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned, st, sizeof(CGState), cudaMemcpyDeviceToHost, s));
      EFGP_CUDA(cudaStreamSynchronize(s));
      std::memcpy(&host, pl->h_pinned, sizeof(CGState));
      pl->iters = host.iter;
      pl->rel_resid = host.bnorm > 0 ? std::sqrt(host.rr) / host.bnorm : 0.0;
      return host.done == 2 ? EFGP_ERR_NOCONVERGE : EFGP_OK;
    }
    pl->cg_persist_split = 0;
    pl->cg_dft2 = 0;
    if (e != cudaErrorNotSupported && e != cudaErrorCooperativeLaunchTooLarge) {
      pl->err = "persistent PCG launch failed";
      return EFGP_ERR_CUDA;
    }
    cudaGetLastError();
  }
  EFGP_TRY(precond_apply(pl, pl->r, pl->z, &st->done, s));          // z0 = M^-1 b
  k_pcg_dot<<<nb, kCGThreads, 0, s>>>(pl->r, pl->z, P.Mh, (int)P.m, st, part_rz);
  k_pcg_p<<<nb, kCGThreads, 0, s>>>(pl->z, pl->p, P.Mh, st, part_rz, (int)nb, 1);  // p0 = z0
  if (D >= 2 && toeplitz_pt(P)) {
    EFGP_TRY(pt_pad<D>(pl, pl->p, s));
    EFGP_CUFFT(cufftSetStream(pl->plan_pt, s));
  } else {
    k_cg_pad0<D><<<nbox, kCGThreads, 0, s>>>(pl->p, pl->D_half, (int)P.m, P.L, pl->Xbox, box);
  }
  EFGP_CUDA(cudaGetLastError());
  EFGP_CUFFT(cufftSetStream(pl->plan_c2r_L, s));
  EFGP_CUFFT(cufftSetStream(pl->plan_r2c_L, s));
  if (D == 2 && toeplitz_direct(P))
    EFGP_CUDA(cudaFuncSetAttribute(k_cg_toep2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)toep2_smem((int)P.m)));
  const int G = P.graph_iters;
  if (!pl->pcg_exec || pl->pcg_exec_iters != G || pl->pcg_exec_sigma2 != pl->sigma2_sys) {
    pl->pcg_exec_sigma2 = pl->sigma2_sys;
    if (pl->pcg_exec) cudaGraphExecDestroy(pl->pcg_exec);
    pl->pcg_exec = nullptr;
    cudaGraph_t graph;
    EFGP_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int it = 0; it < G; ++it) {
      efgp_status e = enqueue_pcg_iteration<D>(pl, s, st, box, Ld, nb, nbox);
      if (e != EFGP_OK) {
        cudaStreamEndCapture(s, &graph);
        return e;
      }
    }
    EFGP_CUDA(cudaStreamEndCapture(s, &graph));
    EFGP_CUDA(cudaGraphInstantiate(&pl->pcg_exec, graph, 0));
    cudaGraphDestroy(graph);
    pl->pcg_exec_iters = G;
  }
  CGState host{};
  for (;;) {
    EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned, st, sizeof(CGState), cudaMemcpyDeviceToHost, s));
    EFGP_CUDA(cudaStreamSynchronize(s));
    std::memcpy(&host, pl->h_pinned, sizeof(CGState));
    if (host.done) break;
    EFGP_CUDA(cudaGraphLaunch(pl->pcg_exec, s));
  }
  pl->iters = host.iter;
  pl->rel_resid = host.bnorm > 0 ? std::sqrt(host.rr) / host.bnorm : 0.0;
  return host.done == 2 ? EFGP_ERR_NOCONVERGE : EFGP_OK;
}

efgp_status pcg_solve(efgp_plan *pl, int64_t N_total) {
  switch (pl->P.d) {
    case 1: return pcg_solve_d<1>(pl, N_total);
    case 2: return pcg_solve_d<2>(pl, N_total);
    case 3: return pcg_solve_d<3>(pl, N_total);
  }
  return EFGP_ERR_INVALID;
}

efgp_status cg_solve(efgp_plan *pl, int64_t N_total) {
  switch (pl->P.d) {
    case 1: return cg_solve_d<1>(pl, N_total);
    case 2: return cg_solve_d<2>(pl, N_total);
    case 3: return cg_solve_d<3>(pl, N_total);
  }
  return EFGP_ERR_INVALID;
}

}  // namespace efgp
