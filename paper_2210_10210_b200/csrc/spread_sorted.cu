// K1, SORTED strategy (d = 2, W <= 6): tile-binned spreading with register accumulation, as ONE
// persistent warp-specialised kernel (type-1 of eqs "88" and "rhs").
//
// Why: a 2D point touches W^2 cells per strength; accumulating each touch with an atomic is bounded
// by the atomic units (shared fp64 atomicAdd is a CAS loop on sm_100a), far below HBM speed
// (DESIGN.md §7).  All points whose footprint starts at the same cell (the "start cell" i0 = ceil(t -
// W/2) per dimension) share one W x W window, so a thread that owns a start cell accumulates all of
// its points in registers and pays the window update once per tile segment.
//
// The start cells reachable from x in [0,1]^2 form an S x S square (S = s_count); it is cut into
// tiles of T1 x T2 start cells (T1 T2 <= 128, one accumulator thread per start cell).  The points
// are processed in chunks of C points; the chunk's records go through L2-resident per-tile lists
// (NBUF buffers).  One CTA per SM (cooperative launch, all CTAs co-resident), 12 warps:
//   binner warps 8-11  : stream batches of 1024 points from HBM by bulk async copy (TMA engine, a
//                        3-stage mbarrier ring that runs ahead across chunks), validate, rank per
//                        tile (shared int atomics; start cell -> tile by lookup table), reserve room
//                        in each tile's list with ONE global atomic per (batch, tile), and write the
//                        records tile-contiguously with coalesced stores: x pairs (16 B) and y (8 B).
//                        A full list spills the point to direct fp64 RED spreading (correct for any
//                        data, fast for spread-out data).  Chunk k is written once all CTAs have
//                        finished accumulating chunk k - NBUF (global counters).
//   accumulator warps 0-7 (one thread per start cell): once all CTAs have binned chunk k, CTA b
//                        takes the b-th equal share of the concatenated tile lists, in rounds of R
//                        records: bulk copy into shared memory; pass 1 (thread per record) start
//                        cell + rank (shared int atomics); scan; pass 2 (thread per record) writes the
//                        record (FP64 mode) or its fp32 kernel weights (FP32 / MIXED) at its
//                        cell-sorted slot; phase C (thread per start cell) accumulates into two
//                        W x W register windows (strength 1 and y, both on the n1 grid).  At the end
//                        of a tile segment the windows are summed in shared memory in W^2
//                        conflict-free steps and flushed with one RED per cell.
// Register budget: setmaxnreg moves registers from the binner warpgroup to the accumulators.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "efgp_internal.cuh"

namespace efgp {

#ifndef EFGP_SORTED_BTRACE
#define EFGP_SORTED_BTRACE 0  // binner phase clocks in the EFGP_SORTED_TRACE buffer (diagnostic builds)
#endif
#ifndef EFGP_BIN_WARPS
#define EFGP_BIN_WARPS 4
#endif
constexpr int kAccThreads = 256;                  // warps 0-7
constexpr int kBinThreads = 32 * EFGP_BIN_WARPS;  // warps 8.. (one or two warpgroups)
// setmaxnreg budgets (multiples of 8; kAccThreads acc + kBinThreads bin <= 64K registers)
#ifndef EFGP_BIN_REGS8
#define EFGP_BIN_REGS8 56
#endif
constexpr int kBinRegs = EFGP_BIN_WARPS == 4 ? 104 : EFGP_BIN_REGS8;
constexpr int kAccRegs = EFGP_BIN_WARPS == 4 ? 200 : (65536 / 256 - EFGP_BIN_REGS8) / 8 * 8;
constexpr int kFusedThreads = kAccThreads + kBinThreads;
constexpr int kBarAcc = 1, kBarBin = 2, kBarAcc2 = 3;  // named barriers (0 = __syncthreads)
constexpr int kModeF64 = 0;   // fp64 weights (evaluated per record in phase C), fp64 accumulation
constexpr int kModeW32 = 1;   // fp32 weights (pass 2), fp64 accumulation
[[maybe_unused]] constexpr int kModeA32 = 2;   // fp32 weights, fp32 (packed FFMA2) sums within a round, fp64 across
constexpr int kModeF64W = 3;  // FP64 with a per-point strength-1 weight (NEXT-3: strengths 1/sigma_n^2 and
                              // y_n/sigma_n^2 in ONE pass; records (x1, x2, w, y), start cell recomputed)

__device__ __forceinline__ int wrap_s(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

// grid coordinate of a point in units of the fine-grid spacing: t = h x n (theta / Delta)
// (explicit roundings: binning, classification and weights must agree on the start cell bit for bit)
__device__ __forceinline__ double grid_t(double h, double x, int n) { return __dmul_rn(__dmul_rn(h, x), (double)n); }
template <int W>
__device__ __forceinline__ int start_cell(double t) {
  return (int)ceil(__dsub_rn(t, 0.5 * W));
}

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
// named barrier that also returns whether the predicate held in any participating thread
__device__ __forceinline__ bool named_sync_or(int id, int n, bool pred) {
  unsigned r;
  asm volatile(
      "{\n .reg .pred p, q;\n setp.ne.u32 p, %1, 0;\n bar.red.or.pred q, %2, %3, p;\n selp.u32 %0, 1, 0, q;\n}"
      : "=r"(r)
      : "r"((unsigned)pred), "r"(id), "r"(n)
      : "memory");
  return r != 0;
}

// exclusive scan of one int per thread over a group of NW warps (group thread index g, named
// barrier id); returns the exclusive prefix, *total gets the sum
template <int NW>
__device__ __forceinline__ int group_scan(int v, int g, int *wsum, int bar, int *total) {
  const int lane = g & 31, wid = g >> 5;
  int s = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, s, o);
    if (lane >= o) s += t;
  }
  if (lane == 31) wsum[wid] = s;
  named_sync(bar, NW * 32);
  if (wid == 0) {
    int w = lane < NW ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < NW; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    if (lane < NW) wsum[lane] = w;
  }
  named_sync(bar, NW * 32);
  if (total && g == 0) *total = wsum[NW - 1];
  const int r = s - v + (wid > 0 ? wsum[wid - 1] : 0);
  named_sync(bar, NW * 32);  // wsum reusable, *total visible
  return r;
}

// exclusive scan in place of n ints in shared memory by a group of NW warps
template <int NW>
__device__ void group_scan_array(int *a, int n, int g, int *wsum, int bar, int *total) {
  const int per = (n + NW * 32 - 1) / (NW * 32);
  const int beg = g * per, end = min(n, beg + per);
  int s = 0;
  for (int i = beg; i < end; ++i) s += a[i];
  int run = group_scan<NW>(s, g, wsum, bar, total);
  for (int i = beg; i < end; ++i) {
    const int c = a[i];
    a[i] = run;
    run += c;
  }
  named_sync(bar, NW * 32);
}

// fp32 kernel weights of both coordinates of a 2D point, packed fp32x2 Horner (FFMA2); the reduced
// coordinate s = 2(i0 - t + W/2) - 1 in [-1, 1] is formed in fp64
template <int W>
__device__ __forceinline__ void es_weights_f32x2(double t1, double t2, const EsPolyF &P, float (&w1)[W],
                                                 float (&w2)[W]) {
  const double tm1 = __dsub_rn(t1, 0.5 * W), tm2 = __dsub_rn(t2, 0.5 * W);
  const float2 s = make_float2((float)(2.0 * (ceil(tm1) - tm1) - 1.0), (float)(2.0 * (ceil(tm2) - tm2) - 1.0));
#pragma unroll
  for (int a = 0; a < W; ++a) {
    constexpr int D = es_degree(W);
    float2 acc = make_float2(P.c[a][D], P.c[a][D]);
#pragma unroll
    for (int k = D - 1; k >= 0; --k) acc = __ffma2_rn(acc, s, make_float2(P.c[a][k], P.c[a][k]));
    w1[a] = acc.x;
    w2[a] = acc.y;
  }
}

// fp32 kernel weights of one coordinate as W/2 (rounded up) pairs (w[2p], w[2p+1]) by packed Horner
// (FFMA2: pair accumulator x scalar s + coefficient pair); the pad weight w[W] (W odd) is 0
template <int W>
__device__ __forceinline__ void es_weights_pairs(double t, const EsPolyP &P, float2 (&w)[(W + 1) / 2]) {
  const double tm = __dsub_rn(t, 0.5 * W);
  const float s = (float)(2.0 * (ceil(tm) - tm) - 1.0);
  const float2 s2 = make_float2(s, s);
#pragma unroll
  for (int q = 0; q < (W + 1) / 2; ++q) {
    constexpr int D = es_degree(W);
    float2 acc = P.c[q][D];
#pragma unroll
    for (int k = D - 1; k >= 0; --k) acc = __ffma2_rn(acc, s2, P.c[q][k]);
    w[q] = acc;
  }
}

// direct fp64 RED spreading of one point (list overflow path; the polynomial is read from global
// memory so the kernel parameters are not copied to the stack)
template <int W>
__device__ __noinline__ void spread_point_red(double x1, double x2, double yv, double h, int n1,
                                              const EsPoly *__restrict__ Pg, double *__restrict__ g1,
                                              double *__restrict__ gy, double s1v = 1.0) {
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
      atomicAdd(g1 + gi, p * s1v);
      atomicAdd(gy + gi, p * yv);
    }
  }
}

// ---- bulk async copies global -> shared with mbarriers (TMA engine, 1D) ------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
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
// 256-bit global store (sm_100: STG.E.ENL2.256): a whole 32-byte record in one instruction
__device__ __forceinline__ void st_v4(double4 *p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}
// shared-memory atomic add with a result, skipped when v == 0 / !pred (returns 0 without touching memory).
// Written as a predicated `atom.shared`; ptxas still emits the BSSY / BRA / BSYNC form around an ATOMS with
// a result (same code as `v ? atomicAdd(p, v) : 0`), and unconditional atomics that add 0 measured slower
// — kept as the one place where that choice is made.
__device__ __forceinline__ int atoms_add_if_nz(int *p, int v) {
  int r;
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.s32 q, %2, 0;\n mov.s32 %0, 0;\n @q atom.shared.add.s32 %0, [%1], %2;\n}"
      : "=r"(r)
      : "r"(smem_u32(p)), "r"(v)
      : "memory");
  return r;
}
__device__ __forceinline__ int atoms_inc_if(int *p, bool pred) {
  int r;
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.s32 q, %2, 0;\n mov.s32 %0, 0;\n @q atom.shared.add.s32 %0, [%1], 1;\n}"
      : "=r"(r)
      : "r"(smem_u32(p)), "r"((int)pred)
      : "memory");
  return r;
}
// one step of an inclusive warp scan: x += (lane >= o ? x of lane - o : 0), the range test taken from the
// shuffle's own predicate (no compare, no select, no predicate kept across the steps)
__device__ __forceinline__ int scan_step_up(int x, int o) {
  asm volatile(
      "{\n .reg .pred q;\n .reg .s32 t;\n shfl.sync.up.b32 t|q, %0, %1, 0, 0xffffffff;\n @q add.s32 %0, %0, t;\n}"
      : "+r"(x)
      : "r"(o));
  return x;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void stamp(const unsigned long long *base, int k, int slot) {
  if (base) const_cast<unsigned long long *>(base)[((size_t)k * gridDim.x + blockIdx.x) * 4 + slot] = gtimer();
}
__device__ __forceinline__ void spin_until(const unsigned *p, unsigned target) {
  while (ld_acquire(p) < target) __nanosleep(256);
}

template <int W, int MODE>
struct StageRec {
  // MODE F64: sorted copy of (x1, x2, y).  Otherwise the fp32 weights of each coordinate padded to an
  // even count WE (pad weight 0): w1e[WE], w2e[WE]; then y: MIXED stores it as fp32 in the pad slot
  // w1e[W] (W odd) or after w2e (W even); W32 stores it as fp64 after w2e.  16-byte padded.
  static constexpr int WE = (W + 1) / 2 * 2;
  static constexpr int kYSlot = (W & 1) ? W : 2 * WE;  // MIXED: float index of y
  static constexpr int kBytes = MODE == kModeF64 ? 24 : MODE == kModeF64W ? 32
                                : MODE == kModeW32 ? (8 * WE + 8 + 15) / 16 * 16
                                                   : (4 * (2 * WE + ((W & 1) ? 0 : 1)) + 15) / 16 * 16;
};

// NB bytes of a stage record as floats (16-byte vector loads)
template <int NB>
__device__ __forceinline__ void load_floats(const unsigned char *sp, float (&f)[NB / 4]) {
  const float4 *q = reinterpret_cast<const float4 *>(sp);
#pragma unroll
  for (int i = 0; i < NB / 16; ++i) {
    const float4 v = q[i];
    f[4 * i] = v.x;
    f[4 * i + 1] = v.y;
    f[4 * i + 2] = v.z;
    f[4 * i + 3] = v.w;
  }
}

// All kernel arguments (passed by value; lives in the constant bank).
struct FusedArgs {
  const double *x, *y;
  const double *s1;    // kModeF64W: per-point strength-1 weight (NEXT-3: 1/sigma_n^2), else nullptr
  int wraw;            // kModeF64W: y is the raw observation and s1 the raw noise sd sigma_n; the kernel
                       // validates sigma_n (err[2]), takes min sigma_n (minbits) and weights in pass 2
  unsigned long long *minbits;  // wraw: min sigma_n as IEEE bits (ordered like the value for sigma_n > 0)
  int64_t N, chunk;
  // ramp-down of the last chunks (in batches): batches >= tail_b0 fall into 5 chunks that halve in
  // size (cut points tail_c[0..3] relative to tail_b0), so the accumulators' drain after the last
  // binned chunk is a 1/16-size chunk instead of a full one; tail_b0 = INT64_MAX: uniform chunks
  int64_t tail_b0, tail_c[4];
  int tail_k0;
  int nchunks, nbuf;
  int debug;           // diagnostics (EFGP_SORTED_DEBUG): 1 = accumulators skip their work
  int own;             // 1: static tile ownership (CTA b accumulates tile b; ntiles <= grid)
  unsigned nconsumers; // accumulator groups that release each chunk (acc_done target)
  double h;
  int n1, s_lo, S, T1, T2, nt2, ntiles;
  int segcap;          // records per (tile, binner CTA) segment per chunk
  int R;               // records per accumulator round
  double4 *rec[kMaxNbuf];  // [buf][tile][cta][segcap] records (x1, x2, y, key bits)
  int *segcnt;         // [nchunks][tile][cta] segment lengths
  int *tilecnt;        // [nchunks][tile] list lengths (sum over CTAs)
  unsigned *bin_done;  // [nchunks] CTAs that finished binning chunk k
  unsigned *acc_done;  // [nchunks] CTAs that finished accumulating chunk k
  unsigned long long *trace;  // optional [nchunks][grid][4] globaltimer stamps (EFGP_SORTED_TRACE)
  const EsPoly *poly_dev;
  double *g1, *gy;
  int *err;
};

#ifndef EFGP_WBATCH
#define EFGP_WBATCH 256
#endif
#ifndef EFGP_WSTAGES
#define EFGP_WSTAGES 2
#endif
constexpr int kWBatch = EFGP_WBATCH;              // points per binner-warp batch
constexpr int kWStages = EFGP_WSTAGES;            // TMA ring depth per binner warp
constexpr int kBinWarps = kBinThreads / 32;
constexpr int kTper = 8;  // tiles per binner lane handled by the fixed-trip scan (ntiles <= 256; else a loop)

template <int W, int MODE>
struct FusedSmem {
  // binner: per warp a TMA ring (x pairs + y (+ the strength-1 weight)), per-tile count / offset /
  // base, perm; shared: the CTA's running segment lengths and the start-cell tables
  static constexpr int kPtBytes = MODE == kModeF64W ? 32 : 24;
  __host__ __device__ static size_t bin_warp_bytes(int ntiles) {
    return (size_t)kWStages * kWBatch * kPtBytes + 4 * (size_t)kWBatch + 4 * 4 * (size_t)ntiles;
  }
  __host__ __device__ static size_t bin_bytes(int ntiles, int S) {
    return kBinWarps * ((bin_warp_bytes(ntiles) + 15) / 16 * 16) + 4 * ((size_t)ntiles + 2 * (size_t)S);
  }
};

// ------------------------------------------------------------------------------- binner role
// Four independent binner warps (no CTA barrier per batch).  Each warp streams batches of 256
// points through its own TMA ring, ranks them per tile with warp-private shared counters, reserves
// room in the CTA's segment of each tile with one shared atomic per (batch, tile), and writes the
// records tile-contiguously.  Per-segment and per-tile lengths are published at each chunk's end.
template <int W, int MODE>
__device__ void binner_role(const FusedArgs &A, unsigned char *sm, int g /* 0..127 */) {
  constexpr bool WGT = MODE == kModeF64W;
  const int lane = g & 31, wid = g >> 5, ntiles = A.ntiles, G = gridDim.x;
  const size_t wbytes = (FusedSmem<W, MODE>::bin_warp_bytes(ntiles) + 15) / 16 * 16;
  unsigned char *wsm = sm + wid * wbytes;
  double *xin = reinterpret_cast<double *>(wsm);                      // [stage][kWBatch * 2]
  double *yin = xin + kWStages * 2 * kWBatch;                         // [stage][kWBatch]
  double *s1in = yin + kWStages * kWBatch;                            // [stage][kWBatch] (WGT only)
  int *perm = reinterpret_cast<int *>(yin + (WGT ? 2 : 1) * kWStages * kWBatch);  // kWBatch
  int *wcnt = perm + kWBatch;                                         // ntiles
  int *wloc = wcnt + ntiles;                                          // ntiles
  // per tile, for this batch: the record offset of batch slot 0 in the tile's list buffer (segment
  // start + reserved base - slot base; a record index, < 2^31 by the host's check) and the slot bound
  // (slot < wlim <=> the record fits the segment): the copy-out's address is one add per point
  int2 *wol = reinterpret_cast<int2 *>(wloc + ntiles);                // ntiles x (woff, wlim): one 8-byte load
  int *off = reinterpret_cast<int *>(sm + kBinWarps * wbytes);        // ntiles (CTA-shared)
  int *rowt = off + ntiles;                                           // S
  int *colt = rowt + A.S;                                             // S
  __shared__ __align__(8) uint64_t bar[kBinWarps][kWStages];
  for (int c = g; c < A.S; c += kBinThreads) {
    // (tile << 8 | cell-in-tile) split over the two tables: their SUM is the packed pair (the cell
    // parts add to < T1 T2 <= 128: no carry into the tile bits), one add per point
    rowt[c] = ((c / A.T1) * A.nt2) << 8 | (c % A.T1) * A.T2;
    colt[c] = (c / A.T2) << 8 | (c % A.T2);
  }
  for (int t = g; t < ntiles; t += kBinThreads) off[t] = 0;
  for (int t = lane; t < ntiles; t += 32) wcnt[t] = 0;
  if (lane == 0) {
    for (int s = 0; s < kWStages; ++s) mbar_init(&bar[wid][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  named_sync(kBarBin, kBinThreads);
  const int64_t nbatch = (A.N + kWBatch - 1) / kWBatch;
  const int64_t bpc = A.chunk / kWBatch;  // batches per chunk
  const int64_t nw = (int64_t)G * kBinWarps, gw = (int64_t)blockIdx.x * kBinWarps + wid;
  auto issue = [&](int64_t i) {  // i-th batch of this warp: global batch gw + i nw
    const int64_t b = gw + i * nw;
    if (lane != 0 || b >= nbatch) return;
    const int s = (int)(i % kWStages);
    const int64_t i0 = b * kWBatch;
    const int nb = (int)(A.N - i0 < kWBatch ? A.N - i0 : kWBatch);
    const int ne = nb & ~1;  // y copies need a multiple of 16 bytes; an odd tail is loaded by hand
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect(&bar[wid][s], (uint32_t)(nb * 16 + (WGT ? 2 : 1) * ne * 8));
    bulk_g2s(xin + s * 2 * kWBatch, A.x + 2 * i0, (uint32_t)(nb * 16), &bar[wid][s]);
    if (ne > 0) bulk_g2s(yin + s * kWBatch, A.y + i0, (uint32_t)(ne * 8), &bar[wid][s]);
    if (WGT && ne > 0) bulk_g2s(s1in + s * kWBatch, A.s1 + i0, (uint32_t)(ne * 8), &bar[wid][s]);
  };
  for (int i = 0; i < kWStages; ++i) issue(i);
  uint32_t phases = 0;
  int cur = -1;  // chunk whose segments this CTA is writing
  auto enter_chunk = [&](int k) {
    // publish chunks cur .. k-1, then wait until buffer k % nbuf is free.  Every step is the same
    // three barriers in all four warps (each warp walks every chunk in order).
    while (cur < k) {
      named_sync(kBarBin, kBinThreads);  // all warps are done with chunk cur
      if (cur >= 0) {
        int *sc = A.segcnt + (int64_t)cur * ntiles * G;
        for (int t = g; t < ntiles; t += kBinThreads) {
          const int c = min(off[t], A.segcap);
          sc[(int64_t)t * G + blockIdx.x] = c;
          if (c) atomicAdd(A.tilecnt + (int64_t)cur * ntiles + t, c);
          off[t] = 0;
        }
      }
      named_sync(kBarBin, kBinThreads);  // published
      if (g == 0) {
        if (cur >= 0) {
          __threadfence();
          asm volatile("fence.proxy.async.global;" ::: "memory");
          atomicAdd(A.bin_done + cur, 1u);
          stamp(A.trace, cur, 0);
        }
        if (cur + 1 < A.nchunks && cur + 1 >= A.nbuf) spin_until(A.acc_done + (cur + 1 - A.nbuf), A.nconsumers);
      }
      ++cur;
      named_sync(kBarBin, kBinThreads);  // buffer cur % nbuf is free
    }
  };
  const int tper = (ntiles + 31) / 32, tb = lane * tper, te = min(ntiles, tb + tper);
  // optional phase timing (EFGP_SORTED_TRACE): lane 0 of each binner warp, clock64 cycles summed over
  // the launch: 0 chunk hand-off, 1 TMA wait, 2 load + classify + rank atomics, 3 tile scan + reserve,
  // 4 permutation, 5 copy-out (+ overflow), 6 batches
  // (compiled in only with -DEFGP_SORTED_BTRACE=1: the counters cost registers in the binner role)
#if EFGP_SORTED_BTRACE
  long long bt_acc[7] = {0, 0, 0, 0, 0, 0, 0}, bt_t = clock64();
#define BT(i)                               \
  if (A.trace && lane == 0) {               \
    const long long t_ = clock64();         \
    bt_acc[(i)] += t_ - bt_t;               \
    bt_t = t_;                              \
  }
#else
#define BT(i)
#endif
  [[maybe_unused]] unsigned long long sdmin = ~0ull;  // wraw: this lane's min sigma_n (IEEE bits)
  for (int64_t i = 0;; ++i) {
    const int64_t b = gw + i * nw;
    // every warp walks the chunks in order; a warp with no batch left in a chunk still enters it
    int k = A.nchunks;
    if (b < nbatch) {
      if (b < A.tail_b0) {
        k = (int)(b / bpc);
      } else {
        const int64_t r = b - A.tail_b0;
        k = A.tail_k0 + (r >= A.tail_c[0]) + (r >= A.tail_c[1]) + (r >= A.tail_c[2]) + (r >= A.tail_c[3]);
      }
    }
    BT(5);
    if (k != cur) enter_chunk(k);
    BT(0);
    if (b >= nbatch) break;
    const int s = (int)(i % kWStages);
    const int64_t i0 = b * kWBatch;
    const int nb = (int)(A.N - i0 < kWBatch ? A.N - i0 : kWBatch);
    double4 *rec = A.rec[k % A.nbuf];
    mbar_wait(&bar[wid][s], (phases >> s) & 1u);
    phases ^= 1u << s;
    BT(1);
#if EFGP_SORTED_BTRACE
    if (A.trace && lane == 0) ++bt_acc[6];
#endif
    const double2 *xs2 = reinterpret_cast<const double2 *>(xin + s * 2 * kWBatch);
    double *ys = yin + s * kWBatch;
    double *s1s = s1in + s * kWBatch;
    if ((nb & 1) && lane == 0) {
      ys[nb - 1] = A.y[i0 + nb - 1];
      if (WGT) s1s[nb - 1] = A.s1[i0 + nb - 1];
    }
    __syncwarp();
    int tk[kWBatch / 32], rk[kWBatch / 32];  // (tile << 8 | key), rank within the batch's tile
    // (written as independent predicated steps so the 8 points of a lane overlap their latencies)
    double2 pv[kWBatch / 32];
    double yvv[kWBatch / 32];
    unsigned sdbad = 0;  // wraw: bit q = sigma_n of point q is not a finite positive number
#pragma unroll
    for (int q = 0; q < kWBatch / 32; ++q) {
      const int j = min(q * 32 + lane, nb - 1);
      pv[q] = xs2[j];
      yvv[q] = ys[j];
      if (WGT && A.wraw) {
        const double sdv = s1s[j];
        const bool sok = sdv > 0.0 && isfinite(sdv);
        sdbad |= sok ? 0u : 1u << q;
        const unsigned long long sb = (unsigned long long)__double_as_longlong(sdv);
        if (sok && sb < sdmin) sdmin = sb;
      }
    }
    bool bad = false;
    int ci[kWBatch / 32];
#pragma unroll
    for (int q = 0; q < kWBatch / 32; ++q) {
      const bool in = q * 32 + lane < nb;
      bool ok = pv[q].x >= 0.0 && pv[q].x <= 1.0 && pv[q].y >= 0.0 && pv[q].y <= 1.0 && isfinite(yvv[q]);
      bad |= in && !ok;
      if (WGT) ok = ok && !((sdbad >> q) & 1u);  // a point with an invalid sigma_n is dropped (the fit fails)
      // a rejected point keeps its coordinates; its (arbitrary) start cells are clamped into the tables
      // (one unsigned min per dimension instead of four selects on the coordinates)
      const unsigned smax = (unsigned)(A.S - 1);
      const int r = rowt[min((unsigned)(start_cell<W>(grid_t(A.h, pv[q].x, A.n1)) - A.s_lo), smax)];
      const int c = colt[min((unsigned)(start_cell<W>(grid_t(A.h, pv[q].y, A.n1)) - A.s_lo), smax)];
      tk[q] = (in && ok) ? r + c : -1;
      EFGP_DCHECK(!(in && ok) || ((tk[q] >> 8) < ntiles && (tk[q] & 0xFF) < A.T1 * A.T2));
      ci[q] = (r + c) >> 8;
    }
#pragma unroll
    for (int q = 0; q < kWBatch / 32; ++q) rk[q] = atoms_inc_if(&wcnt[ci[q]], tk[q] >= 0);  // (ci is a valid tile even for a rejected point)
    if (bad) atomicOr(A.err, 1);
    if (WGT && sdbad) atomicOr(A.err + 2, 1);
    __syncwarp();
    BT(2);
    // warp scan of the per-tile counts -> slot offsets; reserve room in the CTA's segments.  A lane's
    // tiles (<= kTper of them: fixed-trip, predicated) have their counts loaded and their segment
    // reservations (shared atomics with a return value) issued back to back before any result is
    // used: a loop that used each atomic's result before issuing the next serialised kTper round trips
    int nv;
    bool ovl = false;  // one of this lane's tiles overflows its segment in this batch (found here, per
                       // tile, so the copy-out loop carries no per-record flag)
    // (the trip count is a compile-time 6 or 8: c5's 169 tiles are 6 per lane, and two more predicated-off
    // trips cost ~20 instructions per batch and lane in the role whose instruction count sets the pace)
    auto scan_fixed = [&](auto kt) {
      constexpr int KT = decltype(kt)::value;
      int cnt[KT], wbv[KT];
      int sum = 0;
#pragma unroll
      for (int u = 0; u < KT; ++u) {
        cnt[u] = tb + u < te ? wcnt[tb + u] : 0;
        sum += cnt[u];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) incl = scan_step_up(incl, o);
      nv = __shfl_sync(0xffffffffu, incl, 31);
#pragma unroll
      for (int u = 0; u < KT; ++u) wbv[u] = atoms_add_if_nz(&off[tb + u], cnt[u]);
#pragma unroll
      for (int u = 0; u < KT; ++u) ovl |= cnt[u] > 0 && wbv[u] + cnt[u] > A.segcap;
      int run = incl - sum;
#pragma unroll
      for (int u = 0; u < KT; ++u) {
        const int t = tb + u;
        if (t < te) {
          wloc[t] = run;
          wol[t] = make_int2((t * G + (int)blockIdx.x) * A.segcap + wbv[u] - run, A.segcap - wbv[u] + run);
          wcnt[t] = 0;
          run += cnt[u];
        }
      }
    };
    if (tper <= 6) {
      scan_fixed(std::integral_constant<int, 6>{});
    } else if (tper <= kTper) {
      scan_fixed(std::integral_constant<int, kTper>{});
    } else {
      int sum = 0;
      for (int t = tb; t < te; ++t) sum += wcnt[t];
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      nv = __shfl_sync(0xffffffffu, incl, 31);
      int run = incl - sum;
      for (int t = tb; t < te; ++t) {
        const int c = wcnt[t];
        wloc[t] = run;
        const int wb = c ? atomicAdd(&off[t], c) : 0;
        ovl |= c > 0 && wb + c > A.segcap;
        wol[t] = make_int2((t * G + (int)blockIdx.x) * A.segcap + wb - run, A.segcap - wb + run);
        wcnt[t] = 0;
        run += c;
      }
    }
    __syncwarp();
    BT(3);
#pragma unroll
    for (int q = 0; q < kWBatch / 32; ++q)
      if (tk[q] >= 0) perm[wloc[tk[q] >> 8] + rk[q]] = (q * 32 + lane) | (tk[q] << 8);
    __syncwarp();
    BT(4);
    const bool any_ovf = __any_sync(0xffffffffu, ovl);
#pragma unroll 4
    for (int slot = lane; slot < nv; slot += 32) {
      const int v = perm[slot];
      const int j = v & 0xFF, key = (v >> 8) & 0xFF, t = v >> 16;
      const int2 ol = wol[t];
      EFGP_DCHECK(j < nb && t < ntiles && slot >= wloc[t] && ol.x + slot >= (t * G + (int)blockIdx.x) * A.segcap);
      const double2 xx = xs2[j];
      const double yv = ys[j];
      const double s1v = WGT ? s1s[j] : 0.0;
      if (slot < ol.y)  // (record index >= 0: the unsigned sum widens in one instruction)
        st_v4(rec + (unsigned)(ol.x + slot), xx.x, xx.y, WGT ? s1v : yv,
              WGT ? yv : __longlong_as_double((long long)key));  // WGT: (x1, x2, w, y), start cell recomputed
    }
    if (any_ovf) {  // full segments (concentrated data): direct RED spreading,
      for (int slot = lane; slot < nv; slot += 32) {  // kept out of the hot loop above
        const int v = perm[slot];
        const int j = v & 0xFF, t = v >> 16;
        if (slot >= wol[t].y) {
          double yo = ys[j], wo = WGT ? s1s[j] : 1.0;
          if (WGT && A.wraw) {  // the strengths of pass 2, same roundings
            wo = __drcp_rn(wo * wo);
            yo = yo * wo;
          }
          spread_point_red<W>(xs2[j].x, xs2[j].y, yo, A.h, A.n1, A.poly_dev, A.g1, A.gy, wo);
        }
      }
    }
    __syncwarp();  // stage s consumed
    issue(i + kWStages);
  }
  if (WGT && A.wraw) {  // min sigma_n over this warp's points (P:1766's iteration cap uses min sigma_n, G11)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long t = __shfl_xor_sync(0xffffffffu, sdmin, o);
      sdmin = t < sdmin ? t : sdmin;
    }
    if (lane == 0 && sdmin != ~0ull) atomicMin(A.minbits, sdmin);
  }
#if EFGP_SORTED_BTRACE
  if (A.trace && lane == 0) {
    unsigned long long *o = A.trace + (size_t)A.nchunks * G * 4 + (size_t)G * 2 * 8 + ((size_t)blockIdx.x * kBinWarps + wid) * 8;
    for (int q = 0; q < 7; ++q) o[q] = (unsigned long long)bt_acc[q];
  }
#endif
#undef BT
}

// -------------------------------------------------------------------------- accumulator role
// Two independent groups of 4 warps (128 threads, one per start cell of a tile of <= 128 cells),
// each with its own named barrier, shared-memory region and share of the chunk's records (virtual
// CTA 2 blockIdx + group), so one group's barriers and latencies overlap the other's work.
constexpr int kAccGroups = 2, kGrpThreads = kAccThreads / kAccGroups;  // 128 threads per group

template <int W, int MODE>
struct AccSmem {
  // raw round (32 B records, bulk-copied), cell-sorted stage, per-cell counts, tile prefix, two
  // segment prefixes, fp64 tile accumulator; all 16-byte multiples
  __host__ __device__ static size_t bytes(int R, int ntiles, int grid, int T1, int T2) {
    size_t b = 32 * (size_t)R + (size_t)R * StageRec<W, MODE>::kBytes + (MODE == kModeF64W ? 4 * (size_t)R : 0);
    b += ((4 * (size_t)(2 * kGrpThreads + ntiles + 1 + 2 * (grid + 1))) + 15) / 16 * 16;
    b += 16 * (size_t)(T1 + W - 1) * (T2 + W - 1);
    return b;
  }
};

template <int W, int MODE>
__device__ void accumulator_role(const FusedArgs &A, unsigned char *sm, int tid_all, const EsPoly &P,
                                 const EsPolyP &PF) {
  constexpr int SB = StageRec<W, MODE>::kBytes;
  const int gi = tid_all / kGrpThreads, tid = tid_all % kGrpThreads;
  const int bar_id = gi == 0 ? kBarAcc : kBarAcc2;
  const int R = A.R, ntiles = A.ntiles, T1 = A.T1, T2 = A.T2, n1 = A.n1, s_lo = A.s_lo, G = gridDim.x;
  const int VG = G * kAccGroups, vb = blockIdx.x * kAccGroups + gi;  // virtual CTA
  if (R <= 0) __trap();  // the host never launches without a round (sorted_geometry checks)
  const double h = A.h;
  [[maybe_unused]] const bool wraw = A.wraw != 0;
  unsigned char *gsm = sm + gi * AccSmem<W, MODE>::bytes(R, ntiles, G, T1, T2);
  double4 *raw = reinterpret_cast<double4 *>(gsm);                      // R records
  unsigned char *stage = reinterpret_cast<unsigned char *>(raw + R);    // R * SB, cell-sorted
  int *cnt = reinterpret_cast<int *>(stage + (size_t)R * SB);           // 128
  int *coff = cnt + kGrpThreads;                                        // 128: cell offsets
  int *tpre = coff + kGrpThreads;                                       // ntiles + 1
  int *spre = tpre + ntiles + 1;                                        // [2][G + 1]
  double *tacc = reinterpret_cast<double *>(
      gsm + 32 * (size_t)R + (size_t)R * SB + ((4 * (size_t)(2 * kGrpThreads + ntiles + 1 + 2 * (G + 1))) + 15) / 16 * 16);
  // kModeF64W: key | rank << 8 of each raw record (the records carry (x1, x2, w, y), no key)
  int *kr = reinterpret_cast<int *>(tacc + 2 * (size_t)(T1 + W - 1) * (T2 + W - 1));
  __shared__ int wsum_s[kAccGroups][8], total_s[kAccGroups], spre_tile_s[kAccGroups][2];
  __shared__ __align__(8) uint64_t bar_s[kAccGroups];
  int *wsum = wsum_s[gi], *spre_tile = spre_tile_s[gi];
  int &total = total_s[gi];
  uint64_t *bar = &bar_s[gi];
  const int NT = T1 * T2;
  const bool own = tid < NT;
  const int my_r = own ? tid / T2 : 0, my_c = own ? tid % T2 : 0;
  const int A1 = T1 + W - 1, A2 = T2 + W - 1;
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < 2 * A1 * A2; i += kGrpThreads) tacc[i] = 0.0;
  named_sync(bar_id, kGrpThreads);
  uint32_t phase = 0u;
  // optional phase timing (EFGP_SORTED_TRACE): cycles spent between the PH(i) marks, thread 0 of
  // each group, summed over the launch into trace[nchunks*G*4 + (blockIdx*2 + group)*8 + i]
  long long ph_t = clock64(), ph_acc[7] = {0, 0, 0, 0, 0, 0, 0};
#define PH(i)                                    \
  if (A.trace && tid == 0) {                     \
    const long long t_ = clock64();              \
    ph_acc[(i)] += t_ - ph_t;                    \
    ph_t = t_;                                   \
  }
  // register windows of this thread's start cell: fp64 (FP64 / FP32 modes) or fp32 pairs along b
  // (MIXED); the unused set is eliminated by the compiler
  double a1[W][W], ay[W][W];
#pragma unroll
  for (int a = 0; a < W; ++a)
#pragma unroll
    for (int b = 0; b < W; ++b) a1[a][b] = ay[a][b] = 0.0;
  float2 p1[W][(W + 1) / 2], py[W][(W + 1) / 2];
  int pend = 0;
#pragma unroll
  for (int a = 0; a < W; ++a)
#pragma unroll
    for (int b = 0; b < (W + 1) / 2; ++b) p1[a][b] = py[a][b] = make_float2(0.f, 0.f);

  // One round: wait for its records (raw[0..nr), bulk copies issued earlier), pass 1 (rank per start
  // cell), scan, pass 2 (cell-sorted stage), issue_next() (raw is free), phase C (register windows);
  // fold the windows into the fp64 tile accumulator if fold_req (or MIXED overflow), and flush the
  // tile accumulator (tile origin r0, c0 in start cells) into the fine grids if flush.
  auto round_body = [&](const int nr, auto &&issue_next, const bool fold_req, const bool flush, const int r0,
                        const int c0, auto &&on_landed) {
        cnt[tid] = 0;
        PH(0);
        if (nr > 0) {  // (nr = 0: a final fold / flush without records)
          mbar_wait(bar, phase);
          phase ^= 1u;
        }
        on_landed();  // the round's records are in shared memory
        named_sync(bar_id, kGrpThreads);
        PH(1);
        // pass 1 (thread per record): rank within its start cell (key from the binner), kept in
        // the record's key slot
        for (int j0 = tid; j0 < nr; j0 += 4 * kGrpThreads) {  // 4 records at a time (latency)
          int key[4], rnk[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = j0 + u * kGrpThreads;
            if constexpr (MODE == kModeF64W) {  // start cell recomputed from x (same roundings as the binner)
              if (j < nr) {
                const double4 rv = raw[j];
                const int i1 = start_cell<W>(grid_t(h, rv.x, n1)) - s_lo - r0;
                const int i2 = start_cell<W>(grid_t(h, rv.y, n1)) - s_lo - c0;
                EFGP_DCHECK(i1 >= 0 && i1 < T1 && i2 >= 0 && i2 < T2);
                key[u] = i1 * T2 + i2;
              } else {
                key[u] = -1;
              }
            } else {
              key[u] = j < nr ? __double2loint(raw[j].w) : -1;
            }
            EFGP_DCHECK(key[u] < NT);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) rnk[u] = key[u] >= 0 ? atomicAdd(&cnt[key[u]], 1) : 0;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = j0 + u * kGrpThreads;
            if (j < nr) {
              if constexpr (MODE == kModeF64W) kr[j] = key[u] | rnk[u] << 8;
              else reinterpret_cast<int *>(&raw[j].w)[1] = rnk[u];
            }
          }
        }
        named_sync(bar_id, kGrpThreads);
        const int mycnt = cnt[tid];
        if (tid < 32) {  // cell offsets: warp 0 scans the 128 counts (4 per lane)
          const int4 c4 = reinterpret_cast<const int4 *>(cnt)[tid];
          const int sum = c4.x + c4.y + c4.z + c4.w;
          int incl = sum;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (tid >= o) incl += v;
          }
          const int e = incl - sum;
          reinterpret_cast<int4 *>(coff)[tid] = make_int4(e, e + c4.x, e + c4.x + c4.y, e + c4.x + c4.y + c4.z);
        }
        named_sync(bar_id, kGrpThreads);
        PH(2);
        const int myoff = coff[tid];
        // pass 2 (thread per record): the record (FP64) or its fp32 weights at its sorted slot
#pragma unroll 2
        for (int j = tid; j < nr; j += kGrpThreads) {
          const double4 rv = raw[j];
          const int kk = MODE == kModeF64W ? (kr[j] & 0xFF) : __double2loint(rv.w);
          const int rr = MODE == kModeF64W ? (kr[j] >> 8) : __double2hiint(rv.w);
          EFGP_DCHECK(kk >= 0 && kk < NT && rr >= 0 && coff[kk] + rr < nr);
          unsigned char *st = stage + (size_t)(coff[kk] + rr) * SB;
          if constexpr (MODE == kModeF64W) {
            double s1, s2;
            es_reduce<W>(grid_t(h, rv.x, n1), s1);
            es_reduce<W>(grid_t(h, rv.y, n1), s2);
            double wz = rv.z, wy = rv.w;
            if (wraw) {  // raw (sigma_n, y_n) -> strengths 1/sigma_n^2 and y_n/sigma_n^2 (k_het_prep's roundings: y_n * rcp(sigma_n^2))
              wz = __drcp_rn(rv.z * rv.z);  // one IEEE reciprocal, then a product (k_het_prep: the same)
              wy = rv.w * wz;
            }
            reinterpret_cast<double4 *>(st)[0] = make_double4(s1, s2, wz, wy);  // (s1, s2, w, y)
          } else if constexpr (MODE == kModeF64) {
            // the reduced coordinates s1, s2 (es_reduce) are computed here, in the load-balanced
            // thread-per-record pass, instead of in phase C (thread per cell, Poisson-imbalanced)
            double *d = reinterpret_cast<double *>(st);
            double s1, s2;
            es_reduce<W>(grid_t(h, rv.x, n1), s1);
            es_reduce<W>(grid_t(h, rv.y, n1), s2);
            d[0] = s1;
            d[1] = s2;
            d[2] = rv.z;
          } else {
            constexpr int WP = (W + 1) / 2, WE = 2 * WP, NF = SB / 4;
            float2 w1[WP], w2[WP];
            es_weights_pairs<W>(grid_t(h, rv.x, n1), PF, w1);
            es_weights_pairs<W>(grid_t(h, rv.y, n1), PF, w2);
            float f[NF];
#pragma unroll
            for (int q = 0; q < WP; ++q) {
              f[2 * q] = w1[q].x;
              f[2 * q + 1] = w1[q].y;
              f[WE + 2 * q] = w2[q].x;
              f[WE + 2 * q + 1] = w2[q].y;
            }
#pragma unroll
            for (int i = 2 * WE; i < NF; ++i) f[i] = 0.f;
            if constexpr (MODE == kModeA32) {
              f[StageRec<W, MODE>::kYSlot] = (float)rv.z;
            } else {
              f[2 * WE] = __int_as_float(__double2loint(rv.z));
              f[2 * WE + 1] = __int_as_float(__double2hiint(rv.z));
            }
            float4 *q4 = reinterpret_cast<float4 *>(st);
#pragma unroll
            for (int i = 0; i < NF / 4; ++i) q4[i] = make_float4(f[4 * i], f[4 * i + 1], f[4 * i + 2], f[4 * i + 3]);
          }
        }
        named_sync(bar_id, kGrpThreads);
        PH(3);
        issue_next();  // raw is free: the next round's copies land during phase C
        // phase C (thread per start cell): register accumulation of its records
        if (mycnt > 0) {
          const unsigned char *sp = stage + (size_t)myoff * SB;
          if constexpr (MODE == kModeF64 || MODE == kModeF64W) {
#pragma unroll 2
            for (int q = 0; q < mycnt; ++q, sp += SB) {
              const double *d = reinterpret_cast<const double *>(sp);
              const double yv = MODE == kModeF64W ? d[3] : d[2];
              const double wv = MODE == kModeF64W ? d[2] : 1.0;  // strength-1 weight (NEXT-3: 1/sigma_n^2)
              double w1[W], w2[W];
              es_weights_s<W>(d[0], P, w1);
              es_weights_s<W>(d[1], P, w2);
#pragma unroll
              for (int a = 0; a < W; ++a) {
                const double ca = MODE == kModeF64W ? wv * w1[a] : w1[a], cy = yv * w1[a];
#pragma unroll
                for (int b2 = 0; b2 < W; ++b2) {
                  a1[a][b2] = fma(ca, w2[b2], a1[a][b2]);
                  ay[a][b2] = fma(cy, w2[b2], ay[a][b2]);
                }
              }
            }
          } else if constexpr (MODE == kModeW32) {
            constexpr int WE = StageRec<W, MODE>::WE, NF = SB / 4;
#pragma unroll 2
            for (int q = 0; q < mycnt; ++q, sp += SB) {
              float f[NF];
              load_floats<SB>(sp, f);
              const double yv = __hiloint2double(__float_as_int(f[2 * WE + 1]), __float_as_int(f[2 * WE]));
              double w2[W];
#pragma unroll
              for (int b2 = 0; b2 < W; ++b2) w2[b2] = (double)f[WE + b2];
#pragma unroll
              for (int a = 0; a < W; ++a) {
                const double ca = (double)f[a], cy = yv * ca;
#pragma unroll
                for (int b2 = 0; b2 < W; ++b2) {
                  a1[a][b2] = fma(ca, w2[b2], a1[a][b2]);
                  ay[a][b2] = fma(cy, w2[b2], ay[a][b2]);
                }
              }
            }
          } else {
            // MIXED: fp32 pairs along b: (acc[a][2p], acc[a][2p+1]) += w1[a] * (w2[2p], w2[2p+1])
            constexpr int WP = (W + 1) / 2, WE = 2 * WP, NF = SB / 4;
#pragma unroll 2
            for (int q = 0; q < mycnt; ++q, sp += SB) {
              float f[NF];
              load_floats<SB>(sp, f);
              const float yf = f[StageRec<W, MODE>::kYSlot];
#pragma unroll
              for (int a = 0; a < W; ++a) {
                const float c1 = f[a], cy = yf * f[a];
#pragma unroll
                for (int pp = 0; pp < WP; ++pp) {
                  const float2 w2p = make_float2(f[WE + 2 * pp], f[WE + 2 * pp + 1]);
                  p1[a][pp] = __ffma2_rn(w2p, make_float2(c1, c1), p1[a][pp]);
                  py[a][pp] = __ffma2_rn(w2p, make_float2(cy, cy), py[a][pp]);
                }
              }
            }
          }
        }
        // MIXED: the fp32 windows of one tile segment sum at most 64 points per start cell; past that
        // (only for very concentrated data) they are folded into the fp64 tile accumulator early
        PH(4);
        bool fold_now = fold_req;
        if constexpr (MODE == kModeA32) {
          pend += mycnt;
          fold_now = named_sync_or(bar_id, kGrpThreads, pend >= 64) || fold_now;
        } else {
          named_sync(bar_id, kGrpThreads);  // stage and cnt free
        }
        if (fold_now) {
          // add the windows into the fp64 tile accumulator in W^2 conflict-free steps
#pragma unroll
          for (int a = 0; a < W; ++a) {
#pragma unroll
            for (int b2 = 0; b2 < W; ++b2) {
              if (own) {
                const int idx = (my_r + a) * A2 + (my_c + b2);
                if constexpr (MODE == kModeA32) {
                  const float2 v1 = p1[a][b2 / 2], vy = py[a][b2 / 2];
                  tacc[idx] += (double)((b2 & 1) ? v1.y : v1.x);
                  tacc[A1 * A2 + idx] += (double)((b2 & 1) ? vy.y : vy.x);
                } else {
                  tacc[idx] += a1[a][b2];
                  tacc[A1 * A2 + idx] += ay[a][b2];
                }
              }
              named_sync(bar_id, kGrpThreads);
            }
          }
          if constexpr (MODE == kModeA32) {
#pragma unroll
            for (int a = 0; a < W; ++a)
#pragma unroll
              for (int pp = 0; pp < (W + 1) / 2; ++pp) p1[a][pp] = py[a][pp] = make_float2(0.f, 0.f);
            pend = 0;
          } else {
#pragma unroll
            for (int a = 0; a < W; ++a)
#pragma unroll
              for (int b2 = 0; b2 < W; ++b2) a1[a][b2] = ay[a][b2] = 0.0;
          }
        }
        PH(5);
        // end of a tile segment: one RED per cell of the tile accumulator, which is re-zeroed
        if (flush) {
          for (int i = tid; i < A1 * A2; i += kGrpThreads) {
            const double v1 = tacc[i], vy = tacc[A1 * A2 + i];
            const int r = wrap_s(s_lo + r0 + i / A2, n1), c = wrap_s(s_lo + c0 + i % A2, n1);
            const int64_t gidx = (int64_t)r * n1 + c;
            if (v1 != 0.0) atomicAdd(A.g1 + gidx, v1);
            if (vy != 0.0) atomicAdd(A.gy + gidx, vy);
            tacc[i] = tacc[A1 * A2 + i] = 0.0;
          }
          named_sync(bar_id, kGrpThreads);
        }
  };

  // Static ownership (A.own: ntiles <= grid, the c5 geometry): CTA b owns tile b for the whole call;
  // its group g consumes the segments of the binner CTAs p = g, g + 2, ... of tile b, chunk after
  // chunk, as ONE stream: rounds of R records may span chunk boundaries, the windows are never folded
  // before the end (no tile switches), and a chunk's lists are released (acc_done) as soon as this
  // group's rounds have read them.  With small chunks the record lists stay L2-resident.
  auto accumulate_static = [&]() {
    const int t = blockIdx.x;
    if (t >= ntiles) return;  // no tile (not counted among the consumers)
    const int np = (G - gi + 1) / 2;  // producers p = gi + 2 j, j < np
    int *spk = spre;                  // [3][np + 1] segment prefixes of chunks k (slot k % 3)
    __shared__ int tot_s[kAccGroups][3], nr_s[kAccGroups], fin_s[kAccGroups][4];
    int *tot = tot_s[gi];
    if (A.debug & 1) {  // diagnostics: accumulators skip their work, release every chunk
      for (int k = 0; k < A.nchunks; ++k) {
        if (tid == 0) {
          spin_until(A.bin_done + k, G);
          __threadfence();
          atomicAdd(A.acc_done + k, 1u);
        }
      }
      return;
    }
    // warp-0 state (uniform across its lanes): read cursor and prepared chunks
    int kc = 0, pc = 0, kprep = -1;
    auto prepare = [&](int k) {  // warp 0: wait until chunk k is binned, prefix of my segments
      if (tid == 0) spin_until(A.bin_done + k, G);
      __syncwarp();
      asm volatile("fence.proxy.async.global;" ::: "memory");
      const int *segc = A.segcnt + ((int64_t)k * ntiles + t) * G;
      int *sp = spk + (k % 3) * (np + 1);
      const int per = (np + 31) / 32, beg = tid * per, end = min(np, beg + per);
      int sum = 0;
      for (int j = beg; j < end; ++j) sum += __ldcg(segc + gi + 2 * j);
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (tid >= o) incl += v;
      }
      int run = incl - sum;
      for (int j = beg; j < end; ++j) {
        sp[j] = run;
        run += __ldcg(segc + gi + 2 * j);
      }
      const int total_k = __shfl_sync(0xffffffffu, incl, 31);
      if (tid == 31) sp[np] = incl;
      if (tid == 0) tot[k % 3] = total_k;
      __syncwarp();
      kprep = k;
    };
    // warp 0: plan the next round (up to R records from the stream, at most 3 chunk pieces), arm the
    // mbarrier and issue one bulk copy per (chunk, producer) piece; nr_s / fin_s get the round's
    // size and the chunks it finishes
    auto plan_issue = [&]() {
      if (tid >= 32) return;
      int nr = 0, nfin = 0, nrng = 0;
      int rk[3], ra[3], rt[3], rd[3];
      int fin[4];
      while (nr < R && kc < A.nchunks && nrng < 3 && nfin < 4) {
        if (kprep < kc) prepare(kc);
        const int total_k = tot[kc % 3];
        const int take = min(R - nr, total_k - pc);
        if (take > 0) {
          rk[nrng] = kc;
          ra[nrng] = pc;
          rt[nrng] = take;
          rd[nrng] = nr;
          ++nrng;
          nr += take;
          pc += take;
        }
        if (pc < total_k) break;  // round full
        fin[nfin++] = kc;         // chunk kc exhausted by this round
        ++kc;
        pc = 0;
      }
      if (tid == 0) {
        nr_s[gi] = nr;
        for (int f = 0; f < 4; ++f) fin_s[gi][f] = f < nfin ? fin[f] : -1;
        if (nr > 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect(bar, (uint32_t)(nr * 32));
        }
      }
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      for (int q = 0; q < nrng; ++q) {
        const int k = rk[q], a = ra[q], a_end = a + rt[q];
        const int *sp = spk + (k % 3) * (np + 1);
        const double4 *base = A.rec[k % A.nbuf] + (int64_t)t * G * A.segcap;
        for (int j = tid; j < np; j += 32) {
          const int lo = max(a, sp[j]), hi = min(a_end, sp[j + 1]);
          if (hi > lo) {
            EFGP_DCHECK(rd[q] + (hi - a) <= R && hi - sp[j] <= A.segcap);
            bulk_g2s(raw + rd[q] + (lo - a), base + (int64_t)(gi + 2 * j) * A.segcap + (lo - sp[j]),
                     (uint32_t)((hi - lo) * 32), bar);
          }
        }
      }
    };
    const int r0 = (t / A.nt2) * T1, c0 = (t % A.nt2) * T2;
    plan_issue();
    named_sync(bar_id, kGrpThreads);
    int nr = nr_s[gi];
    int fin[4];
#pragma unroll
    for (int f = 0; f < 4; ++f) fin[f] = fin_s[gi][f];
    // a chunk is released as soon as the round that read its last records has landed (before the
    // next round is planned: a plan may wait for chunks whose buffers that release frees)
    auto release = [&] {
      if (tid == 0)
        for (int f = 0; f < 4; ++f)
          if (fin[f] >= 0) {
            __threadfence();
            atomicAdd(A.acc_done + fin[f], 1u);
          }
    };
    while (nr > 0) {
      round_body(nr, [&] { plan_issue(); }, false, false, r0, c0, release);
      // (round_body ends with a group barrier: nr_s / fin_s of the next round are visible)
      nr = nr_s[gi];
#pragma unroll
      for (int f = 0; f < 4; ++f) fin[f] = fin_s[gi][f];
      named_sync(bar_id, kGrpThreads);  // nr_s / fin_s reusable
    }
    release();  // chunks finished without records (empty tail)
    round_body(0, [] {}, true, true, r0, c0, [] {});  // fold the windows, flush the tile accumulator
  };

  if (A.own) {
    accumulate_static();
  } else {
  for (int k = 0; k < A.nchunks; ++k) {
    const double4 *rec = A.rec[k % A.nbuf];
    const int *segc = A.segcnt + (int64_t)k * ntiles * G;
    if (tid == 0) {
      if (gi == 0) stamp(A.trace, k, 1);
      spin_until(A.bin_done + k, G);
      if (gi == 0) stamp(A.trace, k, 2);
      asm volatile("fence.proxy.async.global;" ::: "memory");
      spre_tile[0] = spre_tile[1] = -1;
    }
    named_sync(bar_id, kGrpThreads);
    for (int t = tid; t < ntiles; t += kGrpThreads) tpre[t] = __ldcg(A.tilecnt + (int64_t)k * ntiles + t);
    named_sync(bar_id, kGrpThreads);
    group_scan_array<4>(tpre, ntiles, tid, wsum, bar_id, &total);
    if (tid == 0) tpre[ntiles] = total;
    named_sync(bar_id, kGrpThreads);
    const int all = tpre[ntiles];
    const int gb = (int)((int64_t)vb * all / VG), ge = (int)((int64_t)(vb + 1) * all / VG);
    if (gb < ge && !(A.debug & 1)) {
      int t_first;
      {
        int lo = 0, hi = ntiles;
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (tpre[mid] <= gb) lo = mid;
          else hi = mid;
        }
        t_first = lo;
        while (tpre[t_first + 1] <= gb) ++t_first;
      }
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
      // segment prefix of tile t into slot (t & 1), by the group's first warp (a barrier follows
      // before it is read)
      auto seg_prefix = [&](int t) {
        if (t < 0 || tid >= 32) return;
        const int sl = t & 1;
        if (spre_tile[sl] == t) return;
        int *sp = spre + sl * (G + 1);
        const int per = (G + 31) / 32, beg = tid * per, end = min(G, beg + per);
        int s = 0;
        for (int c = beg; c < end; ++c) s += __ldcg(segc + (int64_t)t * G + c);
        int incl = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (tid >= o) incl += v;
        }
        int run = incl - s;
        for (int c = beg; c < end; ++c) {
          sp[c] = run;
          run += __ldcg(segc + (int64_t)t * G + c);
        }
        if (tid == 31) sp[G] = incl;
        __syncwarp();
        if (tid == 0) spre_tile[sl] = t;
      };
      // bulk copies of round r into raw: one per (tile, binner CTA) segment piece it spans
      auto issue = [&](Rd r) {
        if (tid != 0 || r.tile < 0) return;
        const int *sp = spre + (r.tile & 1) * (G + 1);
        int lo2 = 0, hi2 = G;  // last segment with sp[c] <= r.lo
        while (hi2 - lo2 > 1) {
          const int mid = (lo2 + hi2) >> 1;
          if (sp[mid] <= r.lo) lo2 = mid;
          else hi2 = mid;
        }
        int c = lo2;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect(bar, (uint32_t)(r.n * 32));
        const double4 *tb = rec + (int64_t)r.tile * G * A.segcap;
        for (int done = 0; done < r.n; ++c) {
          const int a0 = r.lo + done - sp[c];
          const int m = min(sp[c + 1] - sp[c] - a0, r.n - done);
          if (m > 0) {
            EFGP_DCHECK(c < G && a0 >= 0 && a0 + m <= A.segcap && done + m <= R);
            bulk_g2s(raw + done, tb + (int64_t)c * A.segcap + a0, (uint32_t)(m * 32), bar);
            done += m;
          }
        }
      };
      Rd cur = round_at(t_first, gb - tpre[t_first]);
      seg_prefix(cur.tile);
      named_sync(bar_id, kGrpThreads);
      issue(cur);
      while (cur.tile >= 0) {
        const Rd nxt = next_round(cur);
        seg_prefix(nxt.tile);  // for issue(nxt) below
        round_body(cur.n, [&] { issue(nxt); }, nxt.tile != cur.tile, nxt.tile != cur.tile,
                   (cur.tile / A.nt2) * T1, (cur.tile % A.nt2) * T2, [] {});
        PH(6);
        cur = nxt;
      }
    }
    PH(0);  // (the chunk hand-off counts as waiting)
    // this group is done reading chunk k's lists
    named_sync(bar_id, kGrpThreads);
    if (tid == 0) {
      __threadfence();
      atomicAdd(A.acc_done + k, 1u);
      if (gi == 0) stamp(A.trace, k, 3);
    }
  }
  }  // share mode
  if (A.trace && tid == 0) {
    unsigned long long *o = A.trace + (size_t)A.nchunks * G * 4 + ((size_t)blockIdx.x * kAccGroups + gi) * 8;
    for (int i = 0; i < 7; ++i) o[i] = (unsigned long long)ph_acc[i];
  }
#undef PH
}

template <int W, int MODE>
__global__ void __launch_bounds__(kFusedThreads, 1) k_spread_fused(const FusedArgs A, const EsPoly P, const EsPolyP PF) {
  extern __shared__ __align__(16) unsigned char fsm[];
  const int tid = threadIdx.x;
  const size_t acc_bytes = 2 * AccSmem<W, MODE>::bytes(A.R, A.ntiles, gridDim.x, A.T1, A.T2);
  if (tid >= kAccThreads) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kBinRegs) : "memory");
    binner_role<W, MODE>(A, fsm + (acc_bytes + 15) / 16 * 16, tid - kAccThreads);
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kAccRegs) : "memory");
    accumulator_role<W, MODE>(A, fsm, tid, P, PF);
  }
}

template <int W, int MODE>
static size_t fused_smem_bytes(int R, int ntiles, int S, int grid, int T1, int T2) {
  return 2 * AccSmem<W, MODE>::bytes(R, ntiles, grid, T1, T2) + FusedSmem<W, MODE>::bin_bytes(ntiles, S);
}

static size_t fused_smem(int w, int mode, int R, int ntiles, int S, int grid, int T1, int T2) {
  switch (w) {
#define EFGP_SZ(WW)                                            \
  case WW:                                                     \
    return mode == 0   ? fused_smem_bytes<WW, 0>(R, ntiles, S, grid, T1, T2) \
           : mode == 1 ? fused_smem_bytes<WW, 1>(R, ntiles, S, grid, T1, T2) \
           : mode == 2 ? fused_smem_bytes<WW, 2>(R, ntiles, S, grid, T1, T2) \
                       : fused_smem_bytes<WW, 3>(R, ntiles, S, grid, T1, T2);
    EFGP_SZ(2) EFGP_SZ(3) EFGP_SZ(4) EFGP_SZ(5) EFGP_SZ(6)
#undef EFGP_SZ
  }
  return ~size_t(0);
}

// Tile shape (T1 x T2 start cells, T1 T2 <= 128, least covered area), chunk, capacity, round size.
bool sorted_geometry(Params &p, int num_sms) {
  p.s_lo = -(p.w / 2);
  const int hi0 = (int)std::ceil(p.h * p.n1 - 0.5 * p.w);
  p.s_count = hi0 - p.s_lo + 1;
  const int S = p.s_count;
  int64_t best = -1;
  for (int T2 = 4; T2 <= 32; ++T2) {
    const int T1 = std::min(kGrpThreads / T2, S);
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
    p.T2 = std::max(4, std::min(32, std::atoi(e)));
    p.T1 = std::min(kGrpThreads / p.T2, S);
    p.nt1 = (S + p.T1 - 1) / p.T1;
    p.nt2 = (S + p.T2 - 1) / p.T2;
  }
  p.ntiles = p.nt1 * p.nt2;
  // 32M points x 3 list buffers: fewer hand-offs, binning two chunks ahead (c5 N = 4e8: 3.76e10 ->
  // 3.86e10 points/s against 16M x 2; records are allocated per call for min(N, chunk) points)
  // static ownership: opt-in (EFGP_SORTED_OWN=1); measured slower than the equal-share mode on c5
  // (25.0 vs 24.0 ms at N = 1e9 with 3M-point chunks; per-chunk coupling of all CTAs dominates with
  // the small chunks that keep the lists in L2)
  p.sorted_own = p.ntiles <= num_sms && std::getenv("EFGP_SORTED_OWN") && std::atoi(std::getenv("EFGP_SORTED_OWN"));
  // the equal-share mode amortises its per-chunk tile switches over large chunks
  p.chunk = p.sorted_own ? int64_t(3) << 20 : int64_t(1) << 25;
  if (const char *e = std::getenv("EFGP_SORTED_CHUNK"))
    p.chunk = std::max<int64_t>(kWBatch, std::atoll(e) / kWBatch * kWBatch);
  p.nbuf = 3;
  if (const char *e = std::getenv("EFGP_SORTED_NBUF")) p.nbuf = std::max(2, std::min(kMaxNbuf, std::atoi(e)));
  p.tiles_grid = num_sms;
  if (const char *e = std::getenv("EFGP_SORTED_GRID")) p.tiles_grid = std::max(1, std::atoi(e));
  // capacity of a (tile, binner CTA) segment: 2x its uniform share + slack; overflow spills to
  // direct RED spreading (correct for any data)
  p.cap = 0;  // segment capacity: per call, from the call's effective chunk (sorted_segcap)
  // round size: the largest multiple of 128 whose shared memory fits 227 KB
  const size_t lim = 227 * 1024 - 256;
  int R = 0;
  for (int r = 256; r <= 16384; r += 128)
    if (fused_smem(p.w, p.spread_mode, r, p.ntiles, S, p.tiles_grid, p.T1, p.T2) <= lim) R = r;
  if (const char *e = std::getenv("EFGP_SORTED_R")) R = std::max(256, std::min(R, std::atoi(e) / 128 * 128));
  p.round = R;
  // the weighted one-pass mode (kModeF64W, NEXT-3) stages 8 more bytes per point and record
  p.round_w = 0;
  for (int r = 256; r <= 16384; r += 128)
    if (fused_smem(p.w, kModeF64W, r, p.ntiles, S, p.tiles_grid, p.T1, p.T2) <= lim) p.round_w = r;
  return R >= 256;  // otherwise the lists / tables do not leave room for a round: use another method
}

// capacity of a (tile, binner CTA) segment for chunks of `chunk` points: 2x the uniform share +
// slack; a fuller segment spills its points to direct RED spreading (correct for any data)
static int sorted_segcap(const Params &p, int64_t chunk) {
  const double share = (double)chunk * p.T1 * p.T2 / ((double)p.s_count * p.s_count) / p.tiles_grid;
  return (int)std::min<double>((double)chunk, 2.0 * share + 256.0);
}

template <int W, int MODE>
static efgp_status launch_fused(efgp_plan *pl, const FusedArgs &A, cudaStream_t s) {
  const Params &P = pl->P;
  const size_t sm = fused_smem_bytes<W, MODE>(A.R, A.ntiles, A.S, P.tiles_grid, A.T1, A.T2);
  auto kern = k_spread_fused<W, MODE>;
  EFGP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int per_sm = 0;
  EFGP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kFusedThreads, sm));
  if (per_sm < 1) {
    pl->err = "SORTED spreading kernel does not fit on an SM";
    return EFGP_ERR_RESOURCE;
  }
  const int grid = P.tiles_grid;  // the segment layout was sized for exactly this many CTAs
  if (grid > pl->num_sms * per_sm) {
    pl->err = "SORTED spreading: not all CTAs can be co-resident";
    return EFGP_ERR_RESOURCE;
  }
  FusedArgs a = A;
  EsPoly poly = P.poly;
  EsPolyP polyf = P.polyp;
  void *args[] = {(void *)&a, (void *)&poly, (void *)&polyf};
  // cooperative launch: all CTAs are co-resident (they wait on one another through global counters).
  // If the device cannot host them all right now (e.g. SMs taken by other work), report it so the
  // caller spreads this call with the GLOBAL method instead.
  const cudaError_t e = cudaLaunchCooperativeKernel((const void *)kern, dim3(grid), dim3(kFusedThreads), args, sm, s);
  if (e == cudaErrorCooperativeLaunchTooLarge) {
    cudaGetLastError();
    return EFGP_ERR_RESOURCE;
  }
  EFGP_CUDA(e);
  return EFGP_OK;
}

efgp_status spread_sorted2(efgp_plan *pl, const double *x, const double *y, int64_t N, cudaStream_t s,
                           const double *s1, unsigned long long *raw_minbits) {
  const Params &P = pl->P;
  FusedArgs A{};
  A.x = x;
  A.y = y;
  A.N = N;
  // effective chunk of this call (a small problem is one chunk) and its list buffers
  const int64_t chunk = std::min<int64_t>(P.chunk, (N + kWBatch - 1) / kWBatch * kWBatch);
  const int segcap = sorted_segcap(P, chunk);
  const size_t rec_need = (size_t)P.ntiles * P.tiles_grid * segcap;
  if (rec_need >= ((size_t)1 << 31)) {  // the binner addresses a list buffer with 32-bit record offsets
    pl->err = "internal: SORTED list buffer over 2^31 records";
    return EFGP_ERR_RESOURCE;
  }
  if (rec_need > pl->rec_cap) {
    for (int k = 0; k < kMaxNbuf; ++k) {
      if (pl->rec[k]) cudaFree(pl->rec[k]);
      pl->rec[k] = nullptr;
    }
    pl->rec_cap = 0;
    for (int k = 0; k < P.nbuf; ++k) EFGP_CUDA(cudaMalloc((void **)&pl->rec[k], rec_need * sizeof(double4)));
    pl->rec_cap = rec_need;
  }
  A.chunk = chunk;
  A.nchunks = (int)((N + chunk - 1) / chunk);
  A.tail_b0 = INT64_MAX;
  {
    // A run ends one chunk's accumulation after its last chunk is binned.  With few chunks that drain
    // is a large share of the run, so the last C..2C batches are cut into chunks of 1/2, 1/4, 1/8,
    // 1/16, 1/16 of that tail (the drain shrinks 8-16x for 4 more chunk hand-offs).  Measured (c5,
    // profiles/r02_sorted_tail_ab.log): N = 4e7 1.44 -> 1.32 ms; N = 1e9 (30 chunks) 23.99 -> 24.16 ms
    // and N = 1e6 0.09 -> 0.18 ms (a hand-off costs ~20 us), so it is on for at most 4 full chunks
    // before the tail and pieces of >= 1M points.  EFGP_SORTED_TAIL=0 / 1: never / whenever the
    // smallest piece has >= 16 batches (tests).
    const int64_t C = chunk / kWBatch, nb = (N + kWBatch - 1) / kWBatch;
    const char *e = std::getenv("EFGP_SORTED_TAIL");
    const int force = e ? std::atoi(e) : -1;
    if (force != 0 && !P.sorted_own && nb >= C && C > 0) {
      const int64_t kf = nb / C - 1, Lt = nb - kf * C;  // Lt in [C, 2C)
      if (force > 0 ? Lt / 16 >= 16 : (kf <= 3 && Lt / 16 >= 4096)) {
        A.tail_b0 = kf * C;
        A.tail_k0 = (int)kf;
        A.tail_c[0] = Lt / 2;
        A.tail_c[1] = Lt / 2 + Lt / 4;
        A.tail_c[2] = A.tail_c[1] + Lt / 8;
        A.tail_c[3] = A.tail_c[2] + Lt / 16;
        A.nchunks = (int)kf + 5;
      }
    }
  }
  A.nbuf = P.nbuf;
  A.debug = std::getenv("EFGP_SORTED_DEBUG") ? std::atoi(std::getenv("EFGP_SORTED_DEBUG")) : 0;
  A.own = P.sorted_own && P.ntiles <= P.tiles_grid;
  A.nconsumers = A.own ? 2u * (unsigned)P.ntiles : 2u * (unsigned)P.tiles_grid;
  A.h = P.h;
  A.n1 = (int)P.n1;
  A.s_lo = P.s_lo;
  A.S = P.s_count;
  A.T1 = P.T1;
  A.T2 = P.T2;
  A.nt2 = P.nt2;
  A.ntiles = P.ntiles;
  A.segcap = segcap;
  A.s1 = s1;
  A.wraw = s1 && raw_minbits ? 1 : 0;
  A.minbits = raw_minbits;
  A.R = s1 ? P.round_w : P.round;
  if (s1 && (P.spread_mode != kModeF64 || A.R < 256)) return EFGP_ERR_RESOURCE;  // caller: two passes
  for (int b = 0; b < kMaxNbuf; ++b) A.rec[b] = pl->rec[b];
  // per-chunk segment and tile lengths and the two handshake counters, zeroed for this call
  const int G = P.tiles_grid;
  const size_t need = (size_t)A.nchunks * ((size_t)P.ntiles * G + P.ntiles + 2);
  if (need > pl->sync_cap) {
    if (pl->sync_buf) cudaFree(pl->sync_buf);
    pl->sync_buf = nullptr;
    pl->sync_cap = 0;
    EFGP_CUDA(cudaMalloc((void **)&pl->sync_buf, need * sizeof(int)));
    pl->sync_cap = need;
  }
  EFGP_CUDA(cudaMemsetAsync(pl->sync_buf, 0, need * sizeof(int), s));
  A.segcnt = pl->sync_buf;
  A.tilecnt = A.segcnt + (size_t)A.nchunks * P.ntiles * G;
  A.bin_done = reinterpret_cast<unsigned *>(A.tilecnt + (size_t)A.nchunks * P.ntiles);
  A.acc_done = A.bin_done + A.nchunks;
  A.trace = nullptr;
  if (std::getenv("EFGP_SORTED_TRACE")) {
    const size_t tn = (size_t)A.nchunks * G * 4 + (size_t)G * kAccGroups * 8 + (size_t)G * kBinWarps * 8;
    if (tn > pl->trace_cap) {
      if (pl->trace) cudaFree(pl->trace);
      EFGP_CUDA(cudaMalloc((void **)&pl->trace, tn * sizeof(unsigned long long)));
      pl->trace_cap = tn;
    }
    EFGP_CUDA(cudaMemsetAsync(pl->trace, 0, tn * sizeof(unsigned long long), s));
    A.trace = pl->trace;
    pl->trace_n = tn;
  }
  A.poly_dev = pl->poly_dev;
  A.g1 = pl->g1;
  A.gy = pl->g2;
  A.err = pl->dflags;
  const int mode = s1 ? kModeF64W : P.spread_mode;
  switch (P.w) {
#define EFGP_CASE(WW)                                  \
  case WW:                                             \
    return mode == 0   ? launch_fused<WW, 0>(pl, A, s) \
           : mode == 1 ? launch_fused<WW, 1>(pl, A, s) \
           : mode == 2 ? launch_fused<WW, 2>(pl, A, s) \
                       : launch_fused<WW, 3>(pl, A, s);
    EFGP_CASE(2) EFGP_CASE(3) EFGP_CASE(4) EFGP_CASE(5) EFGP_CASE(6)
#undef EFGP_CASE
  }
  pl->err = "internal: SORTED spreading needs w <= 6";
  return EFGP_ERR_INVALID;
}

}  // namespace efgp
