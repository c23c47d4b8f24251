// Internal declarations of the EFGP sm_100a library (not part of the C ABI; see include/efgp.h).
#pragma once
#include <cuda_runtime.h>
#include <cufft.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/efgp.h"

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges cost a few ns without a tool attached

namespace efgp {
// NVTX range for the scope of a C-ABI call or one of its phases (nsys / ncu --nvtx timelines)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};
}  // namespace efgp

namespace efgp {

constexpr double kPi = 3.14159265358979323846;
constexpr int kMaxW = 16;  // ES kernel width for nufft_tol down to 1e-15
constexpr int kMaxNbuf = 8;  // SORTED spreading: record-list buffers in flight (at most)
#ifndef EFGP_TOEP_SPLITS
#define EFGP_TOEP_SPLITS 8
#endif
constexpr int kToepSplitsHost = EFGP_TOEP_SPLITS;  // k1 splits of the split direct Toeplitz product (cg.cu kToepSplits)

// Degree of the piecewise-polynomial ES kernel per cell offset: degree W already gives the aliasing
// error of the exact ES kernel to within 2 % for W >= 4 (the deconvolution tables are the
// polynomial's own Fourier transform); narrower kernels keep W + 2.
__host__ __device__ constexpr int es_degree(int W) { return W >= 4 ? W : W + 2; }

// Piecewise-polynomial ES kernel weights (degree es_degree(w) in s = 2u-1 per cell offset a), passed
// to the kernels by value (lives in the constant bank).
struct EsPoly {
  double c[kMaxW][kMaxW + 3];
  int deg;
};
struct EsPolyF {  // the same coefficients rounded to fp32 (fp32-weight spreading)
  float c[kMaxW][kMaxW + 3];
};
struct EsPolyP {  // fp32 coefficients of cell offsets (2q, 2q+1) as pairs (pad offset W: 0); W <= 6
  float2 c[3][9 + 1];
};

// Host-side parameter record.
struct Params {
  int kernel = EFGP_SE;
  double nu = 0, ell = 0, sigma = 0, eps = 0;
  int d = 1;
  double h = 0;
  int64_t m = 0;
  int64_t M = 0;        // (2m+1)^d
  int64_t Mh = 0;       // (2m+1)^(d-1) (m+1): Hermitian half of J_m (j_d >= 0)
  int64_t Kvh = 0;      // (4m+1)^(d-1) (2m+1): Hermitian half of J_2m
  double cg_tol = 0;
  int64_t max_iter_opt = 0;
  double nufft_tol = 0;
  int w = 0;            // ES width in cells
  double beta_es = 0;   // ES shape
  int64_t n1 = 0;       // type-1 fine grid for v (modes J_2m), per dim
  int64_t n2 = 0;       // type-1 fine grid for F^*y and type-2 grid (modes J_m), per dim
  int64_t L = 0;        // Toeplitz FFT box per dim (>= 4m+1)
  int64_t n_rhs = 0;    // grid of the strength-y spread: n1 (SORTED) or n2
  int rescale = EFGP_RESCALE_L2;
  int spread_method = EFGP_SPREAD_AUTO;  // resolved at setup (never AUTO afterwards)
  int spread_method_requested = EFGP_SPREAD_AUTO;
  bool sorted_disabled = false;          // SORTED geometry does not fit: resolve to another method
  int graph_iters = 8;
  EsPoly poly{};
  EsPolyF polyf{};
  EsPolyP polyp{};
  int hetero_method = 0;       // NEXT-3: 0 auto, 1 weighted Toeplitz (G11b), 2 NUFFT pair per iteration
  int precond = 0;             // NEXT-4: 0 none (Alg a1's plain CG), 1 Kronecker (reading G12)
  int spread_mode = 0;         // SORTED precision: 0 fp64, 1 fp32 weights, 2 fp32 weights + round sums
  // SORTED spreading geometry (2D)
  int s_lo = 0, s_count = 0;   // start cells i0 in [s_lo, s_lo + s_count) per dim
  int T1 = 8, T2 = 16;         // tile of T1 x T2 start cells (T1 T2 <= 128)
  int nt1 = 0, nt2 = 0, ntiles = 0;
  int cap = 0;                 // records per (tile, binner CTA) segment per chunk
  int round = 0;               // records per shared-memory round
  int round_w = 0;             // ... of the weighted one-pass mode (NEXT-3)
  int tiles_grid = 0;          // CTAs of the fused spreading kernel (<= one per SM)
  int nbuf = 2;                // tile-list buffers in flight
  int64_t chunk = 0;           // points per chunk
  bool sorted_own = false;     // static tile ownership (CTA b accumulates tile b)
};

// host_setup.cu
std::string validate_and_choose(Params &p, const efgp_options &opt);
double khat_host(const Params &p, double xi_norm);
int64_t next_smooth(int64_t n);                              // smallest 2^a 3^b 5^c 7^d >= n
void gauss_legendre(int n, std::vector<double> &x, std::vector<double> &w);
// phihat[k] = alpha * int_{-1}^{1} exp(beta (sqrt(1 - z^2) - 1)) cos(k alpha z) dz, alpha = w pi / n
std::vector<double> es_fourier_table(int w, double beta, int64_t n, int64_t kmax);
void es_poly_fit(int w, double beta, EsPoly &out);
double es_poly_eval(const EsPoly &P, int a, double u);
std::vector<double> es_fourier_table_poly(const EsPoly &P, int w, int64_t n, int64_t kmax);
// spread.cu: choose the spreading strategy (sets spread_method, n_rhs)
void resolve_spread_method(Params &p);
// spread_sorted.cu: tile geometry of the SORTED strategy
bool sorted_geometry(Params &p, int num_sms);  // false: no room for a round

struct DevBuf {
  void *ptr = nullptr;
  size_t bytes = 0;
};

}  // namespace efgp

struct efgp_plan {
  efgp::Params P;
  cudaStream_t stream = nullptr;       // internal non-blocking stream: all library work (capturable)
  cudaStream_t ustream = nullptr;      // caller's stream (options.stream): ordering at entry/exit only
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  int device = 0;
  int num_sms = 148;
  std::string err;

  // tables
  double *D_half = nullptr;   // Mh spectral weights (eq 117) on the J_m half
  double *psi1 = nullptr;     // ES Fourier transform, grid n1, k = 0..2m
  double *psi2 = nullptr;     // grid n2, k = 0..m
  efgp::EsPoly *poly_dev = nullptr;  // the kernel-weight polynomial in global memory

  // type-1 grids and spectra
  double *g1 = nullptr;       // n1^d real
  double *g2 = nullptr;       // n2^d real
  double2 *G1h = nullptr;     // n1^(d-1) (n1/2+1)
  double2 *G2h = nullptr;     // n2^(d-1) (n2/2+1)
  double *modes = nullptr;    // local partial modes: v half (Kvh cplx) | F^*y half (Mh cplx)
  double *modes_sum = nullptr;

  // Toeplitz operator and CG state
  double2 *Xbox = nullptr;    // L^(d-1) (L/2+1) complex, C2R input
  double *Yr = nullptr;       // L^d real
  double *vhat = nullptr;     // L^d real, C2R(v)/L^d
  double2 *vfull = nullptr;   // (4m+1)^2 complex, full v (direct Toeplitz product, small m, 2D)
  double2 *dft_V = nullptr;   // persistent DFT CG: (4m+1) x L, Vt[d1][x2] = sum_d2 v_{d1,d2} w^(-d2 x2), w = e^(2 pi i/L)
  double2 *dft_roots = nullptr;  // L: w^t
  double2 *dft_W = nullptr;   // (2m+1) x L: the product's per-line stage (columns -> rows exchange)
  unsigned *cg_gbar = nullptr;    // persistent direct CG: software grid-barrier counter
  int cg_persist_split = 0;       // k1 splits of the last persistent direct CG launch (0: not used)
  int cg_dft2 = 0;                // 1: the last CG ran the persistent DFT kernel (2D, m beyond the direct product)
  double2 *toep_part = nullptr;  // split direct product: (2m+1) x kToepSplitsHost x (m+1) partial rows
  unsigned *toep_cnt = nullptr;  // per output row: splits done (reset by the row's last CTA)
  double2 *Zbox = nullptr;    // R2C output
  // partial-transform Toeplitz product (toeplitz_pt, cg.cu): (m+1) slabs of L^(d-1) complex each
  double2 *pt_P = nullptr;    // D p scattered at the J_m bins (zeros elsewhere, set once)
  double2 *pt_T = nullptr;    // inverse DFT over the first d-1 axes; reused for the forward output
  double2 *pt_W = nullptr;    // per-line convolution along the last axis
  double2 *pt_V = nullptr;    // (3m+1) slabs: L^(1-d) x inverse DFT of v over the first d-1 axes
  cufftHandle plan_pt = 0, plan_ptv = 0;  // batched (d-1)-dim Z2Z, batch m+1 / 3m+1
  double2 *b = nullptr, *x = nullptr, *r = nullptr, *p = nullptr, *Ap = nullptr;  // Mh each
  double2 *p2 = nullptr;      // fused direct CG: second search-direction slot (Mh), zeroed at setup
  double *partials = nullptr; // 2 * cg_blocks
  double *scal = nullptr;     // device scalars (see cg.cu)
  double *hist = nullptr;     // residual history, hist_cap entries
  int64_t hist_cap = 0;
  int cg_blocks = 1;
  int *dflags = nullptr;      // [0] invalid-input flag
  double *h_pinned = nullptr; // small pinned host mirror of scalars/flags

  // type-2
  double2 *T2box = nullptr;   // n2^(d-1) (n2/2+1)
  double *t2grid = nullptr;   // n2^d real
  bool t2_valid = false;

  // host-input staging
  double *stage[2] = {nullptr, nullptr};
  int64_t stage_pts = 0;

  // SORTED spreading: per-chunk tile lists (nbuf buffers) of x pairs and y, and the per-call
  // list lengths + handshake counters of the fused kernel
  double4 *rec[efgp::kMaxNbuf] = {};  // ntiles x grid x segcap records (x1, x2, y, key)
  size_t rec_cap = 0;                              // records allocated per buffer
  int *sync_buf = nullptr;
  size_t sync_cap = 0;
  unsigned long long *trace = nullptr;  // EFGP_SORTED_TRACE: per-chunk, per-CTA role timestamps
  size_t trace_cap = 0, trace_n = 0;

  cufftHandle plan_g1 = 0, plan_g2 = 0, plan_c2r_L = 0, plan_r2c_L = 0, plan_t2 = 0;
  cudaGraphExec_t cg_exec = nullptr;

  // posterior variance (NEXT-2, variance.cu): batched CG buffers for var_B targets, created lazily
  int var_B = 0;
  double2 *var_x = nullptr, *var_r = nullptr, *var_p = nullptr, *var_Ap = nullptr;
  double2 *var_X = nullptr, *var_Z = nullptr;
  double *var_Y = nullptr;
  void *var_st = nullptr;
  cufftHandle plan_var_c2r = 0, plan_var_r2c = 0;
  cudaGraphExec_t var_exec = nullptr;
  int var_exec_max_iter = 0;
  int var_exec_pc = 0;  // the captured variance graph uses the preconditioned step
  double var_exec_sigma2 = -1;  // sigma2_sys baked into the captured variance graph
  bool var_pc = false;  // last predict_var used the Kronecker preconditioner
  int var_iters_max = 0;
  bool op_valid = false;  // the Toeplitz operator (vhat) of a fit is in place
  double sigma2_sys = 0;  // diagonal shift of the solved system: sigma^2, or 1 for (D T(v^w) D + I) (G11b)
  double cap_sigma = 0;   // sigma of the default CG cap: sigma, or min sigma_n
  double t_var = 0;
  int cg_exec_iters = 0;

  // heteroskedastic fit (NEXT-3, hetero.cu): type-2 on the strength-y spreading grid n_rhs when it
  // differs from n2 (so interpolation is the exact adjoint of spreading), created lazily
  double2 *het_box = nullptr;
  double *het_grid = nullptr;
  cufftHandle plan_het = 0;
  // NEXT-4 Kronecker preconditioner (precond.cu): eigenvectors/values of the d factors, work grids
  double2 *pc_Q = nullptr, *pc_F0 = nullptr, *pc_F1 = nullptr, *pc_work = nullptr, *z = nullptr;
  double *pc_lam = nullptr;
  double *pc_diag = nullptr;  // Jacobi: D_q^2 v_0 + sigma^2 on the half (reading G12b)
  int pc_used = 0;  // preconditioner of the last fit's solve (0 after a NUFFT-pair hetero fit)
  int *pc_info = nullptr;
  void *pc_solver = nullptr;  // cusolverDnHandle_t
  cudaGraphExec_t pcg_exec = nullptr;
  int pcg_exec_iters = 0;
  double pcg_exec_sigma2 = -1;  // sigma2_sys baked into the captured PCG graph (preconditioner scale)
  // NCCL communicator owned by the handle (comm.cu): efgp_fit sums the partial modes over ranks
  void *comm = nullptr;  // ncclComm_t
  int comm_size = 0, comm_rank = 0;
  double *comm_buf = nullptr;
  int het_path = 0;  // 1: last heteroskedastic fit used the sorted fused product
  cufftHandle plan_het_r2c = 0;  // D2Z on n2 (sorted path), created lazily
  // stream-ordered temporaries (hetero staging and sort, host-input chunks) come from this pool; it
  // keeps freed memory for the next call (release threshold = max) and is destroyed with the handle
  cudaMemPool_t pool = nullptr;

  // state of the last fit
  bool fitted = false;
  int64_t N_last = 0;
  int64_t iters = 0;
  double rel_resid = 0;
  int64_t max_iter_used = 0;
  int spread_used = 0;      // method that actually spread the last fit's points
  int spread_fallback = 0;  // efgp_spread_fallback: why it is not the planned method
  double t_spread = 0, t_modes = 0, t_solve = 0, t_predict = 0;
  cudaEvent_t ev[8] = {};
};

namespace efgp {
// spread.cu
// s1 (optional): per-point strength-1 weight (NEXT-3 one-pass: 1/sigma_n^2); only the SORTED and CELLSORT
// spreaders take it — elsewhere EFGP_ERR_RESOURCE (the caller spreads the two strengths separately)
// raw_minbits (optional, with s1): y and s1 are the RAW observations y_n and noise sds sigma_n; the SORTED
// kernel validates sigma_n (dflags[2]), takes min sigma_n into *raw_minbits (IEEE bits, preset to ~0)
// and forms the two strengths itself — no prep pass and no N-sized temporaries; SORTED only
efgp_status spread_points(efgp_plan *pl, const double *x, const double *y, int64_t N, cudaStream_t s,
                          const double *s1 = nullptr, unsigned long long *raw_minbits = nullptr);
efgp_status spread_begin(efgp_plan *pl, cudaStream_t s);
efgp_status spread_sorted2(efgp_plan *pl, const double *x, const double *y, int64_t N, cudaStream_t s,
                           const double *s1 = nullptr, unsigned long long *raw_minbits = nullptr);
// spread_cellsort.cu: K1 CELLSORT (2D any W, 3D W <= 6); EFGP_ERR_RESOURCE if not applicable
// w1 (optional): per-point weight of the strength-1 grid (default 1): the heteroskedastic TOEPLITZ
// solver spreads (1/sigma_n^2, y_n/sigma_n^2) in one pass
efgp_status spread_cellsort(efgp_plan *pl, const double *x, const double *y, int64_t N, cudaStream_t s,
                            const double *w1 = nullptr);
bool cellsort_geometry(const Params &p, int &lo, int &S, int &ncell);
// CTAs of the counting-sort kernels (count and scatter share the partition): one per SM.  Fewer CTAs
// keep fewer partially written 32-byte sectors open in L2 (the c3 scatter reads 4x and writes 3.5x
// its algorithmic bytes), but measured: 148 -> 17 CTAs made c3 slower (2.1 -> 2.8 ms) and the hetero
// sort 132 -> 119 ms only (profiles/r01_SUMMARY.md).  EFGP_SORT_CTAS overrides.
inline int sort_ctas(int num_sms) {
  const char *e = getenv("EFGP_SORT_CTAS");
  return (e && atoi(e) > 0) ? atoi(e) : num_sms;
}
// hetero.cu: counting-sort offset kernels (shared with CELLSORT)
__global__ void k_het_colscan(unsigned *__restrict__ hist, int nblk, int ncell, long long *__restrict__ tot);
__global__ void k_het_offsets(const long long *__restrict__ tot, int ncell, long long *__restrict__ off);
// modes.cu
// the CG's Toeplitz product by direct 2D convolution (one CTA per output row) instead of the padded
// real FFTs: (2m+1)^4 complex MACs per product, cheaper than four cuFFT launches for small m
inline bool toeplitz_direct(const Params &P) {
  const char *e = getenv("EFGP_TOEP_DIRECT");
  if (e && e[0] == '0') return false;
  if (P.d != 2 || P.m > 32) return false;
  // shared memory of k_cg_toep2 (1024 threads): u (n^2) + v rows (n (4m+1)) + partial sums
  const int64_t n = 2 * P.m + 1, nv = 4 * P.m + 1, nout = P.m + 1, slices = 1024 / ((nout + 3) / 4);
  return 16 * (n * n + n * nv + slices * nout) <= 220 * 1024;
}
// the CG's Toeplitz product for d >= 2 when the direct one does not apply (c2, c4): cuFFT over the
// first d-1 axes (batched over the m+1 half slabs of the last axis), direct 1D convolution along the
// last axis per line (cg.cu "partial-transform product"); EFGP_TOEP_PT=0 selects the padded real FFTs
inline bool toeplitz_pt(const Params &P) {
  const char *e = getenv("EFGP_TOEP_PT");
  if (e && e[0] == '0') return false;
  if (e && e[0] == '2') return P.d >= 2 && !toeplitz_direct(P);  // also 2D (c2: measured slower, 45 vs 27 us)
  return P.d == 3;
}
// 2D CG beyond the direct product's m (c2: m = 49): the whole CG as one cooperative kernel with the
// Toeplitz product by DFTs along the second axis and a direct convolution along the first (cg.cu
// "persistent DFT CG"); every CTA keeps r, p and D in shared memory, so M_h is bounded.
constexpr int kDft2MaxMh = 5100;  // 2 (r, p) x 16 B + 8 B (D) per entry, with the stages: <= 227 KB
inline bool toeplitz_dft2(const Params &P) {
  const char *e = getenv("EFGP_TOEP_DFT2");
  if (e && e[0] == '0') return false;
  return P.d == 2 && !toeplitz_direct(P) && P.Mh <= kDft2MaxMh;
}
efgp_status dft2_setup(efgp_plan *pl, cudaStream_t s);
efgp_status pt_setup(efgp_plan *pl, const double2 *vh, cudaStream_t s);
efgp_status type1_modes(efgp_plan *pl, double *modes_out, cudaStream_t s);
efgp_status toeplitz_setup(efgp_plan *pl, const double *modes, cudaStream_t s);
efgp_status type2_grid(efgp_plan *pl, cudaStream_t s);
efgp_status type2_grid_from(efgp_plan *pl, const double2 *beta, cudaStream_t s);
// deconvolved Hermitian-half modes over J_K of a half-spectrum box G of an n^d grid (K2 for one grid)
efgp_status type1_half(efgp_plan *pl, const double2 *G, int64_t n, int K, const double *psi, double2 *out,
                       cudaStream_t s);
efgp_status type2_grid_on(efgp_plan *pl, const double2 *beta, int64_t n, const double *psi, cufftHandle plan,
                          double2 *boxbuf, double *grid, cudaStream_t s);
// cg.cu
efgp_status cg_solve(efgp_plan *pl, int64_t N_total);
efgp_status pcg_solve(efgp_plan *pl, int64_t N_total);  // NEXT-4
// precond.cu (NEXT-4): build the Kronecker preconditioner from the fit's v; z = M^-1 r
efgp_status precond_setup(efgp_plan *pl, const double *modes);
efgp_status precond_apply(efgp_plan *pl, const double2 *r, double2 *z, const int *done, cudaStream_t s,
                          bool pdl = false);
typedef efgp_status (*CGOp)(efgp_plan *pl, const double2 *p, double2 *Ap, void *ctx);  // Ap = A p
efgp_status cg_solve_op(efgp_plan *pl, int64_t max_iter, CGOp op, void *ctx);
// interp.cu
efgp_status interp_targets(efgp_plan *pl, const double *xt, int64_t q, double *mu, cudaStream_t s);
// out_n = mu(x_n) / sd_n^2 (sd == nullptr: mu(x_n)) from the real type-2 fine grid `grid` (n^d)
efgp_status interp_weighted(efgp_plan *pl, const double *grid, int64_t n, const double *xt, int64_t q,
                            const double *sd, double *out, cudaStream_t s);
// hetero.cu (NEXT-3): fit with per-point noise; x, y, sd device-resident
efgp_status fit_hetero_device(efgp_plan *pl, const double *x, const double *y, const double *sd, int64_t N);
// comm.cu (multi-GPU plumbing; NCCL resolved at run time)
efgp_status comm_unique_id(void *id_out);
efgp_status comm_init(efgp_plan *pl, const void *id, int nranks, int rank);
void comm_destroy(efgp_plan *pl);
efgp_status comm_sum(efgp_plan *pl, double *buf, size_t n);
efgp_status comm_count_min(efgp_plan *pl, int64_t *count, double *minval, int *fail);
// variance.cu
efgp_status variance_targets(efgp_plan *pl, const double *xt, int64_t q, double *out, cudaStream_t s);
}  // namespace efgp

#define EFGP_CUDA(call)                                                                  \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      pl->err = std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " + __FILE__ + \
                ":" + std::to_string(__LINE__);                                          \
      return e_ == cudaErrorMemoryAllocation ? EFGP_ERR_RESOURCE : EFGP_ERR_CUDA;        \
    }                                                                                    \
  } while (0)

#define EFGP_CUFFT(call)                                                                 \
  do {                                                                                   \
    cufftResult r_ = (call);                                                             \
    if (r_ != CUFFT_SUCCESS) {                                                           \
      pl->err = std::string("cuFFT error ") + std::to_string((int)r_) + " at " + __FILE__ + \
                ":" + std::to_string(__LINE__);                                          \
      return r_ == CUFFT_ALLOC_FAILED ? EFGP_ERR_RESOURCE : EFGP_ERR_CUDA;               \
    }                                                                                    \
  } while (0)

// stream-ordered allocation from the handle's pool
#define EFGP_PALLOC(ptr, bytes, stream) \
  EFGP_CUDA(cudaMallocFromPoolAsync((void **)(ptr), (bytes), pl->pool, (stream)))

#define EFGP_TRY(call)                 \
  do {                                 \
    efgp_status s_ = (call);           \
    if (s_ != EFGP_OK) return s_;      \
  } while (0)

// ---- device-side invariant checks ------------------------------------------------------
// compute-sanitizer is closed on the GPU pool (profiles/r02_compute_sanitizer_closed.log), so the
// kernels carry their own bounds/invariant checks: built with -DEFGP_DEVICE_CHECKS=1 (tools/
// build_checked.sh) every EFGP_DCHECK prints the failed condition and traps; the default build
// compiles them out.
#ifndef EFGP_DEVICE_CHECKS
#define EFGP_DEVICE_CHECKS 0
#endif
#define EFGP_DCHECK(c)                                                                       \
  do {                                                                                       \
    if (EFGP_DEVICE_CHECKS && !(c)) {                                                        \
      printf("EFGP_DCHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, blockIdx.x, \
             threadIdx.x, #c);                                                               \
      __trap();                                                                              \
    }                                                                                        \
  } while (0)

// ---- device helpers shared by the kernels ------------------------------------------------
namespace efgp {

// ES kernel phi(z) = exp(beta (sqrt(1 - z^2) - 1)) on |z| <= 1 (FINUFFT's exponential of
// semicircle).  Evaluated directly in fp64 (reference; the kernels use es_weights).
__device__ __forceinline__ double es_kernel(double z, double beta) {
  double a = fma(-z, z, 1.0);
  a = a > 0.0 ? a : 0.0;
  return exp(beta * (sqrt(a) - 1.0));
}

// Weights of the W cells i0 .. i0+W-1 for a point at grid coordinate t: i0 = ceil(t - W/2),
// u = i0 - (t - W/2) in [0,1), w[a] = phi~_a(u) in s = 2u - 1 (degree es_degree(W)).  The ES kernel
// is even, so piece W-1-a is piece a mirrored, p_{W-1-a}(s) = p_a(-s) (es_poly_fit builds them so):
// with p_a = E_a(s^2) + s O_a(s^2), one even and one odd Horner in s^2 give both weights, half the
// FMAs of W separate Horner evaluations.
// Reduced coordinate of es_weights: i0 = ceil(t - W/2) (returned) and s = 2 (i0 - (t - W/2)) - 1.
template <int W>
__device__ __forceinline__ int es_reduce(double t, double &s) {
  const double tm = __dsub_rn(t, 0.5 * W);  // no FMA contraction: the SORTED binning must agree
  const double i0 = ceil(tm);
  s = 2.0 * (i0 - tm) - 1.0;
  return (int)i0;
}

// The W weights from the reduced coordinate s (es_weights = es_reduce + es_weights_s).
template <int W>
__device__ __forceinline__ void es_weights_s(double s, const EsPoly &P, double (&w)[W]) {
  const double s2 = s * s;
  constexpr int D = es_degree(W);
  constexpr int DE = D & ~1, DO = (D & 1) ? D : D - 1;  // highest even / odd power
#pragma unroll
  for (int a = 0; a < W / 2; ++a) {
    double e = P.c[a][DE], o = P.c[a][DO];
#pragma unroll
    for (int k = DE - 2; k >= 0; k -= 2) e = fma(e, s2, P.c[a][k]);
#pragma unroll
    for (int k = DO - 2; k >= 1; k -= 2) o = fma(o, s2, P.c[a][k]);
    w[a] = fma(s, o, e);
    w[W - 1 - a] = fma(-s, o, e);
  }
  if constexpr (W & 1) {
    double e = P.c[W / 2][DE];
#pragma unroll
    for (int k = DE - 2; k >= 0; k -= 2) e = fma(e, s2, P.c[W / 2][k]);
    w[W / 2] = e;
  }
}

template <int W>
__device__ __forceinline__ int es_weights(double t, const EsPoly &P, double (&w)[W]) {
  double s;
  const int i0 = es_reduce<W>(t, s);
  es_weights_s<W>(s, P, w);
  return i0;
}

// Signed mode index of FFT bin k in a length-n transform whose modes satisfy |j| <= jmax
// (jmax < n/2): returns true and j if bin k holds a mode.
__device__ __forceinline__ bool bin_to_mode(int64_t k, int64_t n, int64_t jmax, int64_t &j) {
  if (k <= jmax) { j = k; return true; }
  if (k >= n - jmax) { j = k - n; return true; }
  return false;
}

// Hermitian-half mode vectors and half-spectrum FFT boxes.
template <int D>
__device__ __forceinline__ void decode_half(int64_t loc, int K, int (&j)[D]) {
  j[D - 1] = (int)(loc % (K + 1));
  loc /= (K + 1);
#pragma unroll
  for (int k = D - 2; k >= 0; --k) {
    j[k] = (int)(loc % (2 * K + 1)) - K;
    loc /= (2 * K + 1);
  }
}

template <int D>
__device__ __forceinline__ int64_t encode_half(const int (&j)[D], int K) {
  int64_t idx = 0;
#pragma unroll
  for (int k = 0; k < D - 1; ++k) idx = idx * (2 * K + 1) + (j[k] + K);
  return idx * (K + 1) + j[D - 1];
}

// Box index of mode j in an n^(d-1) x (n/2+1) half-spectrum array.
template <int D>
__device__ __forceinline__ int64_t box_index(const int (&j)[D], int64_t n) {
  int64_t idx = 0;
#pragma unroll
  for (int k = 0; k < D - 1; ++k) idx = idx * n + (j[k] < 0 ? j[k] + n : j[k]);
  return idx * (n / 2 + 1) + j[D - 1];
}

// Inverse: which mode |j_i| <= K sits in box entry idx (false if none).
template <int D>
__device__ __forceinline__ bool box_to_mode(int64_t idx, int64_t n, int K, int (&j)[D]) {
  const int64_t nh = n / 2 + 1;
  const int64_t kd = idx % nh;
  idx /= nh;
  if (kd > K) return false;
  j[D - 1] = (int)kd;
#pragma unroll
  for (int k = D - 2; k >= 0; --k) {
    const int64_t kk = idx % n;
    idx /= n;
    int64_t jj;
    if (!bin_to_mode(kk, n, K, jj)) return false;
    j[k] = (int)jj;
  }
  return true;
}

// Programmatic dependent launch between the CG's own kernels (launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): a kernel lets its successor be scheduled at
// once (launch_dependents) and waits for its predecessor's completion and memory (wait) before
// touching any data, so consecutive launches overlap their latency instead of serialising it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), unsigned grid, unsigned block, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_smem(void (*k)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t s,
                                   Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

}  // namespace efgp
