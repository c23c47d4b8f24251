/*
 * efgp.h — C ABI of the B200 (sm_100a) EFGP hot path.
 *
 * Equispaced-Fourier GP regression (Greengard, Rachh, Barnett et al., arXiv 2210.10210), Algorithm
 * "a1": type-1 NUFFTs build the Toeplitz generating vector v (eq "88",
 * P:816-818) and the right-hand side Phi^* y = D F^* y (eq "rhs"); conjugate gradients
 * solve (D F^*F D + sigma^2 I) beta = Phi^* y (eqs "be"/"97") with the padded-FFT
 * Toeplitz product of Algorithm "a:FF"; a type-2 NUFFT evaluates the posterior mean
 * mu(x*) = sum_j D_j beta_j exp(2 pi i h j.x*) (eq "muws"; steps 5-6).
 *
 * Sign convention (reading G1): v_j = sum_n exp(-2 pi i h j.x_n),
 * (F^* y)_j = sum_n exp(-2 pi i h j.x_n) y_n, mu(x) = Re sum_j D_j beta_j exp(+2 pi i h j.x).
 *
 * Conventions for every entry point:
 *  - Points are (N, d) row-major fp64 (x_n in [0,1]^d), observations N fp64.
 *  - Pointers may be device memory (cudaMalloc / torch CUDA tensors) or host memory; the library
 *    detects which with cudaPointerGetAttributes.  Host inputs are streamed to the device in
 *    chunks inside the call (pinned memory gives overlapped copies).  The caller owns all of them;
 *    the library keeps no pointer after a call returns.
 *  - All device work is enqueued on options.stream (NULL = legacy default stream).  efgp_fit and
 *    efgp_predict return after their work is complete (they synchronise that stream).
 *  - The handle owns every internal buffer and the cuFFT plans.  A handle is not thread-safe.
 *  - Errors are reported by the status code; efgp_last_error() gives a message.  After an
 *    EFGP_ERR_CUDA the handle should be destroyed.
 *  - There is no CPU fallback: every step of the path runs in this library's sm_100a kernels and
 *    cuFFT; if no CUDA device is present, efgp_setup returns EFGP_ERR_CUDA.
 */
#ifndef EFGP_H
#define EFGP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EFGP_ABI_VERSION 6

typedef struct efgp_plan *efgp_handle;

typedef enum { EFGP_SE = 0, EFGP_MATERN = 1 } efgp_kernel;

typedef enum {
  EFGP_OK = 0,
  EFGP_ERR_NOCONVERGE = 1, /* CG hit max_iter; beta and the residual history stay readable */
  EFGP_ERR_INVALID = 2,    /* bad argument or input data                                 */
  EFGP_ERR_RESOURCE = 3,   /* a grid or buffer does not fit in device memory                       */
  EFGP_ERR_CUDA = 4,       /* CUDA runtime / cuFFT failure                                          */
  EFGP_ERR_NCCL = 5        /* NCCL missing or a collective failed (multi-GPU path)                  */
} efgp_status;

/* Matérn eps rescaling (§7.1; reading G3). */
typedef enum { EFGP_RESCALE_NONE = 0, EFGP_RESCALE_L2 = 1, EFGP_RESCALE_PRINTED = 2 } efgp_rescale;

/* Spreading strategy for the type-1 step. AUTO picks the fastest valid one. */
typedef enum {
  EFGP_SPREAD_AUTO = 0, EFGP_SPREAD_GLOBAL = 1, EFGP_SPREAD_SMEM = 2, EFGP_SPREAD_SORTED = 3,
  EFGP_SPREAD_CELLSORT = 4 /* counting sort by (super-)cell + warp-per-run accumulation (2D W >= 7, 3D) */
} efgp_spread_method;

/* Why the last fit's spreading did not run the planned method (efgp_info.spread_fallback).  The
 * fallback (GLOBAL: one fp64 RED per touch) gives the same grids to roundoff, ~10x slower.
 *   UNALIGNED       : SORTED bulk-copies x and y, which needs 16-byte aligned pointers.
 *   CORESIDENCY     : SORTED's cooperative launch could not place one CTA on every SM right now.
 *   TOO_MANY_POINTS : CELLSORT's 32-bit per-call point indices (N >= 2^32 in one call). */
typedef enum {
  EFGP_FALLBACK_NONE = 0, EFGP_FALLBACK_UNALIGNED = 1, EFGP_FALLBACK_CORESIDENCY = 2, EFGP_FALLBACK_TOO_MANY_POINTS = 3
} efgp_spread_fallback;

/* Arithmetic of the SORTED spreader (DESIGN.md §7 "K1 precision").  FFTs, CG, deconvolution, the
 * fine grids and all outputs are fp64 in every mode.
 *   FP64 : kernel weights and accumulation in fp64 (default).
 *   FP32 : kernel weights evaluated in fp32 from the fp64 reduced coordinate (relative error ~1e-7),
 *          fp64 accumulation.
 *   MIXED: fp32 weights; each start cell's window sums one shared-memory round (<= ~40 points) in
 *          fp32 (packed FFMA2) and adds it to its fp64 window.
 * FP32 and MIXED are refused (EFGP_ERR_INVALID) for nufft_tol < 1e-6. */
typedef enum { EFGP_WEIGHTS_FP64 = 0, EFGP_WEIGHTS_FP32 = 1, EFGP_WEIGHTS_MIXED = 2 } efgp_weights;

/* NEXT-4 (reading G12): CG preconditioner of efgp_fit / efgp_fit_solve.
 *   NONE: plain CG (Alg a1 step 4).
 *   KRON: PCG with M = A_1 (x) ... (x) A_d + sigma^2 I, A_i = diag(delta_i) T(v^(i)) diag(delta_i) /
 *         N^((d-1)/d) built from the axis lines of v and D (exact for tensor-product points with a
 *         separable kernel, and in d = 1), factored by a (2m+1)^2 Hermitian eigen-decomposition per
 *         axis (cuSOLVER) and applied by 2d small dense axis contractions per iteration.  Same answer
 *         and stopping rule.  Measured (profiles/r01_configs_v2.jsonl): SE (separable density) c3
 *         N = 1e7 2831 -> 152 iterations; Matérn (non-separable D, the product approximation of D
 *         is poor off the axes) needs MORE iterations (c5 52 -> 2542).  efgp_predict_var uses the same
 *         preconditioner (per target).
 *   JACOBI: PCG with M = diag(D_j^2 v_0 + sigma^2) (reading G12b), the diagonal of the system; for the
 *         Matérn configs 3-8x fewer iterations at the production tolerance (oracle: c5 22 -> 7,
 *         c2 199 -> 36), variance systems more (c5 718 -> 29).
 *   AUTO: KRON for EFGP_SE, JACOBI otherwise. */
typedef enum { EFGP_PRECOND_NONE = 0, EFGP_PRECOND_KRON = 1, EFGP_PRECOND_AUTO = 2, EFGP_PRECOND_JACOBI = 3 } efgp_precond;

/* NEXT-3 solver of efgp_fit_hetero (readings G11, G11b).
 *   TOEPLITZ: Phi^* S^-1 Phi = D T(v^w) D with v^w = eq "88" with strengths sigma_n^-2: one extra
 *             type-1 pass, then the FFT Toeplitz CG of efgp_fit with sigma^2 -> 1 (needs the SORTED or
 *             CELLSORT spreading, whose y grid is the v grid; otherwise NUFFT is used).
 *   NUFFT   : the BBMM-style CG the paper suggests: a type-2 + type-1 NUFFT pair over the
 *             N points per iteration (sorted fused pass for d <= 2).
 *   AUTO    : TOEPLITZ where available. */
typedef enum { EFGP_HETERO_AUTO = 0, EFGP_HETERO_TOEPLITZ = 1, EFGP_HETERO_NUFFT = 2 } efgp_hetero_method;

typedef struct {
  double h;            /* grid spacing override when m > 0                        */
  int64_t m;           /* modes per dimension override (2m+1 per dim), 0 = rule (Alg a1 step 1) */
  double cg_tol;       /* CG relative-residual stop, 0 = eps                      */
  int64_t max_iter;    /* CG cap, 0 = ceil(log(1/tol) sqrt(N)/(2 sigma))           */
  double nufft_tol;    /* NUFFT tolerance, 0 = eps/10                                   */
  int matern_rescale;  /* efgp_rescale, default EFGP_RESCALE_L2                                  */
  int spread_method;   /* efgp_spread_method                                                     */
  int graph_iters;     /* CG iterations per CUDA-graph launch, 0 = default                        */
  int spread_weights;  /* efgp_weights, default EFGP_WEIGHTS_FP64                                  */
  int precond;         /* efgp_precond, default EFGP_PRECOND_NONE (Alg a1's plain CG)             */
  int hetero_method;   /* efgp_hetero_method, default EFGP_HETERO_AUTO                            */
  void *stream;        /* cudaStream_t for all device work (NULL = default stream)               */
} efgp_options;

typedef struct {
  double h;             /* frequency grid spacing                                 */
  int64_t m, M, d;      /* half-width, number of modes (2m+1)^d, dimension          */
  int64_t N;            /* number of points of the last fit (sum over shards)      */
  int64_t iters;        /* CG iterations of the last fit                            */
  double rel_resid;     /* last recursive relative residual ||r||/||b||            */
  double cg_tol;        /* tolerance used                                           */
  int64_t max_iter;     /* cap used                                                 */
  int64_t nf1, nf2, L;  /* type-1 v-grid, rhs/type-2 grid and Toeplitz box sizes per dim */
  int64_t w;            /* ES kernel width (cells per dimension)                   */
  double beta_es;       /* ES kernel shape parameter                               */
  double nufft_tol;
  int spread_method;    /* method that actually spread the last fit's points      */
  double t_spread_ms, t_modes_ms, t_solve_ms, t_predict_ms; /* device time of the last calls */
  int64_t sorted_t1, sorted_t2, sorted_chunk, sorted_round;   /* SORTED geometry (0 unless SORTED ran) */
  int64_t spread_precision;                                   /* efgp_weights of the SORTED path */
  double t_var_ms;                                            /* device time of the last predict_var */
  int64_t var_iters_max, var_batch;                           /* its largest CG count, targets/batch */
  int64_t hetero_sorted; /* last efgp_fit_hetero: 0 unfused NUFFT pair, 1 sorted fused NUFFT pair,
                            2 weighted Toeplitz (G11b) */
  int64_t precond;       /* preconditioner the last fit used (NONE, KRON or JACOBI; AUTO resolved; NONE after a NUFFT-pair hetero fit) */
  int64_t comm_size;     /* ranks of the handle's NCCL communicator (0: none) */
  int64_t spread_fallback; /* efgp_spread_fallback of the last fit (NONE: the planned method ran) */
  int64_t cg_persist_split; /* direct 2D CG (c3, c5): k1 splits of the persistent one-kernel loop of the
                              last fit; 0 when the launched per-iteration kernels ran */
  int64_t cg_dft2;          /* one-launch CG kernels other than the direct 2D one: 1 when the last fit ran
                              the persistent DFT kernel (2D beyond the direct product, c2), 2 the one-CTA
                              1D kernel (c1), 0 otherwise */
} efgp_info;

/* Fill *opt with defaults (all zero / automatic). */
void efgp_default_options(efgp_options *opt);

/* Step 1 of Alg a1: choose (h, m) (Cor c:SEparams P:1113-1124 for SE; Remark r:heur eqs mheur/hheur
 * P:1305-1337 with the §7.1 rescaling for Matérn), tabulate D_j = sqrt(h^d k^(h|j|)) (eq 117,
 * P:783-794), size the NUFFT grids and the Toeplitz box, build the cuFFT plans and allocate device
 * buffers.  nu is used only for EFGP_MATERN (nu >= 1/2).  Returns EFGP_ERR_INVALID for sigma <= 0,
 * ell <= 0, eps outside [1e-14, 1e-1], d not in {1,2,3}, nu < 1/2; EFGP_ERR_RESOURCE if buffers do
 * not fit; EFGP_ERR_CUDA if there is no usable device.  opt may be NULL. */
efgp_status efgp_setup(efgp_handle *out, efgp_kernel kernel, double nu, double ell, double sigma,
                       double eps, int d, const efgp_options *opt);

/* Steps 2-4 of Alg a1 on one process: type-1 spreading of the N points, FFT + deconvolution to v
 * and F^*y, Toeplitz precompute, CG.  x: (N, d), y: (N).  Returns EFGP_ERR_INVALID if N < 1 or any
 * coordinate is outside [0,1] or non-finite, or any y is non-finite; EFGP_ERR_NOCONVERGE if CG hits
 * max_iter (beta is still usable). */
efgp_status efgp_fit(efgp_handle, const double *x, const double *y, int64_t N);

/* NEXT-3: fit with heteroskedastic noise (per-point sigma_n, readings G11,
 * G11b).  Solves (Phi^* S^-1 Phi + I) beta = Phi^* S^-1 y, S = diag(noise_sd^2), with the solver of
 * options.hetero_method (weighted-Toeplitz CG, or the NUFFT-pair CG); mu(x*) = phi(x*) beta as in
 * efgp_predict.  For noise_sd_n = sigma it gives efgp_fit's beta (the same system divided by sigma^2).
 * The sigma given at setup is not used; the CG cap default is P:1766 with sigma = min noise_sd.
 * options.precond applies to the TOEPLITZ solver.  x: (N, d), y: (N), noise_sd: (N); all device or
 * all host (host inputs are copied to the device for the whole solve: N (d + 2) doubles).  Returns
 * EFGP_ERR_INVALID for N < 1, a non-positive or non-finite noise_sd, points outside [0,1]^d,
 * non-finite y; EFGP_ERR_NOCONVERGE as efgp_fit.  After it, efgp_predict works, and
 * efgp_predict_var after a TOEPLITZ solve (sigma^2 -> 1 in eq "eta"; refused after NUFFT). */
efgp_status efgp_fit_hetero(efgp_handle, const double *x, const double *y, const double *noise_sd, int64_t N);

/* Multi-GPU with a library-owned NCCL communicator.
 * efgp_comm_unique_id writes NCCL_UNIQUE_ID_BYTES (128) bytes on one rank; the caller broadcasts
 * them; every rank then calls efgp_comm_init(handle, id, nranks, rank) on its own device.  From then
 * on efgp_fit(x, y, N) takes THIS rank's shard: it spreads it, sums the partial modes (and N) over
 * ranks with one ncclAllReduce on the library stream, and runs the CG replicated; efgp_fit_hetero
 * (TOEPLITZ solver) does the same with its weighted modes (and min sigma_n).  Every rank takes part
 * in the collectives even when its own spreading failed (e.g. an invalid coordinate): a failure
 * flag is reduced with the point counts, and then EVERY rank returns an error (the failing rank its
 * own status, the others EFGP_ERR_INVALID "failed on another rank"), so no rank waits forever.  NCCL
 * is loaded at run time (libnccl.so.2); EFGP_ERR_NCCL if it is missing or a call fails.  nranks = 1
 * is allowed. */
efgp_status efgp_comm_unique_id(void *id_out);
efgp_status efgp_comm_init(efgp_handle, const void *id, int nranks, int rank);

/* Multi-process split of efgp_fit.  efgp_fit_local spreads this rank's
 * shard and writes its partial modes (the Hermitian halves of v and F^*y, efgp_modes_count doubles)
 * to modes_out (device pointer).  The caller sums modes_out over ranks (one allreduce) and calls
 * efgp_fit_solve with the summed buffer and the global N.  Linearity of the type-1 sums in the
 * points (eqs 88, rhs) makes the sum of partial modes equal the modes of the union of shards. */
int64_t efgp_modes_count(efgp_handle);
efgp_status efgp_fit_local(efgp_handle, const double *x, const double *y, int64_t N, double *modes_out);
efgp_status efgp_fit_solve(efgp_handle, const double *modes, int64_t N_total);

/* Steps 5-6 of Alg a1: mu at q targets xt (q, d) written to mu_out (q).  EFGP_ERR_INVALID before a
 * successful fit/load or for targets outside [0,1]^d (their mu is set to NaN). q = 0 is a no-op. */
efgp_status efgp_predict(efgp_handle, const double *xt, int64_t q, double *mu_out);

/* NEXT-2: posterior variance s(x*) = sum_j eta_j phi_j(x*) (eq "sws"), one CG per target
 * on (Phi^*Phi + sigma^2 I) eta = sigma^2 conj(phi(x*)) (eq "eta"), batched
 * over targets with the Toeplitz operator of the last fit, each CG stopped at cg_tol (reading G6).
 * xt: (q, d) row-major; var_out: q doubles (host or device).  Needs a previous successful efgp_fit
 * or efgp_fit_solve (EFGP_ERR_INVALID otherwise); targets outside [0,1]^d give NaN and
 * EFGP_ERR_INVALID.  The CGs use the fit's preconditioner (efgp_info.precond: plain CG, KRON or
 * JACOBI) and its cap max_iter; if any target's CG reaches the cap before cg_tol the variances are
 * still written (the unconverged ones are CG iterates) and EFGP_ERR_NOCONVERGE is returned.
 * q = 0 is a no-op. */
efgp_status efgp_predict_var(efgp_handle, const double *xt, int64_t q, double *var_out);

/* Model state (SPEC S:369 serialisation).  beta is the Hermitian-half weight vector: for j in J_m
 * with j_d >= 0, row-major over (j_1+m, ..., j_{d-1}+m, j_d), interleaved (re, im) doubles;
 * efgp_weights_count() doubles.  Pointers may be host or device; the copies are ordered after the
 * work already enqueued on options.stream and complete before the call returns. */
int64_t efgp_weights_count(efgp_handle);
efgp_status efgp_get_weights(efgp_handle, double *beta_out);
efgp_status efgp_load_weights(efgp_handle, const double *beta_in);

/* Intermediate vectors of the last fit, Hermitian halves as interleaved complex doubles:
 * which = 0: v over J_{2m} (j_d in [0,2m]; (4m+1)^{d-1} (2m+1) complex);
 * which = 1: the right-hand side Phi^* y = D F^* y over J_m half (weights layout);
 * which = 2: beta (same as efgp_get_weights).  Returns the number of doubles written, or -1. */
int64_t efgp_copy_vector(efgp_handle, int which, double *out, int64_t cap_doubles);

efgp_status efgp_get_info(efgp_handle, efgp_info *out);

/* Recursive relative residuals ||r_k||/||b||, k = 0..iters of the last fit, into host_out (cap
 * entries); *n receives the number available. */
efgp_status efgp_get_residual_history(efgp_handle, double *host_out, int64_t cap, int64_t *n);

/* Diagnostics: with EFGP_SORTED_TRACE set at setup, the SORTED spreader records globaltimer stamps
 * [chunk][cta][4] = (binned, acc waits, acc starts, acc done) of the last fit; copies up to cap of
 * them to host_out and returns how many exist (0 if tracing is off). */
int64_t efgp_debug_trace(efgp_handle, unsigned long long *host_out, int64_t cap);

const char *efgp_last_error(efgp_handle);
void efgp_destroy(efgp_handle);
int efgp_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* EFGP_H */
