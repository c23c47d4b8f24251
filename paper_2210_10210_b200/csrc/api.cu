// C-ABI entry points (include/efgp.h): plan lifetime, host/device input handling, phase timing.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>

#include <cusolverDn.h>

#include "efgp_internal.cuh"

using namespace efgp;

namespace {

bool is_device_ptr(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

template <typename T>
efgp_status dalloc(efgp_plan *pl, T **p, size_t count) {
  EFGP_CUDA(cudaMalloc((void **)p, std::max<size_t>(count, 1) * sizeof(T)));
  return EFGP_OK;
}

efgp_status make_plan(efgp_plan *pl, cufftHandle *h, int d, int64_t n, cufftType t) {
  int dims[3] = {(int)n, (int)n, (int)n};
  EFGP_CUFFT(cufftPlanMany(h, d, dims, nullptr, 1, 0, nullptr, 1, 0, t, 1));
  return EFGP_OK;
}

efgp_status build(efgp_plan *pl) {
  if (pl->P.spread_method == EFGP_SPREAD_SORTED && !sorted_geometry(pl->P, pl->num_sms)) {
    pl->P.sorted_disabled = true;  // e.g. too many tiles for shared memory: SMEM or GLOBAL instead
    pl->P.spread_method = pl->P.spread_method_requested;
    resolve_spread_method(pl->P);
  }
  const Params &P = pl->P;
  const int d = P.d;
  // D_j = sqrt(h^d k^(h|j|)) on the J_m half (eq 117)
  std::vector<double> Dh(P.Mh);
  for (int64_t q = 0; q < P.Mh; ++q) {
    int64_t rem = q;
    double r2 = 0;
    const int64_t jd = rem % (P.m + 1);
    rem /= (P.m + 1);
    r2 += (double)jd * jd;
    for (int k = 0; k < d - 1; ++k) {
      const int64_t j = rem % (2 * P.m + 1) - P.m;
      rem /= (2 * P.m + 1);
      r2 += (double)j * j;
    }
    Dh[q] = std::sqrt(std::pow(P.h, d) * khat_host(P, P.h * std::sqrt(r2)));
  }
  // deconvolution tables of the piecewise-polynomial kernel the kernels actually use
  const std::vector<double> psi1 = es_fourier_table_poly(P.poly, P.w, P.n1, 2 * P.m);
  const std::vector<double> psi2 = es_fourier_table_poly(P.poly, P.w, P.n2, P.m);
  EFGP_TRY(dalloc(pl, &pl->poly_dev, 1));
  EFGP_CUDA(cudaMemcpy(pl->poly_dev, &P.poly, sizeof(EsPoly), cudaMemcpyHostToDevice));
  EFGP_TRY(dalloc(pl, &pl->D_half, P.Mh));
  EFGP_TRY(dalloc(pl, &pl->psi1, psi1.size()));
  EFGP_TRY(dalloc(pl, &pl->psi2, psi2.size()));
  EFGP_CUDA(cudaMemcpy(pl->D_half, Dh.data(), sizeof(double) * P.Mh, cudaMemcpyHostToDevice));
  EFGP_CUDA(cudaMemcpy(pl->psi1, psi1.data(), sizeof(double) * psi1.size(), cudaMemcpyHostToDevice));
  EFGP_CUDA(cudaMemcpy(pl->psi2, psi2.data(), sizeof(double) * psi2.size(), cudaMemcpyHostToDevice));

  const int64_t g1 = ipow(P.n1, d), g2 = ipow(P.n2, d), gr = ipow(P.n_rhs, d);
  const int64_t G1h = ipow(P.n1, d - 1) * (P.n1 / 2 + 1), G2h = ipow(P.n2, d - 1) * (P.n2 / 2 + 1);
  const int64_t Grh = ipow(P.n_rhs, d - 1) * (P.n_rhs / 2 + 1);
  const int64_t Ld = ipow(P.L, d), box = ipow(P.L, d - 1) * (P.L / 2 + 1);
  EFGP_TRY(dalloc(pl, &pl->g1, g1));
  EFGP_TRY(dalloc(pl, &pl->g2, gr));
  EFGP_TRY(dalloc(pl, &pl->G1h, G1h));
  EFGP_TRY(dalloc(pl, &pl->G2h, Grh));
  EFGP_TRY(dalloc(pl, &pl->modes, 2 * (P.Kvh + P.Mh)));
  EFGP_TRY(dalloc(pl, &pl->modes_sum, 2 * (P.Kvh + P.Mh)));
  EFGP_TRY(dalloc(pl, &pl->Xbox, box));
  EFGP_TRY(dalloc(pl, &pl->Zbox, box));
  EFGP_TRY(dalloc(pl, &pl->Yr, Ld));
  EFGP_TRY(dalloc(pl, &pl->vhat, Ld));
  for (double2 **v : {&pl->b, &pl->x, &pl->r, &pl->p, &pl->Ap, &pl->p2}) {
    EFGP_TRY(dalloc(pl, v, P.Mh));
    EFGP_CUDA(cudaMemset(*v, 0, sizeof(double2) * P.Mh));
  }
  pl->cg_blocks = pl->num_sms * 4;
  EFGP_TRY(dalloc(pl, &pl->partials, 3 * pl->cg_blocks));  // (p,Ap) | (r,r) | PCG (r,z)
  EFGP_TRY(dalloc(pl, &pl->scal, 32));
  EFGP_TRY(dalloc(pl, &pl->dflags, 4));
  EFGP_CUDA(cudaMallocHost((void **)&pl->h_pinned, 256));
  EFGP_TRY(dalloc(pl, &pl->T2box, G2h));
  EFGP_TRY(dalloc(pl, &pl->t2grid, g2));
  EFGP_TRY(make_plan(pl, &pl->plan_g1, d, P.n1, CUFFT_D2Z));
  EFGP_TRY(make_plan(pl, &pl->plan_g2, d, P.n_rhs, CUFFT_D2Z));
  EFGP_TRY(make_plan(pl, &pl->plan_c2r_L, d, P.L, CUFFT_Z2D));
  EFGP_TRY(make_plan(pl, &pl->plan_r2c_L, d, P.L, CUFFT_D2Z));
  EFGP_TRY(make_plan(pl, &pl->plan_t2, d, P.n2, CUFFT_Z2D));
  for (auto &e : pl->ev) EFGP_CUDA(cudaEventCreate(&e));
  EFGP_CUDA(cudaStreamCreateWithFlags(&pl->copy_stream, cudaStreamNonBlocking));
  pl->spread_used = P.spread_method;  // until a fit spreads: the planned method (and its geometry)
  return EFGP_OK;
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
    cudaGetLastError();
    return 0.f;
  }
  return ms;
}

// Stream host-resident points through two device staging buffers: copies on copy_stream overlap
// spreading on the main stream.
efgp_status spread_host(efgp_plan *pl, const double *x, const double *y, int64_t N) {
  const int d = pl->P.d;
  const int64_t chunk = std::min<int64_t>(N, 1ll << 25);
  if (pl->stage_pts < chunk) {
    for (auto &s : pl->stage) {
      if (s) cudaFree(s);
      s = nullptr;
    }
    pl->stage_pts = 0;
    for (auto &s : pl->stage) EFGP_TRY(dalloc(pl, &s, chunk * (d + 1)));
    pl->stage_pts = chunk;
  }
  cudaEvent_t copied[2], freed[2];
  for (int i = 0; i < 2; ++i) {
    EFGP_CUDA(cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming));
    EFGP_CUDA(cudaEventCreateWithFlags(&freed[i], cudaEventDisableTiming));
    EFGP_CUDA(cudaEventRecord(freed[i], pl->stream));
  }
  efgp_status st = EFGP_OK;
  int c = 0;
  for (int64_t s0 = 0; s0 < N && st == EFGP_OK; s0 += chunk, ++c) {
    const int64_t n = std::min(chunk, N - s0);
    const int b = c & 1;
    double *xs = pl->stage[b], *ys = pl->stage[b] + chunk * d;
    cudaStreamWaitEvent(pl->copy_stream, freed[b], 0);
    cudaMemcpyAsync(xs, x + s0 * d, sizeof(double) * n * d, cudaMemcpyHostToDevice, pl->copy_stream);
    cudaMemcpyAsync(ys, y + s0, sizeof(double) * n, cudaMemcpyHostToDevice, pl->copy_stream);
    cudaEventRecord(copied[b], pl->copy_stream);
    cudaStreamWaitEvent(pl->stream, copied[b], 0);
    st = spread_points(pl, xs, ys, n, pl->stream);
    cudaEventRecord(freed[b], pl->stream);
  }
  cudaError_t e = cudaGetLastError();
  for (int i = 0; i < 2; ++i) {
    cudaEventDestroy(copied[i]);
    cudaEventDestroy(freed[i]);
  }
  if (st == EFGP_OK && e != cudaSuccess) {
    pl->err = std::string("CUDA error: ") + cudaGetErrorString(e);
    return EFGP_ERR_CUDA;
  }
  return st;
}

// Order library work after everything the caller enqueued on its stream, and vice versa.
efgp_status enter(efgp_plan *pl) {
  EFGP_CUDA(cudaEventRecord(pl->ev_in, pl->ustream));
  EFGP_CUDA(cudaStreamWaitEvent(pl->stream, pl->ev_in, 0));
  return EFGP_OK;
}
efgp_status leave(efgp_plan *pl) {
  EFGP_CUDA(cudaEventRecord(pl->ev_out, pl->stream));
  EFGP_CUDA(cudaStreamWaitEvent(pl->ustream, pl->ev_out, 0));
  return EFGP_OK;
}

efgp_status fit_local_impl(efgp_plan *pl, const double *x, const double *y, int64_t N, double *modes_out) {
  if (N < 1 || !x || !y || !modes_out) {
    pl->err = "fit: N must be >= 1 and pointers non-null";
    return EFGP_ERR_INVALID;
  }
  cudaStream_t s = pl->stream;
  NvtxRange nv("efgp: type-1 (spread + modes)");
  EFGP_TRY(enter(pl));
  EFGP_CUDA(cudaEventRecord(pl->ev[0], s));
  EFGP_TRY(spread_begin(pl, s));
  const bool dx = is_device_ptr(x), dy = is_device_ptr(y);
  if (dx && dy) {
    EFGP_TRY(spread_points(pl, x, y, N, s));
  } else if (!dx && !dy) {
    EFGP_TRY(spread_host(pl, x, y, N));
  } else {
    pl->err = "fit: x and y must both be device or both be host memory";
    return EFGP_ERR_INVALID;
  }
  EFGP_CUDA(cudaEventRecord(pl->ev[1], s));
  EFGP_TRY(type1_modes(pl, modes_out, s));
  EFGP_CUDA(cudaEventRecord(pl->ev[2], s));
  EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned, pl->dflags, sizeof(int) * 4, cudaMemcpyDeviceToHost, s));
  EFGP_CUDA(cudaStreamSynchronize(s));
  int flags[4];
  std::memcpy(flags, pl->h_pinned, sizeof(flags));
  pl->t_spread = elapsed(pl->ev[0], pl->ev[1]);
  pl->t_modes = elapsed(pl->ev[1], pl->ev[2]);
  EFGP_TRY(leave(pl));
  if (flags[0]) {
    pl->err = "fit: a coordinate is outside [0,1] or non-finite, or an observation is non-finite";
    return EFGP_ERR_INVALID;
  }
  return EFGP_OK;
}

efgp_status fit_solve_impl(efgp_plan *pl, const double *modes, int64_t N_total) {
  if (!modes || N_total < 1) {
    pl->err = "fit_solve: modes must be non-null and N_total >= 1";
    return EFGP_ERR_INVALID;
  }
  const Params &P = pl->P;
  cudaStream_t s = pl->stream;
  pl->fitted = false;
  pl->t2_valid = false;
  NvtxRange nv("efgp: Toeplitz setup + CG");
  EFGP_TRY(enter(pl));
  EFGP_CUDA(cudaEventRecord(pl->ev[3], s));
  EFGP_CUDA(cudaMemcpyAsync(pl->modes_sum, modes, sizeof(double) * 2 * (P.Kvh + P.Mh), cudaMemcpyDefault, s));
  EFGP_TRY(toeplitz_setup(pl, pl->modes_sum, s));
  pl->op_valid = true;
  pl->sigma2_sys = P.sigma * P.sigma;  // (Phi^*Phi + sigma^2 I)
  pl->cap_sigma = P.sigma;
  efgp_status st;
  pl->pc_used = P.precond;
  if (P.precond) {  // NEXT-4: Kronecker (G12) or Jacobi (G12b) preconditioned CG
    EFGP_TRY(precond_setup(pl, pl->modes_sum));
    st = pcg_solve(pl, N_total);
  } else {
    st = cg_solve(pl, N_total);
  }
  EFGP_CUDA(cudaEventRecord(pl->ev[4], s));
  EFGP_CUDA(cudaEventSynchronize(pl->ev[4]));
  pl->t_solve = elapsed(pl->ev[3], pl->ev[4]);
  EFGP_TRY(leave(pl));
  pl->N_last = N_total;
  if (st == EFGP_OK || st == EFGP_ERR_NOCONVERGE) pl->fitted = true;
  if (st == EFGP_ERR_NOCONVERGE) pl->err = "CG reached max_iter before the relative residual reached cg_tol";
  return st;
}

}  // namespace

extern "C" {

int efgp_abi_version(void) { return EFGP_ABI_VERSION; }

void efgp_default_options(efgp_options *opt) {
  if (!opt) return;
  std::memset(opt, 0, sizeof(*opt));
  opt->matern_rescale = EFGP_RESCALE_L2;
  opt->spread_method = EFGP_SPREAD_AUTO;
}

efgp_status efgp_setup(efgp_handle *out, efgp_kernel kernel, double nu, double ell, double sigma, double eps, int d,
                       const efgp_options *opt) {
  if (!out) return EFGP_ERR_INVALID;
  *out = nullptr;
  efgp_options o;
  efgp_default_options(&o);
  if (opt) o = *opt;
  efgp_plan *pl = new (std::nothrow) efgp_plan();
  if (!pl) return EFGP_ERR_RESOURCE;
  *out = pl;  // returned even on failure so efgp_last_error works; caller must efgp_destroy
  pl->P.kernel = kernel;
  pl->P.nu = nu;
  pl->P.ell = ell;
  pl->P.sigma = sigma;
  pl->P.eps = eps;
  pl->P.d = d;
  const std::string msg = validate_and_choose(pl->P, o);
  if (!msg.empty()) {
    pl->err = msg;
    return EFGP_ERR_INVALID;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
    cudaGetLastError();
    pl->err = "no CUDA device: the EFGP library has no CPU fallback";
    return EFGP_ERR_CUDA;
  }
  EFGP_CUDA(cudaGetDevice(&pl->device));
  EFGP_CUDA(cudaDeviceGetAttribute(&pl->num_sms, cudaDevAttrMultiProcessorCount, pl->device));
  pl->ustream = (cudaStream_t)o.stream;
  EFGP_CUDA(cudaStreamCreateWithFlags(&pl->stream, cudaStreamNonBlocking));
  EFGP_CUDA(cudaEventCreateWithFlags(&pl->ev_in, cudaEventDisableTiming));
  EFGP_CUDA(cudaEventCreateWithFlags(&pl->ev_out, cudaEventDisableTiming));
  {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = pl->device;
    EFGP_CUDA(cudaMemPoolCreate(&pl->pool, &props));
    uint64_t keep = UINT64_MAX;
    EFGP_CUDA(cudaMemPoolSetAttribute(pl->pool, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  return build(pl);
}

efgp_status efgp_fit(efgp_handle pl, const double *x, const double *y, int64_t N) {
  efgp::NvtxRange nv_call("efgp_fit");
  if (!pl) return EFGP_ERR_INVALID;
  const efgp_status st = fit_local_impl(pl, x, y, N, pl->modes);
  if (pl->comm) {
    // the one collective of a multi-GPU fit: partial modes and counts summed over ranks.  Every rank
    // takes part even when its own spreading failed (its modes are then meaningless, and so is the
    // sum): the failure flag travels with the counts and all ranks return an error together.
    const std::string local_err = pl->err;
    int fail = st != EFGP_OK;
    int64_t n = st == EFGP_OK ? N : 0;
    EFGP_TRY(comm_sum(pl, pl->modes, (size_t)2 * (pl->P.Kvh + pl->P.Mh)));
    EFGP_TRY(comm_count_min(pl, &n, nullptr, &fail));
    if (st != EFGP_OK) {
      pl->err = local_err;
      return st;
    }
    if (fail) {
      pl->err = "fit: the spreading failed on another rank (invalid input there); no rank solved";
      return EFGP_ERR_INVALID;
    }
    N = n;
  } else if (st != EFGP_OK) {
    return st;
  }
  return fit_solve_impl(pl, pl->modes, N);
}

efgp_status efgp_comm_unique_id(void *id_out) {
  if (!id_out) return EFGP_ERR_INVALID;
  return comm_unique_id(id_out);
}

efgp_status efgp_comm_init(efgp_handle pl, const void *id, int nranks, int rank) {
  if (!pl || !id) return EFGP_ERR_INVALID;
  return comm_init(pl, id, nranks, rank);
}

efgp_status efgp_fit_hetero(efgp_handle pl, const double *x, const double *y, const double *noise_sd, int64_t N) {
  efgp::NvtxRange nv_call("efgp_fit_hetero");
  if (!pl) return EFGP_ERR_INVALID;
  if (N < 1 || !x || !y || !noise_sd) {
    pl->err = "fit_hetero: N must be >= 1 and pointers non-null";
    return EFGP_ERR_INVALID;
  }
  const int d = pl->P.d;
  cudaStream_t s = pl->stream;
  const bool dx = is_device_ptr(x), dy = is_device_ptr(y), ds = is_device_ptr(noise_sd);
  if (!(dx == dy && dy == ds)) {
    pl->err = "fit_hetero: x, y and noise_sd must all be device or all be host memory";
    return EFGP_ERR_INVALID;
  }
  EFGP_TRY(enter(pl));
  if (dx) {
    EFGP_TRY(fit_hetero_device(pl, x, y, noise_sd, N));
  } else {
    // every CG iteration reads the points again: stage them on the device for the whole solve
    double *buf = nullptr;
    EFGP_PALLOC(&buf, sizeof(double) * N * (d + 2), s);
    EFGP_CUDA(cudaMemcpyAsync(buf, x, sizeof(double) * N * d, cudaMemcpyHostToDevice, s));
    EFGP_CUDA(cudaMemcpyAsync(buf + N * d, y, sizeof(double) * N, cudaMemcpyHostToDevice, s));
    EFGP_CUDA(cudaMemcpyAsync(buf + N * (d + 1), noise_sd, sizeof(double) * N, cudaMemcpyHostToDevice, s));
    const efgp_status st = fit_hetero_device(pl, buf, buf + N * d, buf + N * (d + 1), N);
    cudaFreeAsync(buf, s);
    EFGP_CUDA(cudaStreamSynchronize(s));
    if (st != EFGP_OK) return st;
  }
  return leave(pl);
}

int64_t efgp_modes_count(efgp_handle pl) { return pl ? 2 * (pl->P.Kvh + pl->P.Mh) : -1; }

efgp_status efgp_fit_local(efgp_handle pl, const double *x, const double *y, int64_t N, double *modes_out) {
  if (!pl) return EFGP_ERR_INVALID;
  if (modes_out && !is_device_ptr(modes_out)) {
    pl->err = "fit_local: modes_out must be device memory";
    return EFGP_ERR_INVALID;
  }
  return fit_local_impl(pl, x, y, N, modes_out);
}

efgp_status efgp_fit_solve(efgp_handle pl, const double *modes, int64_t N_total) {
  if (!pl) return EFGP_ERR_INVALID;
  return fit_solve_impl(pl, modes, N_total);
}

efgp_status efgp_predict(efgp_handle pl, const double *xt, int64_t q, double *mu_out) {
  efgp::NvtxRange nv_call("efgp_predict");
  if (!pl) return EFGP_ERR_INVALID;
  if (!pl->fitted) {
    pl->err = "predict before a successful fit or load_weights";
    return EFGP_ERR_INVALID;
  }
  if (q < 0 || (q > 0 && (!xt || !mu_out))) {
    pl->err = "predict: bad arguments";
    return EFGP_ERR_INVALID;
  }
  if (q == 0) return EFGP_OK;
  const int d = pl->P.d;
  cudaStream_t s = pl->stream;
  EFGP_TRY(enter(pl));
  EFGP_CUDA(cudaEventRecord(pl->ev[5], s));
  EFGP_CUDA(cudaMemsetAsync(pl->dflags + 1, 0, sizeof(int), s));
  if (!pl->t2_valid) EFGP_TRY(type2_grid(pl, s));
  const bool dx = is_device_ptr(xt), dm = is_device_ptr(mu_out);
  if (dx && dm) {
    EFGP_TRY(interp_targets(pl, xt, q, mu_out, s));
  } else {
    const int64_t chunk = std::min<int64_t>(q, 1ll << 24);
    double *dxt = nullptr, *dmu = nullptr;
    EFGP_PALLOC(&dxt, sizeof(double) * chunk * d, s);
    EFGP_PALLOC(&dmu, sizeof(double) * chunk, s);
    for (int64_t s0 = 0; s0 < q; s0 += chunk) {
      const int64_t n = std::min(chunk, q - s0);
      EFGP_CUDA(cudaMemcpyAsync(dxt, xt + s0 * d, sizeof(double) * n * d, cudaMemcpyDefault, s));
      EFGP_TRY(interp_targets(pl, dxt, n, dmu, s));
      EFGP_CUDA(cudaMemcpyAsync(mu_out + s0, dmu, sizeof(double) * n, cudaMemcpyDefault, s));
    }
    EFGP_CUDA(cudaFreeAsync(dxt, s));
    EFGP_CUDA(cudaFreeAsync(dmu, s));
  }
  EFGP_CUDA(cudaEventRecord(pl->ev[6], s));
  EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned, pl->dflags, sizeof(int) * 4, cudaMemcpyDeviceToHost, s));
  EFGP_CUDA(cudaStreamSynchronize(s));
  pl->t_predict = elapsed(pl->ev[5], pl->ev[6]);
  EFGP_TRY(leave(pl));
  int flags[4];
  std::memcpy(flags, pl->h_pinned, sizeof(flags));
  if (flags[1]) {
    pl->err = "predict: a target is outside [0,1]^d or non-finite (its mu is NaN)";
    return EFGP_ERR_INVALID;
  }
  return EFGP_OK;
}

efgp_status efgp_predict_var(efgp_handle pl, const double *xt, int64_t q, double *var_out) {
  efgp::NvtxRange nv_call("efgp_predict_var");
  if (!pl) return EFGP_ERR_INVALID;
  if (!pl->fitted || !pl->op_valid) {
    pl->err = "predict_var before a successful fit (the variance needs the fit's Toeplitz operator)";
    return EFGP_ERR_INVALID;
  }
  if (q < 0 || (q > 0 && (!xt || !var_out))) {
    pl->err = "predict_var: bad arguments";
    return EFGP_ERR_INVALID;
  }
  if (q == 0) return EFGP_OK;
  const int d = pl->P.d;
  cudaStream_t s = pl->stream;
  EFGP_TRY(enter(pl));
  EFGP_CUDA(cudaEventRecord(pl->ev[5], s));
  EFGP_CUDA(cudaMemsetAsync(pl->dflags + 1, 0, sizeof(int), s));
  const bool dx = is_device_ptr(xt), dm = is_device_ptr(var_out);
  efgp_status vst = EFGP_OK;  // NOCONVERGE (a target CG hit the cap) is reported after the outputs
  auto var_call = [&](const double *a, int64_t n, double *o) -> efgp_status {
    const efgp_status r = variance_targets(pl, a, n, o, s);
    if (r == EFGP_ERR_NOCONVERGE) {
      vst = r;
      return EFGP_OK;
    }
    return r;
  };
  if (dx && dm) {
    EFGP_TRY(var_call(xt, q, var_out));
  } else {
    const int64_t chunk = std::min<int64_t>(q, 1ll << 20);
    double *dxt = nullptr, *dv = nullptr;
    EFGP_PALLOC(&dxt, sizeof(double) * chunk * d, s);
    EFGP_PALLOC(&dv, sizeof(double) * chunk, s);
    for (int64_t s0 = 0; s0 < q; s0 += chunk) {
      const int64_t n = std::min(chunk, q - s0);
      EFGP_CUDA(cudaMemcpyAsync(dxt, xt + s0 * d, sizeof(double) * n * d, cudaMemcpyDefault, s));
      EFGP_TRY(var_call(dxt, n, dv));
      EFGP_CUDA(cudaMemcpyAsync(var_out + s0, dv, sizeof(double) * n, cudaMemcpyDefault, s));
    }
    EFGP_CUDA(cudaFreeAsync(dxt, s));
    EFGP_CUDA(cudaFreeAsync(dv, s));
  }
  EFGP_CUDA(cudaEventRecord(pl->ev[6], s));
  EFGP_CUDA(cudaMemcpyAsync(pl->h_pinned, pl->dflags, sizeof(int) * 4, cudaMemcpyDeviceToHost, s));
  EFGP_CUDA(cudaStreamSynchronize(s));
  pl->t_var = elapsed(pl->ev[5], pl->ev[6]);
  EFGP_TRY(leave(pl));
  int flags[4];
  std::memcpy(flags, pl->h_pinned, sizeof(flags));
  if (flags[1]) {
    pl->err = "predict_var: a target is outside [0,1]^d or non-finite (its variance is NaN)";
    return EFGP_ERR_INVALID;
  }
  return vst;
}

int64_t efgp_weights_count(efgp_handle pl) { return pl ? 2 * pl->P.Mh : -1; }

efgp_status efgp_get_weights(efgp_handle pl, double *beta_out) {
  if (!pl || !beta_out) return EFGP_ERR_INVALID;
  EFGP_TRY(enter(pl));  // after the caller's pending work (a device beta_out may still be in use)
  EFGP_CUDA(cudaMemcpyAsync(beta_out, pl->x, sizeof(double2) * pl->P.Mh, cudaMemcpyDefault, pl->stream));
  EFGP_CUDA(cudaStreamSynchronize(pl->stream));
  return leave(pl);
}

efgp_status efgp_load_weights(efgp_handle pl, const double *beta_in) {
  if (!pl || !beta_in) return EFGP_ERR_INVALID;
  EFGP_TRY(enter(pl));  // a device beta_in just written on the caller's stream is complete first
  EFGP_CUDA(cudaMemcpyAsync(pl->x, beta_in, sizeof(double2) * pl->P.Mh, cudaMemcpyDefault, pl->stream));
  EFGP_CUDA(cudaStreamSynchronize(pl->stream));
  pl->fitted = true;
  pl->t2_valid = false;
  return leave(pl);
}

int64_t efgp_copy_vector(efgp_handle pl, int which, double *out, int64_t cap) {
  if (!pl || !out) return -1;
  const Params &P = pl->P;
  const void *src = nullptr;
  int64_t n = 0;
  if (which == 0) {
    src = pl->modes_sum;
    n = 2 * P.Kvh;
  } else if (which == 1) {
    src = pl->b;
    n = 2 * P.Mh;
  } else if (which == 2) {
    src = pl->x;
    n = 2 * P.Mh;
  } else {
    return -1;
  }
  if (cap < n) return -1;
  if (enter(pl) != EFGP_OK || cudaMemcpyAsync(out, src, sizeof(double) * n, cudaMemcpyDefault, pl->stream) != cudaSuccess ||
      cudaStreamSynchronize(pl->stream) != cudaSuccess || leave(pl) != EFGP_OK) {
    cudaGetLastError();
    return -1;
  }
  return n;
}

efgp_status efgp_get_info(efgp_handle pl, efgp_info *o) {
  if (!pl || !o) return EFGP_ERR_INVALID;
  const Params &P = pl->P;
  std::memset(o, 0, sizeof(*o));
  o->h = P.h;
  o->m = P.m;
  o->M = P.M;
  o->d = P.d;
  o->N = pl->N_last;
  o->iters = pl->iters;
  o->rel_resid = pl->rel_resid;
  o->cg_tol = P.cg_tol;
  o->max_iter = pl->max_iter_used;
  o->nf1 = P.n1;
  o->nf2 = P.n2;
  o->L = P.L;
  o->w = P.w;
  o->beta_es = P.beta_es;
  o->nufft_tol = P.nufft_tol;
  o->spread_method = pl->spread_used;
  o->t_spread_ms = pl->t_spread;
  o->t_modes_ms = pl->t_modes;
  o->t_solve_ms = pl->t_solve;
  o->t_predict_ms = pl->t_predict;
  o->spread_fallback = pl->spread_fallback;
  o->cg_persist_split = pl->cg_persist_split;
  o->cg_dft2 = pl->cg_dft2;
  if (pl->spread_used == EFGP_SPREAD_SORTED) {
    o->sorted_t1 = P.T1;  // (the SORTED kernel is one cooperative launch per fit)
    o->sorted_t2 = P.T2;
    o->sorted_chunk = P.chunk;
    o->sorted_round = P.round;
    o->spread_precision = P.spread_mode;
  }
  {
    o->t_var_ms = pl->t_var;
    o->var_iters_max = pl->var_iters_max;
    o->var_batch = pl->var_B;
  }
  o->hetero_sorted = pl->het_path;
  o->precond = pl->pc_used;
  o->comm_size = pl->comm_size;
  return EFGP_OK;
}

efgp_status efgp_get_residual_history(efgp_handle pl, double *host_out, int64_t cap, int64_t *n) {
  if (!pl || !n) return EFGP_ERR_INVALID;
  *n = pl->hist ? pl->iters + 1 : 0;
  if (host_out && pl->hist) {
    const int64_t k = std::min<int64_t>(cap, *n);
    EFGP_CUDA(cudaMemcpy(host_out, pl->hist, sizeof(double) * k, cudaMemcpyDeviceToHost));
  }
  return EFGP_OK;
}

int64_t efgp_debug_trace(efgp_handle pl, unsigned long long *host_out, int64_t cap) {
  if (!pl || !pl->trace) return 0;
  const int64_t n = std::min<int64_t>(cap, (int64_t)pl->trace_n);
  if (host_out && n > 0 && cudaMemcpy(host_out, pl->trace, n * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  return (int64_t)pl->trace_n;
}

const char *efgp_last_error(efgp_handle pl) { return pl ? pl->err.c_str() : "null handle"; }

void efgp_destroy(efgp_handle pl) {
  if (!pl) return;
  if (pl->stream) cudaStreamSynchronize(pl->stream);
  comm_destroy(pl);
  if (pl->cg_exec) cudaGraphExecDestroy(pl->cg_exec);
  if (pl->var_exec) cudaGraphExecDestroy(pl->var_exec);
  if (pl->pcg_exec) cudaGraphExecDestroy(pl->pcg_exec);
  if (pl->pc_solver) cusolverDnDestroy(static_cast<cusolverDnHandle_t>(pl->pc_solver));
  for (cufftHandle h : {pl->plan_var_c2r, pl->plan_var_r2c, pl->plan_het, pl->plan_het_r2c})
    if (h) cufftDestroy(h);
  for (void *b : {(void *)pl->var_x, (void *)pl->var_r, (void *)pl->var_p, (void *)pl->var_Ap, (void *)pl->var_X,
                  (void *)pl->var_Z, (void *)pl->var_Y, pl->var_st})
    if (b) cudaFree(b);
  for (cufftHandle h : {pl->plan_g1, pl->plan_g2, pl->plan_c2r_L, pl->plan_r2c_L, pl->plan_t2, pl->plan_pt, pl->plan_ptv})
    if (h) cufftDestroy(h);
  for (void *b : {(void *)pl->pt_P, (void *)pl->pt_T, (void *)pl->pt_W, (void *)pl->pt_V})
    if (b) cudaFree(b);
  void *bufs[] = {pl->poly_dev, pl->D_half, pl->psi1, pl->psi2, pl->g1, pl->g2, pl->G1h, pl->G2h, pl->modes, pl->modes_sum,
                  pl->Xbox, pl->Yr, pl->vhat, pl->Zbox, pl->b, pl->x, pl->r, pl->p, pl->Ap, pl->partials,
                  pl->scal, pl->hist, pl->dflags, pl->T2box, pl->t2grid, pl->stage[0], pl->stage[1],
                  pl->trace,
                  pl->sync_buf, pl->het_box, pl->het_grid, pl->pc_Q, pl->pc_F0, pl->pc_F1, pl->pc_work, pl->z,
                  pl->pc_lam, pl->pc_info, pl->comm_buf, pl->vfull, pl->pc_diag, pl->toep_part, pl->toep_cnt, pl->p2, pl->cg_gbar,
                  pl->dft_V, pl->dft_roots, pl->dft_W};
  for (void *b : bufs)
    if (b) cudaFree(b);
  for (void *b : pl->rec)
    if (b) cudaFree(b);
  if (pl->h_pinned) cudaFreeHost(pl->h_pinned);
  for (auto &e : pl->ev)
    if (e) cudaEventDestroy(e);
  if (pl->copy_stream) cudaStreamDestroy(pl->copy_stream);
  if (pl->ev_in) cudaEventDestroy(pl->ev_in);
  if (pl->ev_out) cudaEventDestroy(pl->ev_out);
  if (pl->stream) cudaStreamDestroy(pl->stream);
  if (pl->pool) cudaMemPoolDestroy(pl->pool);
  delete pl;
}

}  // extern "C"
