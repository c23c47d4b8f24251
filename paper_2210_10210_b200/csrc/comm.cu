// Multi-GPU plumbing inside the library ("each rank calls setup/fit/predict with
// its own shard and the shared communicator"): an NCCL communicator owned by the handle, and the ONE
// collective of a fit — the sum over ranks of the partial Hermitian-half modes (v, F^*y: linearity of
// the type-1 sums in the points, eqs "88" / "rhs") and of the point counts — enqueued on the
// library stream between the local spreading and the replicated Toeplitz CG.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, which returns the copy PyTorch already
// loaded), so the library has no link-time NCCL dependency and never brings a second NCCL into a
// process.  Types come from the system nccl.h.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "efgp_internal.cuh"

namespace efgp {

namespace {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char *(*getErrorString)(ncclResult_t) = nullptr;
};

const NcclApi &nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(h, "ncclAllReduce"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.getErrorString = reinterpret_cast<decltype(api.getErrorString)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.getUniqueId && api.commInitRank && api.allReduce && api.commDestroy && api.getErrorString;
  });
  return api;
}

efgp_status nccl_check(efgp_plan *pl, ncclResult_t r, const char *what) {
  if (r == ncclSuccess) return EFGP_OK;
  if (pl) pl->err = std::string("NCCL ") + what + ": " + nccl().getErrorString(r);
  return EFGP_ERR_NCCL;
}

}  // namespace

efgp_status comm_unique_id(void *id_out) {
  const NcclApi &a = nccl();
  if (!a.ok) return EFGP_ERR_NCCL;
  ncclUniqueId id;
  if (a.getUniqueId(&id) != ncclSuccess) return EFGP_ERR_NCCL;
  std::memcpy(id_out, &id, sizeof(id));
  return EFGP_OK;
}

efgp_status comm_init(efgp_plan *pl, const void *id, int nranks, int rank) {
  const NcclApi &a = nccl();
  if (!a.ok) {
    pl->err = "NCCL: libnccl.so.2 could not be loaded";
    return EFGP_ERR_NCCL;
  }
  if (nranks < 1 || rank < 0 || rank >= nranks) {
    pl->err = "comm_init: need 0 <= rank < nranks";
    return EFGP_ERR_INVALID;
  }
  comm_destroy(pl);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  EFGP_CUDA(cudaSetDevice(pl->device));
  ncclComm_t c = nullptr;
  EFGP_TRY(nccl_check(pl, a.commInitRank(&c, nranks, uid, rank), "commInitRank"));
  pl->comm = c;
  pl->comm_size = nranks;
  pl->comm_rank = rank;
  if (!pl->comm_buf) EFGP_CUDA(cudaMalloc((void **)&pl->comm_buf, 4 * sizeof(double)));  // count | min | fail
  return EFGP_OK;
}

void comm_destroy(efgp_plan *pl) {
  if (pl->comm && nccl().ok) nccl().commDestroy(static_cast<ncclComm_t>(pl->comm));
  pl->comm = nullptr;
  pl->comm_size = 0;
}

// in-place sum over ranks of n doubles (device pointer) on the library stream
efgp_status comm_sum(efgp_plan *pl, double *buf, size_t n) {
  return nccl_check(pl, nccl().allReduce(buf, buf, n, ncclFloat64, ncclSum, static_cast<ncclComm_t>(pl->comm),
                                         pl->stream),
                    "allReduce");
}

// sum of an int64 count, min of a double and max of a failure flag over ranks (host values in,
// host values out).  Every rank calls it after its local step, whether that step failed or not, so
// the collectives always match up; *fail then says whether ANY rank failed.
efgp_status comm_count_min(efgp_plan *pl, int64_t *count, double *minval, int *fail) {
  double h[3] = {(double)*count, minval ? *minval : 0.0, fail ? (double)*fail : 0.0};
  EFGP_CUDA(cudaMemcpyAsync(pl->comm_buf, h, sizeof(h), cudaMemcpyHostToDevice, pl->stream));
  const NcclApi &a = nccl();
  ncclComm_t c = static_cast<ncclComm_t>(pl->comm);
  EFGP_TRY(nccl_check(pl, a.allReduce(pl->comm_buf, pl->comm_buf, 1, ncclFloat64, ncclSum, c, pl->stream), "allReduce"));
  EFGP_TRY(nccl_check(pl, a.allReduce(pl->comm_buf + 1, pl->comm_buf + 1, 1, ncclFloat64, ncclMin, c, pl->stream),
                      "allReduce"));
  EFGP_TRY(nccl_check(pl, a.allReduce(pl->comm_buf + 2, pl->comm_buf + 2, 1, ncclFloat64, ncclMax, c, pl->stream),
                      "allReduce"));
  EFGP_CUDA(cudaMemcpyAsync(h, pl->comm_buf, sizeof(h), cudaMemcpyDeviceToHost, pl->stream));
  EFGP_CUDA(cudaStreamSynchronize(pl->stream));
  *count = (int64_t)(h[0] + 0.5);  // exact below 2^53 points
  if (minval) *minval = h[1];
  if (fail) *fail = h[2] > 0.0;
  return EFGP_OK;
}

}  // namespace efgp
