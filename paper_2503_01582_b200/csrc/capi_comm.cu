// capi_comm.cu -- C ABI: the one collective of the path, the Reptile meta-gradient
// all-reduce over NCCL (BASELINE cfg4 at 2/4/8 GPUs).
//
// meta_train (meta.cpp:94-120) adapts one task per meta-step and interpolates
// theta <- reptile_update(theta, adapted, beta) (meta.cpp:83-92). Batched across
// ranks, every rank adapts its share of a meta-batch of T tasks from the same
// theta, and
//     theta <- (1 - beta) theta + beta (theta + sum_i (theta_i - theta) / T)
// = reptile_update(theta, mean_i theta_i, beta) by linearity.
// prenom_reptile_step does the whole exchange on the context stream with no
// host synchronisation: one pass sums this rank's task deltas
// (k_reptile_delta_sum), ncclAllReduce sums the P floats over the ranks in
// place (NVLink / NVSwitch; NCCL picks ring, tree or NVLS), and k_reptile_apply
// interpolates. The communicator lives in the context (one per GPU process).
//
// NCCL is loaded at run time (dlopen "libnccl.so.2", or PRENOM_NCCL_LIB): the
// library has no link-time NCCL dependency, and in a process that already
// loaded one (e.g. the one bundled with torch) the same copy is used.
#include <dlfcn.h>

#include <mutex>

#include "capi_internal.cuh"

#if __has_include(<nccl.h>)
#include <nccl.h>
#else
// The stable NCCL 2.x C ABI subset used here.
typedef struct ncclComm* ncclComm_t;
typedef enum { ncclSuccess = 0 } ncclResult_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef enum { ncclFloat32 = 7 } ncclDataType_t;
typedef enum { ncclSum = 0 } ncclRedOp_t;
#endif

static_assert(sizeof(ncclUniqueId) == PRENOM_COMM_ID_BYTES, "NCCL unique id size");

using namespace prenom;
using namespace prenom_capi;

namespace {

struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* path = getenv("PRENOM_NCCL_LIB");
    void* h = dlopen(path ? path : "libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      api.err = std::string("cannot load NCCL: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    api.get_version = reinterpret_cast<decltype(api.get_version)>(sym("ncclGetVersion"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.all_reduce && api.comm_destroy && api.error_string;
    if (!api.ok) api.err = "NCCL library lacks the required entry points";
  });
  return api;
}

#define NCCL_TRY(expr)                                                                              \
  do {                                                                                              \
    ncclResult_t _r = (expr);                                                                       \
    if (_r != ncclSuccess) return fail(PRENOM_CUDA, std::string(#expr) + ": " + nccl().error_string(_r)); \
  } while (0)

}  // namespace

namespace prenom_capi {
void comm_destroy(prenom_ctx_t ctx) {
  if (ctx && ctx->comm) {
    nccl().comm_destroy(static_cast<ncclComm_t>(ctx->comm));
    ctx->comm = nullptr;
    ctx->comm_size = 1;
    ctx->comm_rank = 0;
  }
}
}  // namespace prenom_capi

extern "C" {

prenom_status prenom_comm_unique_id(uint8_t* id) {
  if (!id) return fail(PRENOM_USAGE, "NULL argument");
  NcclApi& api = nccl();
  if (!api.ok) return fail(PRENOM_CUDA, api.err);
  ncclUniqueId u;
  NCCL_TRY(api.get_unique_id(&u));
  std::memcpy(id, &u, sizeof u);
  return PRENOM_OK;
}

prenom_status prenom_ctx_init_comm(prenom_ctx_t ctx, int nranks, int rank, const uint8_t* id) {
  if (!ctx || !id) return fail(PRENOM_USAGE, "NULL argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(PRENOM_USAGE, "bad rank / world size");
  NcclApi& api = nccl();
  if (!api.ok) return fail(PRENOM_CUDA, api.err);
  CUDA_TRY(cudaSetDevice(ctx->device));
  comm_destroy(ctx);
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof u);
  ncclComm_t c = nullptr;
  NCCL_TRY(api.comm_init_rank(&c, nranks, u, rank));
  ctx->comm = c;
  ctx->comm_size = nranks;
  ctx->comm_rank = rank;
  return PRENOM_OK;
}

prenom_status prenom_ctx_comm_info(prenom_ctx_t ctx, int* nranks, int* rank, int* nccl_version) {
  if (!ctx) return fail(PRENOM_USAGE, "NULL context");
  if (nranks) *nranks = ctx->comm ? ctx->comm_size : 0;
  if (rank) *rank = ctx->comm_rank;
  if (nccl_version) {
    *nccl_version = 0;
    NcclApi& api = nccl();
    if (api.ok && api.get_version) api.get_version(nccl_version);
  }
  return PRENOM_OK;
}

prenom_status prenom_reptile_step(prenom_object_t meta, const prenom_object_t* adapted, int n_adapted, int n_tasks,
                                  float beta) {
  NvtxRange nvtx_("prenom.reptile_step");
  if (!meta || (n_adapted > 0 && !adapted)) return fail(PRENOM_USAGE, "NULL argument");
  if (n_adapted < 0 || n_tasks < 1 || n_adapted > n_tasks) return fail(PRENOM_USAGE, "bad task counts");
  prenom_ctx_s* c = meta->ctx;
  const bool collective = c->comm != nullptr;  // (a 1-rank communicator still runs the all-reduce)
  if (!collective && n_adapted != n_tasks)
    return fail(PRENOM_USAGE, "reptile_step: tasks on other ranks need a communicator (prenom_ctx_init_comm)");
  for (int i = 0; i < n_adapted; ++i) {
    if (!adapted[i]) return fail(PRENOM_USAGE, "NULL object");
    if (adapted[i]->P != meta->P) return fail(PRENOM_DATA, "reptile_update: parameter vectors differ in length");
  }
  CUDA_TRY(cudaSetDevice(c->device));
  for (int i = 0; i < n_adapted; ++i)
    if (adapted[i]->ctx != c) CUDA_TRY(cudaStreamSynchronize(adapted[i]->ctx->stream));
  cudaStream_t st = c->stream;
  if (!collective && n_tasks == 1) {  // the reference update itself (meta.cpp:83-92)
    CUDA_TRY(launch_reptile_update(meta->P, meta->params.p, adapted[0]->params.p, beta, st));
    c->launches += 1;
    return PRENOM_OK;
  }
  CUDA_TRY(c->reptile_sum.ensure(meta->P));
  if (n_adapted > 0) {
    CUDA_TRY(c->reptile_ptrs.ensure((size_t)n_adapted));
    std::vector<const float*> h(n_adapted);
    for (int i = 0; i < n_adapted; ++i) h[i] = adapted[i]->params.p;
    // (pageable copy: staged by the driver, stream-ordered before the kernel)
    CUDA_TRY(cudaMemcpyAsync(c->reptile_ptrs.p, h.data(), sizeof(const float*) * n_adapted, cudaMemcpyHostToDevice, st));
    CUDA_TRY(launch_reptile_delta_sum(meta->P, meta->params.p, c->reptile_ptrs.p, n_adapted, c->reptile_sum.p, st));
    c->launches += 1;
  } else {
    CUDA_TRY(cudaMemsetAsync(c->reptile_sum.p, 0, meta->P * sizeof(float), st));  // no task here this step
  }
  if (collective)
    NCCL_TRY(nccl().all_reduce(c->reptile_sum.p, c->reptile_sum.p, meta->P, ncclFloat32, ncclSum,
                               static_cast<ncclComm_t>(c->comm), st));
  CUDA_TRY(launch_reptile_apply(meta->P, meta->params.p, c->reptile_sum.p, 1.f / (float)n_tasks, beta, st));
  c->launches += 1;
  return PRENOM_OK;
}

}  // extern "C"
