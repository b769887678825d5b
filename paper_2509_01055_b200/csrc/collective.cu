// N1 / N2 — the data-parallel collectives of the step at the C ABI (NCCL).
//
// Reference being replaced: the serial per-group loop and aggregation of
// cli.loss (cli.py:309-344); groups are independent, so ranks
// own whole groups and only exchange
//   N1  the report's additive partials (12 doubles, include/toolloop_b200.h
//       TL_REPORT_LEN) -> every rank holds the global report, and
//   N2  the LM-head weight gradient dW [V, H] fp32 (all-reduce, or
//       reduce-scatter into a row shard when W is partitioned).
// NCCL is resolved at run time (dlopen "libnccl.so.2": inside a PyTorch
// process that is the NCCL torch already loaded) so the library carries no
// link-time NCCL dependency and the drop-in .so loads on hosts without it
// (tl_nccl_available() == 0; every other entry point still works).
// Everything is stream-ordered on the caller's stream; nothing allocates.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "tl_common.cuh"
#include "toolloop_b200.h"

namespace tl {
namespace {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*comm_count)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*reduce_scatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                 ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      return fn != nullptr;
    };
    api.ok = sym(api.get_unique_id, "ncclGetUniqueId") &&
             sym(api.comm_init_rank, "ncclCommInitRank") &&
             sym(api.comm_destroy, "ncclCommDestroy") && sym(api.comm_count, "ncclCommCount") &&
             sym(api.all_reduce, "ncclAllReduce") &&
             sym(api.reduce_scatter, "ncclReduceScatter") &&
             sym(api.error_string, "ncclGetErrorString") && sym(api.get_version, "ncclGetVersion");
  });
  return api;
}

#define TL_NCCL_TRY(expr)                                                               \
  do {                                                                                  \
    ncclResult_t r_ = (expr);                                                           \
    if (r_ != ncclSuccess) {                                                            \
      set_error("%s:%d: NCCL: %s", __FILE__, __LINE__, nccl().error_string(r_));        \
      return TL_ERR_COMM;                                                               \
    }                                                                                   \
  } while (0)

#define TL_NCCL_REQUIRE() \
  TL_REQUIRE(nccl().ok, TL_ERR_COMM, "NCCL unavailable (libnccl.so.2 could not be loaded)")

// After an element-wise sum of whole reports: the ratio fields are
// recomputed from the summed additive partials (cli.py:337-344 order).
__global__ void report_finalize_kernel(double* rep, int agg) {
  const double masked = rep[2], groups = rep[4];
  if (agg == 1)
    rep[0] = masked > 0 ? rep[11] / masked : 0.0;
  else
    rep[0] = groups > 0 ? rep[11] / groups : 0.0;
  rep[1] = masked > 0 ? rep[8] / masked : 0.0;
  rep[3] = masked > 0 ? rep[9] / masked : 0.0;
}

}  // namespace
}  // namespace tl

using namespace tl;

extern "C" int tl_nccl_available(void) { return nccl().ok ? 1 : 0; }

extern "C" int tl_nccl_version(void) {
  int v = 0;
  if (!nccl().ok || nccl().get_version(&v) != ncclSuccess) return 0;
  return v;
}

extern "C" int tl_nccl_unique_id(uint8_t* id_out) {
  TL_REQUIRE(id_out, TL_ERR_INVALID_ARG, "id_out is NULL");
  TL_NCCL_REQUIRE();
  ncclUniqueId id;
  TL_NCCL_TRY(nccl().get_unique_id(&id));
  static_assert(sizeof(id) == TL_NCCL_UNIQUE_ID_BYTES, "ncclUniqueId size");
  memcpy(id_out, &id, sizeof(id));
  return TL_OK;
}

extern "C" int tl_nccl_comm_init(void** comm_out, const uint8_t* id, int32_t nranks, int32_t rank) {
  TL_REQUIRE(comm_out && id, TL_ERR_INVALID_ARG, "NULL argument");
  TL_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, TL_ERR_INVALID_ARG,
             "rank %d outside [0, %d)", rank, nranks);
  TL_NCCL_REQUIRE();
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  TL_NCCL_TRY(nccl().comm_init_rank(&c, nranks, uid, rank));
  *comm_out = c;
  return TL_OK;
}

extern "C" int tl_nccl_comm_destroy(void* comm) {
  if (!comm) return TL_OK;
  TL_NCCL_REQUIRE();
  TL_NCCL_TRY(nccl().comm_destroy(static_cast<ncclComm_t>(comm)));
  return TL_OK;
}

extern "C" int tl_nccl_comm_size(void* comm, int32_t* nranks) {
  TL_REQUIRE(comm && nranks, TL_ERR_INVALID_ARG, "NULL argument");
  TL_NCCL_REQUIRE();
  int n = 0;
  TL_NCCL_TRY(nccl().comm_count(static_cast<ncclComm_t>(comm), &n));
  *nranks = n;
  return TL_OK;
}

extern "C" int tl_allreduce_scalars(void* comm, double* x, int32_t n, tl_stream_t stream) {
  TL_REQUIRE(comm && (x || n == 0) && n >= 0, TL_ERR_INVALID_ARG, "bad arguments");
  if (n == 0) return TL_OK;
  TL_NCCL_REQUIRE();
  TL_NCCL_TRY(nccl().all_reduce(x, x, static_cast<size_t>(n), ncclFloat64, ncclSum,
                                static_cast<ncclComm_t>(comm), static_cast<cudaStream_t>(stream)));
  return TL_OK;
}

extern "C" int tl_allreduce_report(void* comm, double* report, int32_t agg, tl_stream_t stream) {
  TL_REQUIRE(agg == 0 || agg == 1, TL_ERR_INVALID_ARG, "agg must be 0 or 1");
  if (int e = tl_allreduce_scalars(comm, report, TL_REPORT_LEN, stream)) return e;
  report_finalize_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(report, agg);
  TL_LAUNCH_CHECK();
  count_launch();
  return TL_OK;
}

extern "C" int tl_allreduce_f32(void* comm, float* buf, int64_t n, tl_stream_t stream) {
  TL_REQUIRE(comm && (buf || n == 0) && n >= 0, TL_ERR_INVALID_ARG, "bad arguments");
  if (n == 0) return TL_OK;
  TL_NCCL_REQUIRE();
  TL_NCCL_TRY(nccl().all_reduce(buf, buf, static_cast<size_t>(n), ncclFloat32, ncclSum,
                                static_cast<ncclComm_t>(comm), static_cast<cudaStream_t>(stream)));
  return TL_OK;
}

extern "C" int tl_reduce_scatter_f32(void* comm, const float* buf, float* shard, int64_t shard_n,
                                     tl_stream_t stream) {
  TL_REQUIRE(comm && buf && shard && shard_n >= 0, TL_ERR_INVALID_ARG, "bad arguments");
  if (shard_n == 0) return TL_OK;
  TL_NCCL_REQUIRE();
  TL_NCCL_TRY(nccl().reduce_scatter(buf, shard, static_cast<size_t>(shard_n), ncclFloat32, ncclSum,
                                    static_cast<ncclComm_t>(comm),
                                    static_cast<cudaStream_t>(stream)));
  return TL_OK;
}
