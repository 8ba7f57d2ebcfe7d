// In-library NCCL rank exchange of point-sharded solves (include/pba_gpu.h pba_gpu_set_exchange_nccl).
//
// The engine's exchange points (Engine::xreduce / xsum_i64) call an exchange function
// on the handle's stream; this one issues the NCCL collectives itself (all-gather of the rank
// partials, exact int64 all-reduce of the fixed-point Schur accumulator) on that stream, so a
// sharded candidate evaluation makes no call back into the host language and no host round trip.
// NCCL is resolved with dlopen when the first communicator is created: libpba_gpu.so keeps no link
// dependency on it, and in a process that already loaded NCCL (e.g. through torch) the loaded
// library is reused.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include "engine.hpp"

namespace pba_b200 {
namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string error;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) {
      api.error = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) { return dlsym(lib, n); };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    if (!api.get_unique_id || !api.comm_init_rank || !api.all_gather || !api.all_reduce || !api.comm_destroy)
      api.error = "libnccl.so.2 lacks the collective entry points";
  });
  return api;
}

void check_nccl(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw PbaError(PBA_E_CUDA, std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "NCCL error"));
}

struct NcclCtx {
  ncclComm_t comm = nullptr;
  ~NcclCtx() {
    if (comm) nccl().comm_destroy(comm);
  }
};

// the exchange function (pba_exchange_fn) over the handle's communicator, on the handle's stream
int nccl_exchange(void* ctx, int op, void* send, void* recv, int64_t count, void* stream) {
  const NcclCtx* c = static_cast<const NcclCtx*>(ctx);
  const NcclApi& api = nccl();
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ncclResult_t r = ncclInvalidUsage;
  if (op == PBA_X_GATHER) r = api.all_gather(send, recv, static_cast<size_t>(count), ncclFloat64, c->comm, s);
  else if (op == PBA_X_SUM_I64)  // uint64 wrap-around sum == the int64 sum of the fixed-point accumulators
    r = api.all_reduce(send, send, static_cast<size_t>(count), ncclUint64, ncclSum, c->comm, s);
  return r == ncclSuccess ? 0 : 1;
}

}  // namespace

void nccl_unique_id(void* out128) {
  const NcclApi& api = nccl();
  if (!api.error.empty()) throw PbaError(PBA_E_CUDA, api.error);
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  check_nccl(api.get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
}

void Engine::set_exchange_nccl(const void* id128, int rank, int world, int64_t n_total) {
  const NcclApi& api = nccl();
  if (!api.error.empty()) throw PbaError(PBA_E_CUDA, api.error);
  if (world < 1 || rank < 0 || rank >= world) throw PbaError(PBA_E_ARG, "set_exchange_nccl: need 0 <= rank < world");
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  auto ctx = std::make_shared<NcclCtx>();
  check_nccl(api.comm_init_rank(&ctx->comm, world, id, rank), "ncclCommInitRank");
  set_exchange(rank, world, n_total, nccl_exchange, ctx.get());
  xch_owner_ = ctx;  // destroyed with the handle (or when the exchange is replaced)
}

}  // namespace pba_b200
