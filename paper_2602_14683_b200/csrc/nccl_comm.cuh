// Native NCCL communicator of a context: the packed fp64
// Num/Den partials of a sharded block update are summed in place with
// ncclAllReduce on the engine's own stream, so the whole outer iteration
// (collectives included) stays inside one captured CUDA graph and no host
// code runs per block update.
//
// libnccl is resolved at run time (dlopen of the already-loaded
// libnccl.so.2 when torch brought one in, else the system one): libntfg.so
// itself has no NCCL dependency, and single-device fits never touch it.
// Only the NCCL *types* come from <nccl.h>.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "engine.cuh"

namespace ntfg {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  int (*version)(int*) = nullptr;

  static NcclApi& get() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
      void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
      if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
      if (!h) {
        err = std::string("libnccl.so.2 not found: ") + dlerror();
        return;
      }
      api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
      api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
      api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
      api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
      api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
      api.version = reinterpret_cast<decltype(api.version)>(dlsym(h, "ncclGetVersion"));
      if (!api.get_unique_id || !api.comm_init_rank || !api.all_reduce || !api.comm_destroy)
        err = "libnccl.so.2 lacks the required entry points";
    });
    if (!api.all_reduce || !err.empty()) throw Error(NTFG_ERR_COMM, err.empty() ? "NCCL unavailable" : err);
    return api;
  }
  void check(ncclResult_t r, const char* what) const {
    if (r != ncclSuccess)
      throw Error(NTFG_ERR_COMM, std::string(what) + ": " + (error_string ? error_string(r) : "NCCL error"));
  }
};

// In-place fp64 sum across the communicator, ordered on `stream`.  NCCL's
// ring / tree / NVLS algorithms deliver the same bytes to every rank (each
// chunk is reduced once, then broadcast), so replicated factors stay
// bitwise identical after the identical MU step on every rank.
inline void nccl_allreduce_sum(void* comm, double* buf, size_t count, cudaStream_t stream) {
  NcclApi& api = NcclApi::get();
  api.check(api.all_reduce(buf, buf, count, ncclDouble, ncclSum, static_cast<ncclComm_t>(comm), stream),
            "ncclAllReduce");
}

inline void* nccl_comm_init(const void* id_bytes, int nranks, int rank) {
  NcclApi& api = NcclApi::get();
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, sizeof(id));
  ncclComm_t comm = nullptr;
  api.check(api.comm_init_rank(&comm, nranks, id, rank), "ncclCommInitRank");
  return comm;
}

inline void nccl_comm_destroy(void* comm) {
  if (!comm) return;
  NcclApi& api = NcclApi::get();
  api.comm_destroy(static_cast<ncclComm_t>(comm));
}

inline void nccl_unique_id(void* out) {
  NcclApi& api = NcclApi::get();
  ncclUniqueId id;
  api.check(api.get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
}

}  // namespace ntfg
