// Host-side engine: context, device buffers, errors, launch helpers.
#pragma once
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ntfg.h"

namespace ntfg {

// Internal exception carrying an ntfg_status; converted at the C ABI.
struct Error : std::runtime_error {
  ntfg_status code;
  Error(ntfg_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    if (e == cudaErrorMemoryAllocation)
      throw Error(NTFG_ERR_OOM, std::string(what) + ": " + cudaGetErrorString(e));
    throw Error(NTFG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}
#define NTFG_CUDA(x) ::ntfg::cuda_check((x), #x)
#define NTFG_LAUNCHED(ctx) do { ::ntfg::cuda_check(cudaPeekAtLastError(), "kernel launch"); (ctx).stats.kernel_launches++; } while (0)

// Named, growable device allocations reused across calls of one context.
class BufferCache {
 public:
  ~BufferCache() { release(); }
  void* get(const std::string& name, size_t bytes) {
    auto it = bufs_.find(name);
    if (it != bufs_.end() && it->second.bytes >= bytes) return it->second.ptr;
    if (it != bufs_.end()) {
      cudaFree(it->second.ptr);
      bufs_.erase(it);
    }
    void* p = nullptr;
    if (bytes > 0) cuda_check(cudaMalloc(&p, bytes), ("cudaMalloc " + name).c_str());
    bufs_[name] = {p, bytes};
    return p;
  }
  void release() {
    for (auto& kv : bufs_) cudaFree(kv.second.ptr);
    bufs_.clear();
  }

 private:
  struct Buf { void* ptr; size_t bytes; };
  std::map<std::string, Buf> bufs_;
};

// Pinned host staging, growable.
class PinnedCache {
 public:
  ~PinnedCache() { if (ptr_) cudaFreeHost(ptr_); }
  void* get(size_t bytes) {
    if (bytes > bytes_) {
      if (ptr_) cudaFreeHost(ptr_);
      ptr_ = nullptr;
      cuda_check(cudaMallocHost(&ptr_, bytes), "cudaMallocHost");
      bytes_ = bytes;
    }
    return ptr_;
  }
 private:
  void* ptr_ = nullptr;
  size_t bytes_ = 0;
};

struct Context {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ntfg_allreduce_fn allreduce = nullptr;
  void* allreduce_user = nullptr;
  ntfg_stats stats{};
  bool profile = false;
  double* comm_buf = nullptr;
  size_t comm_cap = 0;
  void* nccl = nullptr;  // native communicator (nccl_comm.cuh); preferred over the hook
  int nccl_ranks = 0;
  bool has_comm() const { return allreduce != nullptr || nccl != nullptr; }
  BufferCache bufs;
  PinnedCache pinned;
  int sm_count = 148;

  // ---- per-kernel-class profiling (eager mode) ----
  struct ProfEv { int cls; cudaEvent_t a, b; };
  std::vector<ProfEv> prof_events;
  size_t prof_used = 0;
  int prof_begin(int cls) {
    if (!profile) return -1;
    if (prof_used == prof_events.size()) {
      ProfEv p{cls, nullptr, nullptr};
      cuda_check(cudaEventCreate(&p.a), "cudaEventCreate");
      cuda_check(cudaEventCreate(&p.b), "cudaEventCreate");
      prof_events.push_back(p);
    }
    ProfEv& p = prof_events[prof_used];
    p.cls = cls;
    cuda_check(cudaEventRecord(p.a, stream), "cudaEventRecord");
    return int(prof_used++);
  }
  void prof_end(int h) {
    if (h < 0) return;
    cuda_check(cudaEventRecord(prof_events[size_t(h)].b, stream), "cudaEventRecord");
  }
  void prof_collect() {
    if (!profile) return;
    cuda_check(cudaStreamSynchronize(stream), "sync");
    for (size_t i = 0; i < prof_used; ++i) {
      float ms = 0.f;
      cuda_check(cudaEventElapsedTime(&ms, prof_events[i].a, prof_events[i].b), "elapsed");
      switch (prof_events[i].cls) {
        case 0: stats.recon_ms += ms; stats.recon_launches++; break;
        case 1: stats.contract_ms += ms; stats.contract_launches++; break;
        default: stats.other_ms += ms; stats.other_launches++; break;
      }
    }
    prof_used = 0;
  }
  ~Context() {
    for (auto& p : prof_events) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
  }

  void activate() const { cuda_check(cudaSetDevice(device), "cudaSetDevice"); }
  template <typename T>
  T* buf(const std::string& name, size_t count) {
    return static_cast<T*>(bufs.get(name, count * sizeof(T)));
  }
  void sync() { cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize"); }
  void h2d(void* dst, const void* src, size_t bytes) {
    if (bytes) cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream), "H2D");
  }
  void d2h(void* dst, const void* src, size_t bytes) {
    if (bytes) cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, stream), "D2H");
  }
  void d2d(void* dst, const void* src, size_t bytes) {
    if (bytes && dst != src)
      cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, stream), "D2D");
  }
};

// Host-side config checks: validate_fit_config (reference config.cpp:7-18).
inline void validate_config(const ntfg_fit_config& c) {
  if (!(c.beta >= 0.0 && c.beta < 2.0)) throw Error(NTFG_ERR_DOMAIN, "beta must lie in [0, 2)");
  if (!(c.eps > 0.0)) throw Error(NTFG_ERR_DOMAIN, "eps must be positive");
  if (c.inner_steps < 1) throw Error(NTFG_ERR_DOMAIN, "inner_steps must be >= 1");
  if (c.rank < 1) throw Error(NTFG_ERR_DOMAIN, "rank must be >= 1");
  for (uint32_t i = 0; i < c.n_ranks; ++i)
    if (c.ranks[i] < 1) throw Error(NTFG_ERR_DOMAIN, "every core rank must be >= 1");
  if (c.has_data_floor && !(c.data_floor > 0.0)) throw Error(NTFG_ERR_DOMAIN, "data_floor must be positive");
  if (!(c.extrap_cap >= 0.0) || !(c.extrap_delta > 0.0))
    throw Error(NTFG_ERR_DOMAIN, "invalid extrapolation constants");
}

inline double gamma_of(double beta) {
  if (!(beta >= 0.0 && beta < 2.0)) throw Error(NTFG_ERR_DOMAIN, "beta must lie in [0, 2)");
  return beta < 1.0 ? 1.0 / (2.0 - beta) : 1.0;
}

// Fit-loop bookkeeping shared by CP and Tucker drivers (reference
// fit_common.hpp:14-53).
inline void check_finite_loss(double loss, double beta) {
  if (std::isnan(loss)) throw Error(NTFG_ERR_NUMERICAL, "fit aborted: objective is NaN");
  if (std::isinf(loss)) {
    if (beta == 0.0)
      throw Error(NTFG_ERR_NUMERICAL,
                  "fit aborted: objective is infinite (beta = 0 with zero data entries; "
                  "apply a positive data floor, e.g. --data-floor)");
    throw Error(NTFG_ERR_NUMERICAL, "fit aborted: objective is infinite");
  }
}

// Domain flags raised by kernels (see device_math.cuh).
inline void raise_flags(unsigned f) {
  if (f & 1u) throw Error(NTFG_ERR_DOMAIN, "d_beta: second argument must be positive");
  if (f & 2u) throw Error(NTFG_ERR_DOMAIN, "d_beta: first argument must be nonnegative");
  if (f & 4u) throw Error(NTFG_ERR_DOMAIN, "chi1: entries must be strictly positive");
}

inline int pad_rank(int64_t r) {
  if (r <= 8) return 8;
  if (r <= 16) return 16;
  if (r <= 32) return 32;
  if (r <= 64) return 64;
  throw Error(NTFG_ERR_SHAPE, "rank above 64 is not supported by the streaming kernels");
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace ntfg
