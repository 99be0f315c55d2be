// Device-side COO ingestion for the sparse path (K7): linear keys, a stable
// radix sort, duplicate merge in input order (read_coo's dense `+=`,
// reference io.cpp:138) and, per mode, a stable re-sort by that mode's index
// cut into pieces of <= kCooPiece nonzeros that never straddle two keys.
// Everything runs on the device (CUB radix sorts and scans); the only host
// round trips are the merged count and each mode's piece count, which size
// the later launches.
#pragma once
#include <cub/cub.cuh>

#include <cstdint>
#include <string>

#include "coo_kernels.cuh"
#include "engine.cuh"

namespace ntfg {

struct CooKeyParams {
  int order;
  int64_t dims[kMaxOrder];
  int64_t nnz;
  const int32_t* idx;  // [nnz][order]
  int64_t* key;        // row-major linear index
  int64_t* pos;        // iota
  unsigned* bad;       // out-of-range flag
};

static __global__ void coo_key_kernel(const CooKeyParams p) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < p.nnz; j += int64_t(gridDim.x) * blockDim.x) {
    int64_t k = 0;
    bool ok = true;
    for (int m = 0; m < p.order; ++m) {
      const int32_t i = p.idx[j * p.order + m];
      ok = ok && i >= 0 && int64_t(i) < p.dims[m];
      k = k * p.dims[m] + (i >= 0 ? i : 0);
    }
    if (!ok) atomicOr(p.bad, 1u);
    p.key[j] = ok ? k : 0;
    p.pos[j] = j;
  }
}

// head[j] = 1 where a run of equal keys starts
static __global__ void coo_head_kernel(const int64_t* key, int64_t n, int32_t* head) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x)
    head[j] = (j == 0 || key[j] != key[j - 1]) ? 1 : 0;
}

// one thread per run head: the run's values summed in input order (the radix
// sort is stable, so positions within a run ascend), indices of the first
struct CooMergeParams {
  int order;
  int64_t n;
  const int64_t* key;
  const int64_t* pos;
  const int32_t* head;
  const int32_t* uid;   // exclusive scan of head
  const int32_t* idx;   // [nnz][order] input
  const void* val;      // input values
  int f32;
  int32_t* midx[kMaxOrder];  // merged SoA indices
  double* mval;
};

static __global__ void coo_merge_kernel(const CooMergeParams p) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < p.n; j += int64_t(gridDim.x) * blockDim.x) {
    if (!p.head[j]) continue;
    const int64_t u = p.uid[j];
    double v = 0.0;
    for (int64_t t = j; t < p.n && (t == j || !p.head[t]); ++t) {
      const int64_t q = p.pos[t];
      v += p.f32 ? double(static_cast<const float*>(p.val)[q]) : static_cast<const double*>(p.val)[q];
    }
    const int64_t first = p.pos[j];
    for (int m = 0; m < p.order; ++m) p.midx[m][u] = p.idx[first * p.order + m];
    p.mval[u] = v;
  }
}

static __global__ void coo_iota_kernel(int64_t n, int32_t* out) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x)
    out[j] = int32_t(j);
}

// sorted copy of one mode: every index column and the values gathered by perm
struct CooGatherParams {
  int order;
  int64_t n;
  const int32_t* perm;
  const int32_t* src_idx[kMaxOrder];
  const double* src_val;
  int32_t* dst_idx[kMaxOrder];
  double* dst_val;
};

static __global__ void coo_gather_kernel(const CooGatherParams p) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < p.n; j += int64_t(gridDim.x) * blockDim.x) {
    const int32_t q = p.perm[j];
    for (int m = 0; m < p.order; ++m) p.dst_idx[m][j] = p.src_idx[m][q];
    p.dst_val[j] = p.src_val[q];
  }
}

// nonzeros per key of a SORTED key array: the last element of each run finds
// the run's first element by binary search (one atomicAdd per nonzero on a few
// hundred hot addresses took 1.25 ms per mode at C4; this is a few microseconds)
static __global__ void coo_count_kernel(const int32_t* keys, int64_t n, int32_t* cnt) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x) {
    const int32_t k = keys[j];
    if (j + 1 < n && keys[j + 1] == k) continue;
    int64_t lo = 0, hi = j;  // first index with keys[idx] == k
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < k) lo = mid + 1;
      else hi = mid;
    }
    cnt[k] = int32_t(j + 1 - lo);
  }
}

static __global__ void coo_npieces_kernel(const int32_t* cnt, int64_t In, int64_t* np) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < In; i += int64_t(gridDim.x) * blockDim.x)
    np[i] = (int64_t(cnt[i]) + kCooPiece - 1) / kCooPiece;
}

// key i owns pieces [kpiece[i], kpiece[i+1]) starting at start[i] + t * kCooPiece
static __global__ void coo_pieces_kernel(const int64_t* start, const int32_t* cnt, const int64_t* kpiece, int64_t In,
                                         int64_t M, int64_t* piece_start) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < In; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t np = kpiece[i + 1] - kpiece[i];
    for (int64_t t = 0; t < np; ++t) piece_start[kpiece[i] + t] = start[i] + t * kCooPiece;
    if (i == In - 1) piece_start[kpiece[In]] = M;
  }
}

static __global__ void widen_kernel(const int32_t* in, int64_t n, int64_t* out) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x)
    out[j] = in[j];
}

inline int bits_for(int64_t v) {
  int b = 1;
  while (b < 63 && (int64_t(1) << b) <= v) ++b;
  return b;
}

}  // namespace ntfg
