// Tucker-specific kernels.  The E-sized streaming passes reuse the CP
// kernels with a row table: X^ = sum_j Y(row, j) A_L(k, j) where Y is the
// partial reconstruction over the prefix modes (reference tucker_reconstruct,
// tensor.cpp:408-419), and Num_L(k, j) = sum_rows P(row,k) Y(row,j).  What is
// left here is the small (O(E J / I_L)) fp64 machinery:
//   ttm_kernel       one mode product of a small tensor (replace_axis,
//                    tensor.cpp:315-337; mode_n_product 165-190)
//   rowgemm_kernel   T(row, j) = sum_k S(row,k) F(k,j): the first, E-sized
//                    step of tucker_multimode_contract (tensor.cpp:421-456)
//                    and of the fused factor contraction (514-560)
//   core_pair_kernel Num(i_n, j_n) = sum_{j_-n} S(j_-n, i_n, j_L) G(j)
//                    (the core pairing of tensor.cpp:545-558)
//   mu_dense_kernel  MU step + chi transforms on dense num/den blocks
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "device_math.cuh"

namespace ntfg {

// out[o][a][q] = sum_b in[o][b][q] * F(a, b), F(a,b) = trans ? M[b*na + a] : M[a*nb + b]
static __global__ void ttm_kernel(const double* __restrict__ in, int64_t outer, int64_t nb, int64_t inner,
                           const double* __restrict__ M, int64_t na, int trans,
                           double* __restrict__ out) {
  const int64_t total = outer * na * inner;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t q = idx % inner;
    const int64_t a = (idx / inner) % na;
    const int64_t o = idx / (inner * na);
    const double* src = in + o * nb * inner + q;
    double acc = 0.0;
    if (trans) {
      for (int64_t b = 0; b < nb; ++b) acc += src[b * inner] * M[b * na + a];
    } else {
      const double* mrow = M + a * nb;
      for (int64_t b = 0; b < nb; ++b) acc += src[b * inner] * mrow[b];
    }
    out[idx] = acc;
  }
}

// T(row, j) = sum_k S(row, k) F(k, j); F staged as T [K][JP] (zero padded).
// One warp per row, lanes stride k; fp64 result.
template <typename T, int JP>
static __global__ void __launch_bounds__(256) rowgemm_kernel(const T* __restrict__ S, int64_t rows,
                                                      int64_t K, const T* __restrict__ F, int J,
                                                      double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t row = warp; row < rows; row += nwarps) {
    T acc[JP];
#pragma unroll
    for (int j = 0; j < JP; ++j) acc[j] = T(0);
    const T* srow = S + row * K;
    for (int64_t k = lane; k < K; k += 32) {
      const T s = __ldg(srow + k);
      const T* f = F + k * JP;
#pragma unroll
      for (int j = 0; j < JP; ++j) acc[j] = fma(s, __ldg(f + j), acc[j]);
    }
#pragma unroll
    for (int j = 0; j < JP; ++j) {
      double v = warp_sum(double(acc[j]));
      if (lane == 0 && j < J) out[row * J + j] = v;
    }
  }
}

// Num(i_n, j_n) = sum over j_-n of S[d_0..d_{L-1}, j_L] * G[j_0..j_L], where
// d_m = J_m for m != n and d_n = I_n (S is the contraction of T over every
// prefix mode but n); L = order - 1 is the last mode (its j_L is shared).
struct PairParams {
  int order, n;
  int64_t In;
  int64_t J[8];
  const double* S;
  const double* G;
  double* out;  // [In][J_n]
};

static __global__ void core_pair_kernel(const PairParams p) {
  const int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t Jn = p.J[p.n];
  if (idx >= p.In * Jn) return;
  const int64_t i = idx / Jn, jn = idx % Jn;
  int64_t rest = 1;
  for (int m = 0; m < p.order; ++m)
    if (m != p.n) rest *= p.J[m];
  double acc = 0.0;
  for (int64_t t = 0; t < rest; ++t) {
    // decode t over modes != n (row-major, last fastest)
    int64_t rem = t, gidx = 0, sidx = 0, gstride = 1, sstride = 1;
    int64_t coords[8];
    for (int m = p.order - 1; m >= 0; --m) {
      if (m == p.n) {
        coords[m] = -1;
        continue;
      }
      coords[m] = rem % p.J[m];
      rem /= p.J[m];
    }
    for (int m = p.order - 1; m >= 0; --m) {
      const int64_t gc = (m == p.n) ? jn : coords[m];
      const int64_t sc = (m == p.n) ? i : coords[m];
      const int64_t sdim = (m == p.n) ? p.In : p.J[m];
      gidx += gc * gstride;
      gstride *= p.J[m];
      sidx += sc * sstride;
      sstride *= sdim;
    }
    acc += p.S[sidx] * p.G[gidx];
  }
  p.out[idx] = acc;
}

// out[o][q][m] = in[o][m][q]  (moves one axis to the back)
static __global__ void moveaxis_last_kernel(const double* in, int64_t outer, int64_t mid, int64_t inner,
                                     double* out) {
  const int64_t total = outer * mid * inner;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t m = idx % mid;
    const int64_t q = (idx / mid) % inner;
    const int64_t o = idx / (mid * inner);
    out[idx] = in[(o * mid + m) * inner + q];
  }
}

// out = max(anchor (num / max(den, eps))^gamma, eps) elementwise, + chi.
static __global__ void mu_dense_kernel(const double* anchor, const double* num, const double* den,
                                int64_t n, double gamma, double eps, double beta, double* out,
                                const double* ref, double* c1, double* c2, unsigned* flags) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double v = mu_step(anchor[i], num[i], den[i], gamma, eps);
  out[i] = v;
  if (ref) {
    unsigned bad = 0;
    c1[i] = chi1_entry(v, ref[i], beta, bad);
    c2[i] = chi2_entry(v, ref[i], beta, bad);
    if (bad && flags) atomicOr(flags, bad);
  }
}

}  // namespace ntfg
