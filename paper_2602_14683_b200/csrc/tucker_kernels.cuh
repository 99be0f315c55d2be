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

// ---------------------------------------------------------------------------
// Tiled versions for the sizes the Tucker configs use (C3: 256^3, core 16^3).
// ncu of the one-output-per-thread kernels above at C3 (profiles/r02_c3_launches.txt):
// rowgemm 525 us per call for a 67 MB stream (2% of HBM), ttm 75 us,
// core_pair 180 us -- all latency-bound, none near a roof.

// T(row, j) = sum_k S(row, k) F(k, j), fp32 streaming (the E-sized first step).
// CTA = 64 * (JP / 8) threads on a 128-row tile: thread = (row pair, 8 ranks).
// S moves global -> shared with 16-byte cp.async in 32-column stages (4-deep
// ring, XOR-swizzled 16-byte chunks so both the row-wise fills and the
// column-wise LDS.128 reads are conflict-free); F ([K][JP] fp32) stays in
// shared memory.  Per 4 columns a thread issues 2 + 8 LDS.128 and 32 FFMA2.
// fp32 partial sums per stage, fp64 across stages; fp64 result.
constexpr int kRgRows = 128, kRgCols = 32, kRgStages = 4;
template <int JP>
struct RgSmem {
  static constexpr size_t stage = size_t(kRgRows) * kRgCols * 4;
  static size_t total(int64_t K) { return kRgStages * stage + size_t(K) * JP * 4; }
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int sz = valid ? 16 : 0;  // zero-fill rows past the end
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(sz) : "memory");
}

template <int JP>
static __global__ void __launch_bounds__(64 * (JP / 8)) rowgemm_tiled_kernel(const float* __restrict__ S, int64_t rows,
                                                                              int64_t K, const float* __restrict__ F,
                                                                              int J, double* __restrict__ out) {
  constexpr int JH = JP / 8, NT = 64 * JH;
  extern __shared__ __align__(16) unsigned char rg_smem[];
  float* fs = reinterpret_cast<float*>(rg_smem + kRgStages * RgSmem<JP>::stage);  // [K][JP]
  const uint32_t sbase = uint32_t(__cvta_generic_to_shared(rg_smem));
  const int tid = threadIdx.x;
  const int rp = tid / JH, jh = tid % JH;  // rows 2 rp, 2 rp + 1; ranks 8 jh .. 8 jh + 7
  for (int i = tid; i < int(K) * JP / 4; i += NT)
    reinterpret_cast<float4*>(fs)[i] = __ldg(reinterpret_cast<const float4*>(F) + i);
  const int nks = int(K / kRgCols);
  const int64_t ntiles = (rows + kRgRows - 1) / kRgRows;
  // fill: 128 rows x 8 chunks of 16 B per stage; chunk c of row r lands at r * 128 + ((c ^ (r & 7)) * 16)
  auto fill = [&](int64_t tile, int ks, int slot) {
    const int64_t row0 = tile * kRgRows;
    for (int i = tid; i < kRgRows * 8; i += NT) {
      const int r = i >> 3, c = i & 7;
      const bool ok = row0 + r < rows;
      const float* src = S + (ok ? (row0 + r) : 0) * K + ks * kRgCols + c * 4;
      cp_async16(sbase + uint32_t(slot) * uint32_t(RgSmem<JP>::stage) + uint32_t(r * 128 + ((c ^ (r & 7)) << 4)), src, ok);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  __syncthreads();
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    double dacc[2][8];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int j = 0; j < 8; ++j) dacc[a][j] = 0.0;
    for (int s = 0; s < kRgStages - 1; ++s) {
      if (s < nks) fill(tile, s, s);
      else asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    for (int ks = 0; ks < nks; ++ks) {
      asm volatile("cp.async.wait_group %0;\n" ::"n"(kRgStages - 2) : "memory");
      __syncthreads();  // stage ks visible; slot of stage ks - 1 free
      if (ks + kRgStages - 1 < nks) fill(tile, ks + kRgStages - 1, (ks + kRgStages - 1) % kRgStages);
      else asm volatile("cp.async.commit_group;\n" ::: "memory");
      const unsigned char* st = rg_smem + size_t(ks % kRgStages) * RgSmem<JP>::stage;
      float2 acc[2][4];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[a][q] = make_float2(0.f, 0.f);
      const int r0 = 2 * rp, r1 = r0 + 1;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float4 s0 = *reinterpret_cast<const float4*>(st + r0 * 128 + ((c ^ (r0 & 7)) << 4));
        const float4 s1 = *reinterpret_cast<const float4*>(st + r1 * 128 + ((c ^ (r1 & 7)) << 4));
        const float sv0[4] = {s0.x, s0.y, s0.z, s0.w}, sv1[4] = {s1.x, s1.y, s1.z, s1.w};
        const float* frow = fs + size_t(ks * kRgCols + c * 4) * JP + jh * 8;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const float4 fa = *reinterpret_cast<const float4*>(frow + kk * JP);
          const float4 fb = *reinterpret_cast<const float4*>(frow + kk * JP + 4);
          const float2 f2[4] = {make_float2(fa.x, fa.y), make_float2(fa.z, fa.w), make_float2(fb.x, fb.y),
                                make_float2(fb.z, fb.w)};
          const float2 b0 = make_float2(sv0[kk], sv0[kk]), b1 = make_float2(sv1[kk], sv1[kk]);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            acc[0][q] = __ffma2_rn(f2[q], b0, acc[0][q]);
            acc[1][q] = __ffma2_rn(f2[q], b1, acc[1][q]);
          }
        }
      }
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          dacc[a][2 * q] += double(acc[a][q].x);
          dacc[a][2 * q + 1] += double(acc[a][q].y);
        }
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();  // every slot drained before the next tile refills them
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int64_t row = tile * kRgRows + 2 * rp + a;
      if (row < rows) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (jh * 8 + j < J) out[row * J + jh * 8 + j] = dacc[a][j];
      }
    }
  }
}

// Contracting mode product out[o][a][q] = sum_b in[o][b][q] M[b * NA + a]
// (trans form, NA = J_m <= 32, nb = I_m large): CTA = 8 warps on one
// (o, 32-wide q tile); warp w sums its eighth of b for all NA outputs with
// coalesced reads along q, then a fixed-order shared-memory reduction over
// the warps.  The one-output-per-thread ttm_kernel above runs a serial
// 256-term chain per thread on a few thousand threads.
template <int NA>
static __global__ void __launch_bounds__(256) ttm_contract_kernel(const double* __restrict__ in, int64_t outer,
                                                                  int64_t nb, int64_t inner,
                                                                  const double* __restrict__ M,
                                                                  double* __restrict__ out) {
  __shared__ double red[8][NA][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t qtiles = (inner + 31) / 32;
  for (int64_t blk = blockIdx.x; blk < outer * qtiles; blk += gridDim.x) {
    const int64_t o = blk / qtiles, q = (blk % qtiles) * 32 + lane;
    double acc[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) acc[a] = 0.0;
    const int64_t b0 = nb * w / 8, b1 = nb * (w + 1) / 8;
    if (q < inner) {
      const double* src = in + o * nb * inner + q;
#pragma unroll 4
      for (int64_t b = b0; b < b1; ++b) {
        const double v = src[b * inner];
        const double* mrow = M + b * NA;
#pragma unroll
        for (int a = 0; a < NA; ++a) acc[a] = fma(v, mrow[a], acc[a]);
      }
    }
#pragma unroll
    for (int a = 0; a < NA; ++a) red[w][a][lane] = acc[a];
    __syncthreads();
    for (int i = threadIdx.x; i < NA * 32; i += 256) {
      const int a = i >> 5, l = i & 31;
      const int64_t qq = (blk % qtiles) * 32 + l;
      if (qq < inner) {
        double s = red[0][a][l];
#pragma unroll
        for (int ww = 1; ww < 8; ++ww) s += red[ww][a][l];
        out[(o * NA + a) * inner + qq] = s;
      }
    }
    __syncthreads();
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

constexpr int kPairTab = 1024;  // offset-table entries (prod of the J_m, m != n)
static __global__ void core_pair_kernel(const PairParams p) {
  // offsets of every j_-n into S and G, decoded once per block instead of
  // per (thread, term)
  __shared__ int stab[kPairTab], gtab[kPairTab];
  const int64_t Jn = p.J[p.n];
  int64_t rest = 1;
  for (int m = 0; m < p.order; ++m)
    if (m != p.n) rest *= p.J[m];
  int64_t gstride_n = 1, sstride_n = 1;
  for (int m = p.order - 1; m > p.n; --m) {
    gstride_n *= p.J[m];
    sstride_n *= p.J[m];
  }
  const bool tab = rest <= kPairTab;
  if (tab) {
    for (int64_t t = threadIdx.x; t < rest; t += blockDim.x) {
      int64_t rem = t, gidx = 0, sidx = 0, gstride = 1, sstride = 1;
      for (int m = p.order - 1; m >= 0; --m) {
        const int64_t sdim = (m == p.n) ? p.In : p.J[m];
        if (m != p.n) {
          const int64_t c = rem % p.J[m];
          rem /= p.J[m];
          gidx += c * gstride;
          sidx += c * sstride;
        }
        gstride *= p.J[m];
        sstride *= sdim;
      }
      stab[t] = int(sidx);
      gtab[t] = int(gidx);
    }
    __syncthreads();
  }
  const int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (idx >= p.In * Jn) return;
  const int64_t i = idx / Jn, jn = idx % Jn;
  double acc = 0.0;
  if (tab) {
    const double* sp = p.S + i * sstride_n;
    const double* gp = p.G + jn * gstride_n;
#pragma unroll 4
    for (int64_t t = 0; t < rest; ++t) acc += sp[stab[t]] * gp[gtab[t]];
    p.out[idx] = acc;
    return;
  }
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
