// Streaming kernels of the contraction-only MU engine (CUDA-core path).
//
// Layout contract (reference include/ntf/tensor.hpp:20-82): the data tensor is
// row-major with the last mode contiguous.  We view it as `rows x K` where
// K = I_{N-1} and a "row" is one prefix multi-index (i_0..i_{N-2}); factors
// are row-major I_n x R fp64 masters.
//
// Kernels
//   recon_kernel     K2/K5: Xhat = sum_r H(row,r) A_last(k,r) computed in
//                    registers, fused with the beta weights (reference
//                    kernels.hpp:30-66) and the d_beta objective
//                    (divergence.cpp:16-44).  Writes P~/Q~ (J-CoMM reference
//                    cache, cp.cpp:202-208) or only the objective (loss
//                    lambdas cp.cpp:264,293).  Xhat itself is never stored.
//   contract_kernel  K3: the mode-n contraction of reference cp_contract
//                    (tensor.cpp:372-406) for one or two weight streams
//                    (Num from P, Den from Q), via the per-unit "G trick":
//                    G(k,r) = sum_{rows of unit} S(row,k) * M(row,r), with
//                    M the Hadamard product of the row-mode factors.
//                    target = last mode: Num(k,r) = sum_units G;
//                    target n < N-1 (units share i_n):
//                    Num(i_n,r) = sum_units sum_k F_last(k,r) G(k,r).
//                    Per entry that is R FMAs per stream, no cross-lane
//                    reduction in the inner loop, and no float atomics
//                    (per-unit partials + fixed-order fp64 second stage).
//   finalize_kernel  K4: fp64 reduction of the partials, beta = 1 closed-form
//                    denominator (cp.cpp:90-105), MU step (kernels.hpp:69-75),
//                    chi transforms for J-CoMM (divergence.cpp:57-80) and the
//                    staged T copy of the updated factor.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "device_math.cuh"

namespace ntfg {

// Division by a loop-invariant divisor via a multiply-high (round-up method):
// q = (n * m) >> (32 + l), m = floor(2^(32+l) / d) + 1, l = ceil(log2 d);
// exact for 0 <= n < 2^31 (Geom::small_rows guards larger indices).
struct FastDiv {
  uint64_t m = 1;
  int shift = 32;
  int64_t d = 1;
  void init(int64_t dv) {
    d = dv < 1 ? 1 : dv;
    int l = 0;
    while ((int64_t(1) << l) < d) ++l;
    const unsigned __int128 num = (unsigned __int128)1 << (32 + l);
    m = uint64_t(num / uint64_t(d)) + 1;
    shift = 32 + l;
  }
  __host__ __device__ int64_t div(int64_t n) const { return int64_t((uint64_t(n) * m) >> shift); }
};

struct Geom {
  int order;
  int64_t dims[kMaxOrder];
  int64_t K;                  // dims[order-1]
  int64_t rows;               // prod dims[0..order-2] (1 for order 1)
  int64_t rstride[kMaxOrder]; // row index decomposition for m < order-1
  FastDiv fs[kMaxOrder];      // division by rstride[m]
  FastDiv fd[kMaxOrder];      // division by dims[m]
  bool small_rows;            // rows < 2^31: FastDiv exact
  void init_fast() {
    small_rows = rows < (int64_t(1) << 31);
    for (int m = 0; m < order; ++m) {
      fs[m].init(rstride[m]);
      fd[m].init(dims[m]);
    }
  }
  __host__ __device__ int64_t coord(int64_t row, int m) const {
    if (small_rows) {
      const int64_t q = fs[m].div(row);
      return q - fd[m].div(q) * dims[m];
    }
    return (row / rstride[m]) % dims[m];
  }
};

constexpr int kRB = 8;  // rows per register block

template <typename T> struct Vec2;
template <> struct Vec2<float> { using type = float2; };
template <> struct Vec2<double> { using type = double2; };

// ---------------------------------------------------------------------------
// K2 / K5: reconstruction + weights (+ objective)

template <typename T>
struct ReconParams {
  Geom g;
  int R;
  const double* fac[kMaxOrder];  // model factors (fp64) for the prefix product H
  const double* htab;            // nullable: H(row, r) = htab[row * R + r] (Tucker partial chain)
  const T* alast;                // staged last factor, [K][RP] (zero padded)
  const float* hfac32;           // nullable: fp32 copy [I_f][R] of the fastest row mode's factor (recon_tc H producers)
  const T* x;
  T* pout;                       // nullable
  T* qout;                       // nullable
  T* xhout;                      // nullable: materialised Xhat (cp_reconstruct API only)
  void* planes[4];               // nullable: bf16 hi/lo planes of P and Q (tensor-core K3)
  double* obj;                   // per-CTA objective partial (nullable)
  unsigned* flags;               // domain flags (nullable)
  double beta, eps;
  int bk;
  int ktiles;
  int64_t work;                  // row_blocks * ktiles
};

// ---------------------------------------------------------------------------
// K3: contraction of one or two weight streams against the off-mode factors

template <typename T, int NS>
struct ContractParams {
  Geom g;
  int n;            // target mode
  int R, RP;        // rank and partial stride
  int r0;           // first rank of this chunk
  const T* src[NS];
  const double* mfac[NS][kMaxOrder];  // row-mode factors per stream (fp64)
  const double* lastfac[NS];          // last-mode factor per stream (case B epilogue)
  const double* mtab[NS];             // nullable: M(row, r) = mtab[s][row * R + r] (case A)
  int caseA;        // target == last mode
  int64_t units;
  int64_t S;        // case B: splits per target index
  int64_t An, Bn;   // case B: row = (j / Bn) * (I_n * Bn) + i_n * Bn + j % Bn
  FastDiv fB;       // division by Bn
  T* partA;         // case A: [NS][units][K][RP]
  double* partB;    // case B: [NS][I_n][S][RP]
  int ktiles;
};

// ---------------------------------------------------------------------------
// K4: fp64 second stage + MU step (+ chi transforms, staged copy)

template <typename T>
struct FinalizeParams {
  int caseA;
  int64_t In;
  int R, RP;
  int64_t units;         // case A partial count
  int64_t S;             // case B splits
  const T* partA;        // [NS][units][In][RP]
  const double* partAd;  // nullable: [NS][units][In][RP] chunk sums (reduce_units_kernel)
  const double* partB;   // [NS][In][S][RP]
  int den_closed;        // beta = 1 CP: den = colprod[r]
  const double* colprod; // [R]
  // split mode for data-parallel fits: phase 1 writes numden = [num | den]
  // ([2][In][R]) and returns; phase 2 reads numden (after the allreduce).
  int phase;             // 0 fused, 1 reduce only, 2 MU only
  double* numden;
  const double* anchor;  // [In][R]
  double* out;           // [In][R]
  const double* ref;     // J-CoMM reference block (nullable => no chi)
  double* chi1;
  double* chi2;
  T* stage;              // staged copy [In][RP] (nullable)
  double gamma, eps, beta;
  unsigned* flags;
};

template <typename T>
static __global__ void finalize_kernel(const FinalizeParams<T> p) {
  const int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (idx >= p.In * p.RP) return;
  const int64_t i = idx / p.RP;
  const int r = int(idx % p.RP);
  if (r >= p.R) {
    if (p.stage && p.phase != 1) p.stage[i * p.RP + r] = T(0);
    return;
  }
  double num = 0.0, den = 0.0;
  if (p.phase == 2) {
    num = p.numden[i * p.R + r];
    den = p.numden[(p.In + i) * p.R + r];
  } else if (p.caseA && p.partAd) {
    const int64_t sstride = p.units * p.In * p.RP;
    for (int64_t u = 0; u < p.units; ++u) {
      num += p.partAd[(u * p.In + i) * p.RP + r];
      if (!p.den_closed) den += p.partAd[sstride + (u * p.In + i) * p.RP + r];
    }
  } else if (p.caseA) {
    const int64_t sstride = p.units * p.In * p.RP;
    for (int64_t u = 0; u < p.units; ++u) {
      num += double(p.partA[(u * p.In + i) * p.RP + r]);
      if (!p.den_closed) den += double(p.partA[sstride + (u * p.In + i) * p.RP + r]);
    }
  } else {
    const int64_t sstride = p.In * p.S * p.RP;
    for (int64_t s = 0; s < p.S; ++s) {
      num += p.partB[(i * p.S + s) * p.RP + r];
      if (!p.den_closed) den += p.partB[sstride + (i * p.S + s) * p.RP + r];
    }
  }
  if (p.phase == 1) {
    p.numden[i * p.R + r] = num;
    p.numden[(p.In + i) * p.R + r] = den;
    return;
  }
  if (p.den_closed) den = p.colprod[r];
  const double v = mu_step(p.anchor[i * p.R + r], num, den, p.gamma, p.eps);
  p.out[i * p.R + r] = v;
  if (p.ref) {
    unsigned bad = 0;
    const double z = p.ref[i * p.R + r];
    p.chi1[i * p.R + r] = chi1_entry(v, z, p.beta, bad);
    p.chi2[i * p.R + r] = chi2_entry(v, z, p.beta, bad);
    if (bad && p.flags) atomicOr(p.flags, bad);
  }
  if (p.stage) p.stage[i * p.RP + r] = T(v);
}

// First stage of the case-A cross-unit reduction: out[s][c][i][r] = sum of
// units [c*per, (c+1)*per) of in[s][u][i][r] in fp64 (fixed order).
template <typename T>
static __global__ void reduce_units_kernel(const T* in, int64_t units, int64_t per, int64_t chunks,
                                           int64_t slice, int ns, double* out) {
  const int64_t total = int64_t(ns) * chunks * slice;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t e = idx % slice;
    const int64_t c = (idx / slice) % chunks;
    const int64_t s = idx / (slice * chunks);
    const int64_t u0 = c * per, u1 = u0 + per < units ? u0 + per : units;
    const T* src = in + (s * units) * slice + e;
    double acc = 0.0;
    for (int64_t u = u0; u < u1; ++u) acc += double(src[u * slice]);
    out[idx] = acc;
  }
}

// Column sums sum_i F_m(i, r) for every mode m != skip (reference
// ones_denominator, cp.cpp:90-105), one CTA per mode, fixed reduction tree.
// out: [order][R]; rows of the skipped mode are left untouched.
struct ColsumParams {
  int order, skip, R;
  int64_t rows[kMaxOrder];
  const double* fac[kMaxOrder];
  double* out;
  // fused closed-form denominator (nullable): the last block to finish writes
  // prod[r] = prod_{m != skip} out[m][r] (ascending m) and re-arms the counter
  double* prod;
  int* done;
};

// column sums of every factor but `skip`, one 1024-thread block per mode:
// thread t sums column t % RC over the rows i = g, g + G, ... (g = t / RC,
// G = 1024 / RC row groups, coalesced across r) into four interleaved
// partials (four loads in flight), then column r adds its G group sums in
// group order -- a fixed order, so results are reproducible (and identical
// on every rank of a sharded fit).
constexpr int kColsumThreads = 1024;
static __global__ void __launch_bounds__(kColsumThreads) colsum_kernel(const ColsumParams p) {
  __shared__ double red[kColsumThreads];
  const int m = blockIdx.x;
  if (m == p.skip) return;
  const int R = p.R, t = threadIdx.x;
  const int64_t rows = p.rows[m];
  for (int r0 = 0; r0 < R; r0 += kColsumThreads) {
    const int RC = R - r0 < kColsumThreads ? R - r0 : kColsumThreads;
    const int G = kColsumThreads / RC;
    const int r = r0 + t % RC, g = t / RC;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    if (g < G) {
      const double* f = p.fac[m] + r;
      int64_t i = g;
      for (; i + 3 * int64_t(G) < rows; i += 4 * int64_t(G)) {
        s0 += f[i * R];
        s1 += f[(i + G) * R];
        s2 += f[(i + 2 * G) * R];
        s3 += f[(i + 3 * G) * R];
      }
      for (; i < rows; i += G) s0 += f[i * R];
    }
    red[t] = (s0 + s1) + (s2 + s3);
    __syncthreads();
    if (t < RC) {
      double tot = 0.0;
      for (int q = 0; q < G; ++q) tot += red[q * RC + t];
      p.out[m * R + r0 + t] = tot;
    }
    __syncthreads();
  }
  if (p.prod) {
    // one launch instead of two per beta = 1 block update: the block that
    // completes the set of column sums forms the product (fixed order, from the
    // values every block published before its arrival)
    __shared__ int last;
    __threadfence();
    __syncthreads();
    if (t == 0) {
      const int parts = p.order - ((p.skip >= 0 && p.skip < p.order) ? 1 : 0);
      last = atomicAdd(p.done, 1) == parts - 1;
    }
    __syncthreads();
    if (last) {
      __threadfence();
      for (int r = t; r < R; r += kColsumThreads) {
        double prod = 1.0;
        for (int mm = 0; mm < p.order; ++mm)
          if (mm != p.skip) prod *= __ldcg(p.out + mm * R + r);
        p.prod[r] = prod;
      }
      if (t == 0) *p.done = 0;
    }
  }
}

// colprod[r] = prod_{m != skip} colsum[m][r] (ascending m, as cp.cpp:93-100)
static __global__ void colprod_kernel(const double* colsum, int order, int skip, int R, double* out) {
  const int r = threadIdx.x + blockIdx.x * blockDim.x;
  if (r >= R) return;
  double prod = 1.0;
  for (int m = 0; m < order; ++m)
    if (m != skip) prod *= colsum[m * R + r];
  out[r] = prod;
}

// objective partials -> loss array slot losses[*counter] (fixed order);
// with raw != nullptr only the unnormalised sum is written (data-parallel
// fits allreduce it before normalising with objective_scale_kernel).
static __global__ void objective_finalize_kernel(const double* partials, int n, double inv_entries,
                                          double* losses, int* counter, double* raw,
                                          const double* xconst = nullptr) {
  __shared__ double red[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += partials[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (int(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double tot = xconst ? red[0] + *xconst : red[0];
    if (raw) {
      *raw = tot;
    } else {
      const int c = *counter;
      losses[c] = tot * inv_entries;
      *counter = c + 1;
    }
  }
}

// x-only part of d_beta summed over the data tensor (fp64, fixed grid ->
// deterministic): sum x^b / (b (b-1)), for the tensor-core recon's split
// objective (stream3_kernels.cuh, tc_weights).  Two stages: per-CTA partials
// then one CTA.
// x^beta of one data entry: fp32 data with beta = 0.5 / 1.5 uses the
// correctly rounded sqrtf (unbiased, ~6e-8 relative; the fp64 pow is ~40 fp64
// instructions per entry and made this pass compute-bound)
template <typename T>
__device__ __forceinline__ double xpow_term(T x, double beta) {
  if constexpr (sizeof(T) == 4) {
    if (beta == 0.5) return double(sqrtf(x));
    if (beta == 1.5) return double(x) * double(sqrtf(x));
  }
  return fpow64(double(x), beta);
}
template <typename T>
static __global__ void xconst_kernel(const T* x, int64_t n, double beta, double* partials) {
  __shared__ double red[256];
  double s = 0.0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t i0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if constexpr (sizeof(T) == 4) {
    // four entries per load and four independent fp64 partials (the single
    // DADD chain made this pass latency-bound); fixed order -> deterministic
    if ((reinterpret_cast<uintptr_t>(x) & 15) == 0) {
      const int64_t n4 = n / 4;
      double s1 = 0.0, s2 = 0.0, s3 = 0.0;
      for (int64_t i = i0; i < n4; i += stride) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(x) + i);
        s += xpow_term(v.x, beta);
        s1 += xpow_term(v.y, beta);
        s2 += xpow_term(v.z, beta);
        s3 += xpow_term(v.w, beta);
      }
      s = (s + s1) + (s2 + s3);
      i0 += n4 * 4;
    }
  }
  for (int64_t i = i0; i < n; i += stride) s += xpow_term(x[i], beta);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (int(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = red[0];
}

static __global__ void xconst_finish_kernel(double* partials, int n, double scale, double* out) {
  __shared__ double red[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += partials[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (int(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0] * scale;
}

static __global__ void objective_scale_kernel(const double* raw, double inv_entries, double* losses,
                                       int* counter) {
  const int c = *counter;
  losses[c] = *raw * inv_entries;
  *counter = c + 1;
}

// fp64 factor -> staged T copy [I][RP] (zero padded)
template <typename T>
static __global__ void stage_kernel(const double* src, int64_t rows, int R, int RP, T* dst) {
  const int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (idx >= rows * RP) return;
  const int64_t i = idx / RP;
  const int r = int(idx % RP);
  dst[idx] = r < R ? T(src[i * R + r]) : T(0);
}

// data tensor conversion S -> T
template <typename T, typename S>
static __global__ void convert_kernel(const S* src, int64_t n, T* dst) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = T(src[i]);
}

// chi1 / chi2 of every entry of the concatenated factor blocks (step-level API)
static __global__ void chi_all_kernel(const double* z, const double* zref, int64_t n, double beta,
                               double* c1, double* c2, unsigned* flags) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  unsigned bad = 0;
  c1[i] = chi1_entry(z[i], zref[i], beta, bad);
  c2[i] = chi2_entry(z[i], zref[i], beta, bad);
  if (bad) atomicOr(flags, bad);
}

// ---- BMMe extrapolation (reference cp.cpp:137-198, tucker.cpp:151-217) ----
// alpha = min(alpha_nes[it], cap / (||[cur - prev]_+||_F + delta)); it = (*iter)++
// The squared norm is split into the entries of the sharded range [s0, s1)
// (the mode-0 factor rows this rank owns in a data-parallel fit) and the
// replicated rest, so a sharded fit allreduces part[0] before finishing and
// every rank computes the same alpha over the WHOLE model (cp.cpp:178-194).
static __global__ void extrap_norm_kernel(const double* cur, const double* prev, int64_t n, int64_t s0,
                                          int64_t s1, double* part) {
  __shared__ double red[2][256];
  double a = 0.0, b = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = cur[i] - prev[i];
    if (d > 0.0) {
      if (i >= s0 && i < s1) a += d * d;
      else b += d * d;
    }
  }
  red[0][threadIdx.x] = a;
  red[1][threadIdx.x] = b;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (int(threadIdx.x) < w) {
      red[0][threadIdx.x] += red[0][threadIdx.x + w];
      red[1][threadIdx.x] += red[1][threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[0] = red[0][0];
    part[1] = red[1][0];
  }
}

static __global__ void extrap_alpha_finish_kernel(const double* part, const double* alpha_nes, int* iter,
                                                  double cap, double delta, double* alpha_out) {
  const int it = *iter;
  const double a = cap / (sqrt(part[0] + part[1]) + delta);
  const double an = alpha_nes[it];
  *alpha_out = an < a ? an : a;  // std::min(alpha_nes, cap / (...))
  *iter = it + 1;
}

// out = max(cur + alpha [cur - prev]_+, eps)
static __global__ void extrap_apply_kernel(const double* cur, const double* prev, int64_t n,
                                    const double* alpha, double eps, double* out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double d = cur[i] - prev[i];
  const double v = cur[i] + *alpha * (d > 0.0 ? d : 0.0);
  out[i] = v < eps ? eps : v;
}

// D_beta over explicit arrays: per-CTA partials (divergence.cpp:35-40)
static __global__ void dbeta_sum_kernel(const double* x, const double* y, int64_t n, int bk, double beta,
                                 double* partials, unsigned* flags) {
  __shared__ double red[256];
  unsigned bad = 0;
  double s = 0.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    s += dbeta_entry(x[i], y[i], bk, beta, bad);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (int(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = red[0];
  if (bad) atomicOr(flags, bad);
}

}  // namespace ntfg
