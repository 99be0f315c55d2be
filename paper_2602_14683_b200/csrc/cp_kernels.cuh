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

struct Geom {
  int order;
  int64_t dims[kMaxOrder];
  int64_t K;                  // dims[order-1]
  int64_t rows;               // prod dims[0..order-2] (1 for order 1)
  int64_t rstride[kMaxOrder]; // row index decomposition for m < order-1
  __host__ __device__ int64_t coord(int64_t row, int m) const {
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
  const T* x;
  T* pout;                       // nullable
  T* qout;                       // nullable
  T* xhout;                      // nullable: materialised Xhat (cp_reconstruct API only)
  double* obj;                   // per-CTA objective partial (nullable)
  unsigned* flags;               // domain flags (nullable)
  double beta, eps;
  int bk;
  int ktiles;
  int64_t work;                  // row_blocks * ktiles
};

template <typename T, int RP, int KT>
__global__ void __launch_bounds__(256) recon_kernel(const ReconParams<T> p) {
  __shared__ __align__(16) T hs[8][kRB][RP];  // one H block per warp
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t K = p.g.K;
  const int nprefix = p.g.order - 1;
  const int64_t tile_w = int64_t(blockDim.x) * KT;
  double obj = 0.0;
  unsigned bad = 0;

  for (int64_t w = blockIdx.x; w < p.work; w += gridDim.x) {
    const int kt = int(w % p.ktiles);
    const int64_t rb = w / p.ktiles;
    const int64_t row0 = rb * kRB;
    const int64_t k0 = kt * tile_w + int64_t(threadIdx.x) * KT;

    // issue the data loads of this row block first (latency overlaps H)
    T xv[kRB][KT];
#pragma unroll
    for (int rr = 0; rr < kRB; ++rr) {
      const int64_t row = row0 + rr;
#pragma unroll
      for (int kk = 0; kk < KT; ++kk) {
        const int64_t k = k0 + kk;
        xv[rr][kk] = (row < p.g.rows && k < K) ? __ldg(p.x + row * K + k) : T(0);
      }
    }
    // last-factor rows of this thread's k (registers)
    T a[KT][RP];
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) {
      const int64_t k = k0 + kk;
#pragma unroll
      for (int r = 0; r < RP; ++r) a[kk][r] = (k < K) ? __ldg(p.alast + k * RP + r) : T(0);
    }
    // warp-local H block: H(row, r) = prod_{m < N-1} A_m(i_m, r)
    __syncwarp();
    for (int idx = lane; idx < kRB * RP; idx += 32) {
      const int rr = idx / RP, r = idx % RP;
      const int64_t row = row0 + rr;
      double h = 0.0;
      if (r < p.R && row < p.g.rows) {
        if (p.htab) {
          h = p.htab[row * p.R + r];
        } else {
          h = 1.0;
          for (int m = 0; m < nprefix; ++m) h *= p.fac[m][p.g.coord(row, m) * p.R + r];
        }
      }
      hs[warp][rr][r] = T(h);
    }
    __syncwarp();

#pragma unroll
    for (int rr = 0; rr < kRB; ++rr) {
      const int64_t row = row0 + rr;
      T xh[KT];
#pragma unroll
      for (int kk = 0; kk < KT; ++kk) xh[kk] = T(0);
#pragma unroll
      for (int r = 0; r < RP; ++r) {
        const T h = hs[warp][rr][r];
#pragma unroll
        for (int kk = 0; kk < KT; ++kk) xh[kk] = fma(h, a[kk][r], xh[kk]);
      }
      if (row >= p.g.rows) continue;
#pragma unroll
      for (int kk = 0; kk < KT; ++kk) {
        const int64_t k = k0 + kk;
        if (k >= K) continue;
        if (p.xhout) p.xhout[row * K + k] = xh[kk];
        if (p.pout) {
          T pw, qw;
          weights_entry(xv[rr][kk], xh[kk], p.bk, p.beta, p.eps, pw, qw);
          p.pout[row * K + k] = pw;
          if (p.qout) p.qout[row * K + k] = qw;
        }
        if (p.obj) obj += dbeta_entry(double(xv[rr][kk]), double(xh[kk]), p.bk, p.beta, bad);
      }
    }
  }

  if (p.obj) {
    __shared__ double red[8];
    obj = warp_sum(obj);
    if (lane == 0) red[warp] = obj;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int i = 0; i < int(blockDim.x >> 5); ++i) s += red[i];
      p.obj[blockIdx.x] = s;
    }
  }
  if (bad && p.flags) atomicOr(p.flags, bad);
}

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
  T* partA;         // case A: [NS][units][K][RP]
  double* partB;    // case B: [NS][I_n][S][RP]
  int ktiles;
};

template <typename T, int RC, int KT, int NS>
__global__ void __launch_bounds__(NS * 128) contract_kernel(const ContractParams<T, NS> p) {
  constexpr int TPS = 128;              // threads per stream
  constexpr int WPS = TPS / 32;         // warps per stream
  __shared__ __align__(16) T ms[NS * WPS][kRB][RC];
  __shared__ double wsum[NS][WPS][RC];
  __shared__ double usum[NS][RC];

  const int s = threadIdx.x / TPS;
  const int t = threadIdx.x % TPS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wis = t >> 5;               // warp index within stream
  const int64_t K = p.g.K;
  const int nrow_modes = p.g.order - 1;
  const T* __restrict__ src = p.src[s];
  const int64_t In = p.g.dims[p.n];

  for (int64_t u = blockIdx.x; u < p.units; u += gridDim.x) {
    // unit -> row range (j0, j1) and target index
    int64_t j0, j1, itgt = 0, split = 0;
    if (p.caseA) {
      j0 = u * p.g.rows / p.units;
      j1 = (u + 1) * p.g.rows / p.units;
    } else {
      itgt = u / p.S;
      split = u % p.S;
      const int64_t tot = p.An * p.Bn;
      j0 = split * tot / p.S;
      j1 = (split + 1) * tot / p.S;
    }
    if (!p.caseA) {
      if (threadIdx.x < NS * RC) usum[threadIdx.x / RC][threadIdx.x % RC] = 0.0;
    }

    for (int kt = 0; kt < p.ktiles; ++kt) {
      const int64_t k0 = int64_t(kt) * TPS * KT + int64_t(t) * KT;
      T gacc[KT][RC];
#pragma unroll
      for (int kk = 0; kk < KT; ++kk)
#pragma unroll
        for (int r = 0; r < RC; ++r) gacc[kk][r] = T(0);

      for (int64_t jb = j0; jb < j1; jb += kRB) {
        // data loads for this block of rows
        T sv[kRB][KT];
#pragma unroll
        for (int rr = 0; rr < kRB; ++rr) {
          const int64_t j = jb + rr;
          int64_t row = j;
          if (!p.caseA) row = (j / p.Bn) * (In * p.Bn) + itgt * p.Bn + (j % p.Bn);
#pragma unroll
          for (int kk = 0; kk < KT; ++kk) {
            const int64_t k = k0 + kk;
            sv[rr][kk] = (j < j1 && k < K) ? __ldg(src + row * K + k) : T(0);
          }
        }
        // warp-local M block
        __syncwarp();
        for (int idx = lane; idx < kRB * RC; idx += 32) {
          const int rr = idx / RC, r = idx % RC;
          const int64_t j = jb + rr;
          double mval = 0.0;
          if (j < j1 && p.r0 + r < p.R) {
            int64_t row = j;
            if (!p.caseA) row = (j / p.Bn) * (In * p.Bn) + itgt * p.Bn + (j % p.Bn);
            if (p.mtab[s]) {
              mval = p.mtab[s][row * p.R + p.r0 + r];
            } else {
              mval = 1.0;
              for (int m = 0; m < nrow_modes; ++m) {
                if (m == p.n) continue;
                mval *= p.mfac[s][m][p.g.coord(row, m) * p.R + p.r0 + r];
              }
            }
          }
          ms[warp][rr][r] = T(mval);
        }
        __syncwarp();
#pragma unroll
        for (int rr = 0; rr < kRB; ++rr) {
#pragma unroll
          for (int r = 0; r < RC; ++r) {
            const T mv = ms[warp][rr][r];
#pragma unroll
            for (int kk = 0; kk < KT; ++kk) gacc[kk][r] = fma(sv[rr][kk], mv, gacc[kk][r]);
          }
        }
      }

      if (p.caseA) {
#pragma unroll
        for (int kk = 0; kk < KT; ++kk) {
          const int64_t k = k0 + kk;
          if (k >= K) continue;
          T* dst = p.partA + ((int64_t(s) * p.units + u) * K + k) * p.RP + p.r0;
#pragma unroll
          for (int r = 0; r < RC; ++r)
            if (p.r0 + r < p.R) dst[r] = gacc[kk][r];
        }
      } else {
        // contract G with the last-mode factor: sum_k F(k, r) G(k, r)
#pragma unroll
        for (int r = 0; r < RC; ++r) {
          double v = 0.0;
          if (p.r0 + r < p.R) {
#pragma unroll
            for (int kk = 0; kk < KT; ++kk) {
              const int64_t k = k0 + kk;
              if (k < K) v += double(gacc[kk][r]) * p.lastfac[s][k * p.R + p.r0 + r];
            }
          }
          v = warp_sum(v);
          if (lane == 0) wsum[s][wis][r] = v;
        }
        __syncthreads();
        if (threadIdx.x < NS * RC) {
          const int ss = threadIdx.x / RC, r = threadIdx.x % RC;
          double acc = usum[ss][r];
          for (int w = 0; w < WPS; ++w) acc += wsum[ss][w][r];
          usum[ss][r] = acc;
        }
        __syncthreads();
      }
    }
    if (!p.caseA) {
      if (threadIdx.x < NS * RC) {
        const int ss = threadIdx.x / RC, r = threadIdx.x % RC;
        if (p.r0 + r < p.R)
          p.partB[((int64_t(ss) * In + itgt) * p.S + split) * p.RP + p.r0 + r] = usum[ss][r];
      }
      __syncthreads();
    }
  }
}

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
__global__ void finalize_kernel(const FinalizeParams<T> p) {
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

// Column sums sum_i F_m(i, r) for every mode m != skip (reference
// ones_denominator, cp.cpp:90-105), one CTA per mode, fixed reduction tree.
// out: [order][R]; rows of the skipped mode are left untouched.
struct ColsumParams {
  int order, skip, R;
  int64_t rows[kMaxOrder];
  const double* fac[kMaxOrder];
  double* out;
};

__global__ void colsum_kernel(const ColsumParams p) {
  __shared__ double red[256];
  const int m = blockIdx.x;
  if (m == p.skip) return;
  for (int r = 0; r < p.R; ++r) {
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < p.rows[m]; i += blockDim.x) s += p.fac[m][i * p.R + r];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
      if (int(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) p.out[m * p.R + r] = red[0];
    __syncthreads();
  }
}

// colprod[r] = prod_{m != skip} colsum[m][r] (ascending m, as cp.cpp:93-100)
__global__ void colprod_kernel(const double* colsum, int order, int skip, int R, double* out) {
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
__global__ void objective_finalize_kernel(const double* partials, int n, double inv_entries,
                                          double* losses, int* counter, double* raw) {
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
    if (raw) {
      *raw = red[0];
    } else {
      const int c = *counter;
      losses[c] = red[0] * inv_entries;
      *counter = c + 1;
    }
  }
}

__global__ void objective_scale_kernel(const double* raw, double inv_entries, double* losses,
                                       int* counter) {
  const int c = *counter;
  losses[c] = *raw * inv_entries;
  *counter = c + 1;
}

// fp64 factor -> staged T copy [I][RP] (zero padded)
template <typename T>
__global__ void stage_kernel(const double* src, int64_t rows, int R, int RP, T* dst) {
  const int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (idx >= rows * RP) return;
  const int64_t i = idx / RP;
  const int r = int(idx % RP);
  dst[idx] = r < R ? T(src[i * R + r]) : T(0);
}

// data tensor conversion S -> T
template <typename T, typename S>
__global__ void convert_kernel(const S* src, int64_t n, T* dst) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = T(src[i]);
}

// chi1 / chi2 of every entry of the concatenated factor blocks (step-level API)
__global__ void chi_all_kernel(const double* z, const double* zref, int64_t n, double beta,
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
__global__ void extrap_alpha_kernel(const double* cur, const double* prev, int64_t n,
                                    const double* alpha_nes, int* iter, double cap, double delta,
                                    double* alpha_out) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = cur[i] - prev[i];
    if (d > 0.0) s += d * d;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (int(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int it = *iter;
    const double a = cap / (sqrt(red[0]) + delta);
    const double an = alpha_nes[it];
    *alpha_out = an < a ? an : a;  // std::min(alpha_nes, cap / (...))
    *iter = it + 1;
  }
}

// out = max(cur + alpha [cur - prev]_+, eps)
__global__ void extrap_apply_kernel(const double* cur, const double* prev, int64_t n,
                                    const double* alpha, double eps, double* out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double d = cur[i] - prev[i];
  const double v = cur[i] + *alpha * (d > 0.0 ? d : 0.0);
  out[i] = v < eps ? eps : v;
}

// D_beta over explicit arrays: per-CTA partials (divergence.cpp:35-40)
__global__ void dbeta_sum_kernel(const double* x, const double* y, int64_t n, int bk, double beta,
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
