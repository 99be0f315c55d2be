// Streaming passes, pipelined version (CUDA cores).
//
// Both kernels stream `rows x K` row-major data (X, P~ or Q~) with every
// thread owning KT consecutive columns k, so each thread's data never leaves
// its own registers / smem slots: stage s of the ring holds kRows rows and
// is filled with per-thread cp.async (LDGSTS) copies issued kDepth stages
// ahead.  The per-row vectors (H for the reconstruction, M = Hadamard product
// of the off-mode factor rows for the contraction) are computed
// cooperatively once per stage in fp64, rounded to T, and shared through
// smem; one named barrier per stage (per stream) orders them.
//
//   recon2    X^(row,k) = sum_r H(row,r) A_last(k,r), A_last in registers,
//             fused weights (kernels.hpp:30-66) and d_beta objective.
//   contract2 G(k,r) += S(row,k) M(row,r) with packed FFMA2 (fp32) on the
//             thread's two columns; per-unit epilogue as in cp_kernels.cuh.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "cp_kernels.cuh"

namespace ntfg {

constexpr int kRows = 8;    // rows per stage
constexpr int kDepth = 3;   // stages in flight

template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int src_size = valid ? BYTES : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(s), "l"(gmem), "n"(BYTES),
               "r"(src_size));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
__device__ __forceinline__ void named_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(threads));
}

template <typename T, int KT> struct Pack;
template <> struct Pack<float, 2> { using type = float2; };
template <> struct Pack<float, 1> { using type = float; };
template <> struct Pack<double, 1> { using type = double; };

// fp32 objective term, accumulated in fp64 by the caller (fp32 build only;
// accuracy ~1e-6 relative per entry).
__device__ __forceinline__ float dbeta_f32(float x, float y, int bk, float b, unsigned& bad) {
  if (!(y > 0.f)) { bad |= 1u; return 0.f; }
  if (x < 0.f) { bad |= 2u; return 0.f; }
  if (bk == kBeta1) return (x > 0.f ? x * __logf(__fdividef(x, y)) : 0.f) - x + y;
  if (bk == kBeta0) {
    if (x == 0.f) return __int_as_float(0x7f800000);
    const float r = __fdividef(x, y);
    return r - __logf(r) - 1.f;
  }
  if (bk == kBetaHalf) {  // (x^.5 - .5 y^.5 - .5 x y^-.5) / (-.25)
    const float ry = rsqrtf(y);
    const float sx = sqrtf(x), sy = y * ry;
    return (sx - 0.5f * sy - 0.5f * x * ry) * -4.f;
  }
  if (bk == kBeta3Half) {  // (x^1.5 + .5 y^1.5 - 1.5 x y^.5) / .75
    const float sy = sqrtf(y), sx = sqrtf(x);
    return (x * sx + 0.5f * y * sy - 1.5f * x * sy) * (1.f / 0.75f);
  }
  const float ly = __log2f(y);
  const float yb = exp2f(b * ly), yb1 = exp2f((b - 1.f) * ly);
  const float xb = x > 0.f ? exp2f(b * __log2f(x)) : 0.f;
  return (xb + (b - 1.f) * yb - b * x * yb1) / (b * (b - 1.f));
}

template <typename T>
__device__ __forceinline__ double objective_term(T x, T y, int bk, double beta, unsigned& bad);
template <>
__device__ __forceinline__ double objective_term<double>(double x, double y, int bk, double beta,
                                                         unsigned& bad) {
  return dbeta_entry(x, y, bk, beta, bad);
}
template <>
__device__ __forceinline__ double objective_term<float>(float x, float y, int bk, double beta,
                                                        unsigned& bad) {
  return double(dbeta_f32(x, y, bk, float(beta), bad));
}

// ---------------------------------------------------------------------------
// K2 / K5

template <typename T, int RP, int KT, int TPB>
static __global__ void __launch_bounds__(TPB) recon2_kernel(const ReconParams<T> p) {
  using V = typename Pack<T, KT>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // dynamic smem: X ring [kDepth][kRows][TPB*KT] T
  T (*xs)[kRows][TPB * KT] = reinterpret_cast<T (*)[kRows][TPB * KT]>(smem_raw);
  __shared__ __align__(16) T hs[2][kRows][RP];
  __shared__ double red[TPB / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t K = p.g.K;
  const int nprefix = p.g.order - 1;
  const int kt = int(blockIdx.x % p.ktiles);
  const int64_t rb_stride = gridDim.x / p.ktiles;
  const int64_t row_blocks = (p.g.rows + kRows - 1) / kRows;
  const int64_t k0 = int64_t(kt) * TPB * KT + int64_t(tid) * KT;
  const bool kvalid = k0 < K;  // KT columns valid together (K % KT == 0 enforced by host)

  T a[KT][RP];
#pragma unroll
  for (int kk = 0; kk < KT; ++kk)
#pragma unroll
    for (int r = 0; r < RP; ++r) a[kk][r] = kvalid ? __ldg(p.alast + (k0 + kk) * RP + r) : T(0);

  auto issue = [&](int64_t rb, int slot) {
#pragma unroll
    for (int rr = 0; rr < kRows; ++rr) {
      const int64_t row = rb * kRows + rr;
      const bool v = kvalid && rb < row_blocks && row < p.g.rows;
      const T* src = p.x + (v ? row * K + k0 : 0);
      cp_async<sizeof(T) * KT>(&xs[slot][rr][tid * KT], src, v);
    }
  };
  auto make_h = [&](int64_t rb, int slot) {
    for (int idx = tid; idx < kRows * RP; idx += TPB) {
      const int rr = idx / RP, r = idx % RP;
      const int64_t row = rb * kRows + rr;
      double h = 0.0;
      if (r < p.R && row < p.g.rows && rb < row_blocks) {
        if (p.htab) {
          h = p.htab[row * p.R + r];
        } else {
          h = 1.0;
          for (int m = 0; m < nprefix; ++m) h *= p.fac[m][p.g.coord(row, m) * p.R + r];
        }
      }
      hs[slot][rr][r] = T(h);
    }
  };

  double obj = 0.0;
  unsigned bad = 0;
  int64_t rb = blockIdx.x / p.ktiles;
  // prologue: stages 0..kDepth-2 in flight, H of the first block
#pragma unroll
  for (int d = 0; d < kDepth - 1; ++d) {
    issue(rb + d * rb_stride, d);
    cp_async_commit();
  }
  make_h(rb, 0);
  int it = 0;
  for (; rb < row_blocks; rb += rb_stride, ++it) {
    const int slot = it % kDepth;
    issue(rb + (kDepth - 1) * rb_stride, (it + kDepth - 1) % kDepth);
    cp_async_commit();
    cp_async_wait<kDepth - 1>();
    __syncthreads();  // H(slot) visible; previous H buffer free
    make_h(rb + rb_stride, (it + 1) & 1);
#pragma unroll
    for (int rr = 0; rr < kRows; ++rr) {
      const int64_t row = rb * kRows + rr;
      T xh[KT];
#pragma unroll
      for (int kk = 0; kk < KT; ++kk) xh[kk] = T(0);
#pragma unroll
      for (int r = 0; r < RP; ++r) {
        const T h = hs[it & 1][rr][r];
#pragma unroll
        for (int kk = 0; kk < KT; ++kk) xh[kk] = fma(h, a[kk][r], xh[kk]);
      }
      if (row >= p.g.rows || !kvalid) continue;
      const V xv = *reinterpret_cast<const V*>(&xs[slot][rr][tid * KT]);
      const T* xp = reinterpret_cast<const T*>(&xv);
      T pw[KT], qw[KT];
#pragma unroll
      for (int kk = 0; kk < KT; ++kk) {
        if (p.xhout) p.xhout[row * K + k0 + kk] = xh[kk];
        if (p.pout) weights_entry(xp[kk], xh[kk], p.bk, p.beta, p.eps, pw[kk], qw[kk]);
        if (p.obj) obj += objective_term<T>(xp[kk], xh[kk], p.bk, p.beta, bad);
      }
      if (p.pout) {
        *reinterpret_cast<V*>(p.pout + row * K + k0) = *reinterpret_cast<const V*>(pw);
        if (p.qout) *reinterpret_cast<V*>(p.qout + row * K + k0) = *reinterpret_cast<const V*>(qw);
      }
    }
  }
  cp_async_wait<0>();
  if (p.obj) {
    obj = warp_sum(obj);
    if (lane == 0) red[warp] = obj;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int i = 0; i < TPB / 32; ++i) s += red[i];
      p.obj[blockIdx.x] = s;
    }
  }
  if (bad && p.flags) atomicOr(p.flags, bad);
}

// ---------------------------------------------------------------------------
// K3

template <typename T, int RC, int KT, int NS, int TPS>
static __global__ void __launch_bounds__(NS * TPS) contract2_kernel(const ContractParams<T, NS> p) {
  using V = typename Pack<T, KT>::type;
  constexpr int WPS = TPS / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // layout: S ring [NS][kDepth][kRows][TPS*KT] T | M [NS][2][kRows][RC] T | wsum [NS][WPS][RC] double
  T* ring = reinterpret_cast<T*>(smem_raw);
  T* mbuf = ring + size_t(NS) * kDepth * kRows * TPS * KT;
  double* wsum = reinterpret_cast<double*>(mbuf + size_t(NS) * 2 * kRows * RC);
  __shared__ double usum[NS][RC];

  const int s = threadIdx.x / TPS;
  const int t = threadIdx.x % TPS;
  const int lane = threadIdx.x & 31;
  const int wis = t >> 5;
  const int64_t K = p.g.K;
  const int nrow_modes = p.g.order - 1;
  const T* __restrict__ src = p.src[s];
  const int64_t In = p.g.dims[p.n];
  T* myring = ring + size_t(s) * kDepth * kRows * TPS * KT;
  T* mym = mbuf + size_t(s) * 2 * kRows * RC;
  const int bar = 1 + s;  // named barrier per stream (0 is __syncthreads)

  for (int64_t u = blockIdx.x; u < p.units; u += gridDim.x) {
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
    const int64_t nblk = (j1 - j0 + kRows - 1) / kRows;
    auto row_of = [&](int64_t j) -> int64_t {
      if (p.caseA) return j;
      const int64_t aa = p.g.small_rows ? p.fB.div(j) : j / p.Bn;
      return aa * (In * p.Bn) + itgt * p.Bn + (j - aa * p.Bn);
    };
    if (!p.caseA && t < RC) usum[s][t] = 0.0;

    for (int kt = 0; kt < p.ktiles; ++kt) {
      const int64_t k0 = int64_t(kt) * TPS * KT + int64_t(t) * KT;
      const bool kvalid = k0 < K;
      auto issue = [&](int64_t b, int slot) {
#pragma unroll
        for (int rr = 0; rr < kRows; ++rr) {
          const int64_t j = j0 + b * kRows + rr;
          const bool v = kvalid && b < nblk && j < j1;
          const T* g = src + (v ? row_of(j) * K + k0 : 0);
          cp_async<sizeof(T) * KT>(myring + (size_t(slot) * kRows + rr) * TPS * KT + t * KT, g, v);
        }
      };
      auto make_m = [&](int64_t b, int slot) {
        for (int idx = t; idx < kRows * RC; idx += TPS) {
          const int rr = idx / RC, r = idx % RC;
          const int64_t j = j0 + b * kRows + rr;
          double mval = 0.0;
          if (b < nblk && j < j1 && p.r0 + r < p.R) {
            const int64_t row = row_of(j);
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
          mym[(size_t(slot) * kRows + rr) * RC + r] = T(mval);
        }
      };

      V g[RC];
#pragma unroll
      for (int r = 0; r < RC; ++r) g[r] = V{};
#pragma unroll
      for (int d = 0; d < kDepth - 1; ++d) {
        issue(d, d);
        cp_async_commit();
      }
      named_sync(bar, TPS);  // previous unit / k-tile done with M buffers
      make_m(0, 0);
      for (int64_t b = 0; b < nblk; ++b) {
        const int slot = int(b % kDepth);
        issue(b + kDepth - 1, int((b + kDepth - 1) % kDepth));
        cp_async_commit();
        cp_async_wait<kDepth - 1>();
        named_sync(bar, TPS);
        make_m(b + 1, int((b + 1) & 1));
        const T* mrow = mym + size_t(b & 1) * kRows * RC;
        const T* srow = myring + size_t(slot) * kRows * TPS * KT + t * KT;
#pragma unroll
        for (int rr = 0; rr < kRows; ++rr) {
          const V sv = *reinterpret_cast<const V*>(srow + rr * TPS * KT);
#pragma unroll
          for (int r = 0; r < RC; r += 4) {
            if constexpr (sizeof(T) == 4) {
              const float4 m4 = *reinterpret_cast<const float4*>(mrow + rr * RC + r);
              if constexpr (KT == 2) {
                g[r + 0] = __ffma2_rn(sv, make_float2(m4.x, m4.x), g[r + 0]);
                g[r + 1] = __ffma2_rn(sv, make_float2(m4.y, m4.y), g[r + 1]);
                g[r + 2] = __ffma2_rn(sv, make_float2(m4.z, m4.z), g[r + 2]);
                g[r + 3] = __ffma2_rn(sv, make_float2(m4.w, m4.w), g[r + 3]);
              } else {
                g[r + 0] = fmaf(sv, m4.x, g[r + 0]);
                g[r + 1] = fmaf(sv, m4.y, g[r + 1]);
                g[r + 2] = fmaf(sv, m4.z, g[r + 2]);
                g[r + 3] = fmaf(sv, m4.w, g[r + 3]);
              }
            } else {
              const double2 m0 = *reinterpret_cast<const double2*>(mrow + rr * RC + r);
              const double2 m1 = *reinterpret_cast<const double2*>(mrow + rr * RC + r + 2);
              g[r + 0] = fma(sv, m0.x, g[r + 0]);
              g[r + 1] = fma(sv, m0.y, g[r + 1]);
              g[r + 2] = fma(sv, m1.x, g[r + 2]);
              g[r + 3] = fma(sv, m1.y, g[r + 3]);
            }
          }
        }
      }
      cp_async_wait<0>();

      const T* gp = reinterpret_cast<const T*>(g);  // gp[r * KT + kk] = G(k0 + kk, r)
      if (p.caseA) {
        if (kvalid) {
#pragma unroll
          for (int kk = 0; kk < KT; ++kk) {
            T* dst = p.partA + ((int64_t(s) * p.units + u) * K + k0 + kk) * p.RP + p.r0;
#pragma unroll
            for (int r = 0; r < RC; ++r)
              if (p.r0 + r < p.R) dst[r] = gp[r * KT + kk];
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < RC; ++r) {
          double v = 0.0;
          if (kvalid && p.r0 + r < p.R) {
#pragma unroll
            for (int kk = 0; kk < KT; ++kk)
              v += double(gp[r * KT + kk]) * p.lastfac[s][(k0 + kk) * p.R + p.r0 + r];
          }
          v = warp_sum(v);
          if (lane == 0) wsum[(s * WPS + wis) * RC + r] = v;
        }
        named_sync(bar, TPS);
        if (t < RC) {
          double acc = usum[s][t];
          for (int w = 0; w < WPS; ++w) acc += wsum[(s * WPS + w) * RC + t];
          usum[s][t] = acc;
        }
      }
    }
    if (!p.caseA) {
      named_sync(bar, TPS);
      if (t < RC && p.r0 + t < p.R)
        p.partB[((int64_t(s) * In + itgt) * p.S + split) * p.RP + p.r0 + t] = usum[s][t];
    }
  }
}

template <typename T, int KT, int TPB>
constexpr size_t recon2_smem() {
  return size_t(kDepth) * kRows * TPB * KT * sizeof(T);
}

template <typename T, int RC, int KT, int NS, int TPS>
constexpr size_t contract2_smem() {
  return size_t(NS) * kDepth * kRows * TPS * KT * sizeof(T) + size_t(NS) * 2 * kRows * RC * sizeof(T) +
         size_t(NS) * (TPS / 32) * RC * sizeof(double);
}


}  // namespace ntfg
