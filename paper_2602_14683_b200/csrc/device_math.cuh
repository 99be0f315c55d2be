// Device-side scalar algebra of the beta-divergence MU engine.
//
// Everything O(sum I_n R) (MU step, chi transforms, objective terms) runs in
// fp64 and mirrors the reference's special-cased exponent handling exactly
// (reference src/kernels.hpp:12-23 fast_pow, divergence.cpp:16-33 d_beta,
// kernels.hpp:69-75 multiplicative_step, divergence.cpp:57-80 chi1/chi2).
// The E-sized streaming weights (kernels.hpp:30-66) are evaluated in the
// streaming type T: fp64 reproduces the reference formulas operation for
// operation; fp32 uses the SFU paths (rsqrt / ex2 / lg2 / fast divide).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ntfg {

constexpr int kMaxOrder = 8;

// beta classes with dedicated weight loops (kernels.hpp:32-65)
enum BetaKind : int { kBeta0 = 0, kBetaHalf = 1, kBeta1 = 2, kBeta3Half = 3, kBetaGeneric = 4 };

__host__ __device__ inline int beta_kind_of(double beta) {
  if (beta == 1.0) return kBeta1;
  if (beta == 1.5) return kBeta3Half;
  if (beta == 0.5) return kBetaHalf;
  if (beta == 0.0) return kBeta0;
  return kBetaGeneric;
}

// fast_pow (kernels.hpp:12-23): identical branch structure, IEEE fp64 ops.
__device__ __forceinline__ double fpow64(double x, double e) {
  if (e == 0.0) return 1.0;
  if (e == 1.0) return x;
  if (e == -1.0) return 1.0 / x;
  if (e == 2.0) return x * x;
  if (e == -2.0) return 1.0 / (x * x);
  if (e == 0.5) return sqrt(x);
  if (e == -0.5) return 1.0 / sqrt(x);
  if (e == 1.5) return x * sqrt(x);
  if (e == -1.5) return 1.0 / (x * sqrt(x));
  return pow(x, e);
}

// P = x c^(b-2), Q = c^(b-1) with c = max(xhat, eps) -- fp64 flavour.
__device__ __forceinline__ void weights_entry(double x, double xhat, int bk, double beta,
                                              double eps, double& p, double& q) {
  const double c = xhat < eps ? eps : xhat;  // std::max(xhat, eps)
  switch (bk) {
    case kBeta1: p = x / c; q = 1.0; break;
    case kBeta3Half: { const double s = sqrt(c); p = x / s; q = s; break; }
    case kBetaHalf: { const double s = sqrt(c); p = x / (c * s); q = 1.0 / s; break; }
    case kBeta0: p = x / (c * c); q = 1.0 / c; break;
    default: p = x * fpow64(c, beta - 2.0); q = fpow64(c, beta - 1.0); break;
  }
}

// fp32 flavour: SFU reciprocal / rsqrt / ex2 / lg2 (<= 2 ulp each).
__device__ __forceinline__ void weights_entry(float x, float xhat, int bk, double beta,
                                              double eps, float& p, float& q) {
  const float e = static_cast<float>(eps);
  const float c = xhat < e ? e : xhat;
  switch (bk) {
    case kBeta1: p = __fdividef(x, c); q = 1.f; break;
    case kBeta3Half: { const float rs = rsqrtf(c); q = c * rs; p = x * rs; break; }
    case kBetaHalf: { const float rs = rsqrtf(c); q = rs; p = x * __fdividef(rs, c); break; }
    case kBeta0: { const float ic = __fdividef(1.f, c); q = ic; p = x * ic * ic; break; }
    default: {
      const float lg = __log2f(c);
      q = exp2f(static_cast<float>(beta - 1.0) * lg);
      p = x * exp2f(static_cast<float>(beta - 2.0) * lg);
      break;
    }
  }
}

// d_beta (divergence.cpp:16-33) in fp64.  Domain violations are reported
// through `bad` (bit 0: y <= 0, bit 1: x < 0) instead of throwing.
__device__ __forceinline__ double dbeta_entry(double x, double y, int bk, double beta,
                                              unsigned& bad) {
  if (!(y > 0.0)) { bad |= 1u; return 0.0; }
  if (x < 0.0) { bad |= 2u; return 0.0; }
  if (bk == kBeta1) return (x > 0.0 ? x * log(x / y) : 0.0) - x + y;
  if (bk == kBeta0) {
    if (x == 0.0) return __longlong_as_double(0x7ff0000000000000ll);  // +inf
    const double r = x / y;
    return r - log(r) - 1.0;
  }
  const double b = beta;
  return (fpow64(x, b) + (b - 1.0) * fpow64(y, b) - b * x * fpow64(y, b - 1.0)) / (b * (b - 1.0));
}

// multiplicative_step (kernels.hpp:69-75)
__device__ __forceinline__ double mu_step(double anchor, double num, double den, double gamma,
                                          double eps) {
  const double d = den < eps ? eps : den;
  const double v = anchor * fpow64(num / d, gamma);
  return v < eps ? eps : v;  // std::max(v, eps)
}

__device__ __forceinline__ double chi1_entry(double z, double zref, double beta, unsigned& bad) {
  if (!(z > 0.0) || !(zref > 0.0)) bad |= 4u;
  return zref * fpow64(z / zref, beta - 1.0);
}

__device__ __forceinline__ double chi2_entry(double z, double zref, double beta, unsigned& bad) {
  if (!(z > 0.0) || !(zref > 0.0)) bad |= 4u;
  return beta < 1.0 ? z : zref * fpow64(z / zref, beta);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace ntfg
