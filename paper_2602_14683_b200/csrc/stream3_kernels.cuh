// Streaming passes, v3: TMA bulk-copy staging (cp.async.bulk + mbarrier).
//
// 128 threads per stream; each thread owns KT consecutive columns (4 fp32 /
// 2 fp64) so ~128 accumulators stay in registers and every broadcast
// row-vector load feeds 2*KT FMAs (packed FFMA2 for fp32).  Producer lanes of
// warp 0 bulk-copy one row segment each into a kDepth-deep smem ring; the
// per-row vectors (M for the contraction, H for the reconstruction) are
// gathered from the fp64 factors ONE STAGE AHEAD into registers and
// multiplied/stored the next stage, so the gather latency is hidden behind a
// full stage of FMA work.  Rows must be 16-byte multiples
// (K * sizeof(T) % 16 == 0); the v2 kernels cover everything else.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include <cuda_bf16.h>

#include "stream_kernels.cuh"

namespace ntfg {

namespace tma {
__device__ __forceinline__ unsigned saddr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(saddr(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(saddr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar))
      : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "NTFG_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra NTFG_WAIT_%=;\n"
      "}\n" ::"r"(saddr(bar)),
      "r"(phase)
      : "memory");
}
}  // namespace tma

template <typename T, int KT> struct VecT;
template <> struct VecT<float, 4> { using type = float4; };
template <> struct VecT<float, 2> { using type = float2; };
template <> struct VecT<float, 1> { using type = float; };
template <> struct VecT<double, 2> { using type = double2; };
template <> struct VecT<double, 1> { using type = double; };

// accumulator lane type: packed pairs for fp32 with an even column count
template <typename T, int KT> struct Acc { using type = T; static constexpr int W = 1; };
template <> struct Acc<float, 4> { using type = float2; static constexpr int W = 2; };
template <> struct Acc<float, 2> { using type = float2; static constexpr int W = 2; };

template <typename A> __device__ __forceinline__ A acc_fma(A s, double m, A g);
template <> __device__ __forceinline__ float2 acc_fma<float2>(float2 s, double m, float2 g) {
  const float mf = float(m);
  return __ffma2_rn(s, make_float2(mf, mf), g);
}
template <> __device__ __forceinline__ float acc_fma<float>(float s, double m, float g) { return fmaf(s, float(m), g); }
template <> __device__ __forceinline__ double acc_fma<double>(double s, double m, double g) { return fma(s, m, g); }

constexpr int kPre = 3;  // row-mode factor values prefetched per item

// p ~= hi + lo with hi = RN_bf16(p), lo = RN_bf16(p - hi), except that lo is
// rounded toward zero when hi + lo would be a bf16 tie that rounds away from
// hi: then RN_bf16(hi + lo) == hi always, so planes written here survive the
// fp64 round trip of the step-level API (join -> host -> split) bit for bit.
// hi + lo is exact in fp32 (lo only rounds when d spans > 8 bits below hi).
__device__ __forceinline__ uint32_t bf16x2_bits(__nv_bfloat162 v) { return *reinterpret_cast<uint32_t*>(&v); }
__device__ __forceinline__ float bf16_lo_f(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16_hi_f(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }

// two values at once (packed cvt): element a in the low half, b in the high half
__device__ __forceinline__ void bf16_split_pair(float a, float b, uint32_t& hi, uint32_t& lo) {
  const uint32_t hu = bf16x2_bits(__floats2bfloat162_rn(a, b));
  const float da = a - bf16_lo_f(hu), db = b - bf16_hi_f(hu);  // exact
  uint32_t lu = bf16x2_bits(__floats2bfloat162_rn(da, db));
  const uint32_t chk =
      bf16x2_bits(__floats2bfloat162_rn(bf16_lo_f(hu) + bf16_lo_f(lu), bf16_hi_f(hu) + bf16_hi_f(lu)));
  if (chk != hu) {  // rare
    if ((chk ^ hu) & 0xffffu)
      lu = (lu & 0xffff0000u) | uint32_t(__bfloat16_as_ushort(__float2bfloat16_rz(da)));
    if ((chk ^ hu) >> 16) lu = (lu & 0xffffu) | (uint32_t(__bfloat16_as_ushort(__float2bfloat16_rz(db))) << 16);
  }
  hi = hu;
  lo = lu;
}

__device__ __forceinline__ void bf16_split_stable(float p, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  uint32_t h, l;
  bf16_split_pair(p, 0.f, h, l);
  hi = __ushort_as_bfloat16((unsigned short)(h & 0xffffu));
  lo = __ushort_as_bfloat16((unsigned short)(l & 0xffffu));
}

// Per-thread prefetch of row-vector entries (fp64 factor gathers), one stage ahead.
template <int ITEMS>
struct RowPrefetch {
  double v[ITEMS][kPre];
};

template <typename T, int RC, int KT, int NS>
struct C3Smem {
  static constexpr int TPS = 128;
  static constexpr int W = TPS * KT;
  static constexpr size_t ring = size_t(NS) * kDepth * kRows * W * sizeof(T);
  static constexpr size_t mbuf = size_t(NS) * 2 * kRows * RC * sizeof(T);
  static constexpr size_t wsum = size_t(NS) * (TPS / 32) * RC * sizeof(double);
  static constexpr size_t bars = size_t(NS) * kDepth * sizeof(uint64_t);
  static constexpr size_t total = ring + mbuf + wsum + bars;
};

template <typename T, int RC, int KT, int NS>
static __global__ void __launch_bounds__(NS * 128, 1) contract3_kernel(const ContractParams<T, NS> p) {
  using L = C3Smem<T, RC, KT, NS>;
  using A = typename Acc<T, KT>::type;
  constexpr int AW = Acc<T, KT>::W;
  constexpr int TPS = L::TPS, W = L::W, WPS = TPS / 32;
  constexpr int ITEMS = (kRows * RC + TPS - 1) / TPS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* ring = reinterpret_cast<T*>(smem_raw);
  T* mbuf = reinterpret_cast<T*>(smem_raw + L::ring);
  double* wsum = reinterpret_cast<double*>(smem_raw + L::ring + L::mbuf);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + L::ring + L::mbuf + L::wsum);
  __shared__ double usum[NS][RC];

  const int s = threadIdx.x / TPS;
  const int t = threadIdx.x % TPS;
  const int lane = threadIdx.x & 31;
  const int wis = t >> 5;
  const int64_t K = p.g.K;
  const int nrow_modes = p.g.order - 1;
  const T* __restrict__ src = p.src[s];
  const double* __restrict__ mtab = p.mtab[s];
  const int64_t In = p.g.dims[p.n];
  T* myring = ring + size_t(s) * kDepth * kRows * W;
  T* mym = mbuf + size_t(s) * 2 * kRows * RC;
  uint64_t* mybar = bars + s * kDepth;
  const int bar = 1 + s;
  const bool producer = (t < 32);
  // row modes contributing to M (all prefix modes but the target)
  int mm[kMaxOrder];
  int nmm = 0;
  for (int m = 0; m < nrow_modes; ++m)
    if (m != p.n) mm[nmm++] = m;

  if (t == 0)
    for (int d = 0; d < kDepth; ++d) tma::mbar_init(&mybar[d], 1);
  tma::fence_barrier_init();
  __syncthreads();

  uint32_t seq = 0;
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
      const int64_t kbase = int64_t(kt) * W;
      const int64_t seg = (K - kbase < W ? K - kbase : W);
      const int64_t k0 = kbase + int64_t(t) * KT;
      const bool kvalid = k0 < K;
      auto issue = [&](int64_t b) {
        if (!producer || b >= nblk) return;
        const uint32_t q = seq + uint32_t(b);
        T* dst = myring + size_t(q % kDepth) * kRows * W;
        const int64_t jb = j0 + b * kRows;
        const int nrows = int(j1 - jb < kRows ? j1 - jb : kRows);
        if (lane == 0) {
          tma::fence_proxy_async();
          tma::expect_tx(&mybar[q % kDepth], unsigned(nrows * seg * sizeof(T)));
        }
        __syncwarp();
        if (lane < nrows)
          tma::bulk_g2s(dst + size_t(lane) * W, src + row_of(jb + lane) * K + kbase, unsigned(seg * sizeof(T)),
                        &mybar[q % kDepth]);
      };
      RowPrefetch<ITEMS> pre;
      auto load_m = [&](int64_t b) {
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const int idx = t + i * TPS;
          const int rr = idx / RC, r = idx % RC;
          const int64_t j = j0 + b * kRows + rr;
          pre.v[i][0] = 0.0;
          pre.v[i][1] = 1.0;
          pre.v[i][2] = 1.0;
          if (idx < kRows * RC && b < nblk && j < j1 && p.r0 + r < p.R) {
            const int64_t row = row_of(j);
            if (mtab) {
              pre.v[i][0] = mtab[row * p.R + p.r0 + r];
            } else {
              pre.v[i][0] = 1.0;
#pragma unroll
              for (int c = 0; c < kPre; ++c)
                if (c < nmm) pre.v[i][c] = p.mfac[s][mm[c]][p.g.coord(row, mm[c]) * p.R + p.r0 + r];
            }
          }
        }
      };
      auto store_m = [&](int64_t b, int slot) {
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const int idx = t + i * TPS;
          if (idx >= kRows * RC) continue;
          const int rr = idx / RC, r = idx % RC;
          double v = pre.v[i][0] * pre.v[i][1] * pre.v[i][2];
          if (!mtab && nmm > kPre) {  // high-order tensors: remaining modes gathered here
            const int64_t j = j0 + b * kRows + rr;
            if (b < nblk && j < j1 && p.r0 + r < p.R) {
              const int64_t row = row_of(j);
              for (int c = kPre; c < nmm; ++c) v *= p.mfac[s][mm[c]][p.g.coord(row, mm[c]) * p.R + p.r0 + r];
            }
          }
          mym[(size_t(slot) * kRows + rr) * RC + r] = T(v);
        }
      };

      A g[RC][KT / AW];
#pragma unroll
      for (int r = 0; r < RC; ++r)
#pragma unroll
        for (int h = 0; h < KT / AW; ++h) g[r][h] = A{};

      named_sync(bar, TPS);  // ring + M buffers free
#pragma unroll 1
      for (int d = 0; d < kDepth - 1; ++d) issue(d);
      load_m(0);
      store_m(0, 0);
      load_m(1);
#pragma unroll 1
      for (int64_t b = 0; b < nblk; ++b) {
        named_sync(bar, TPS);  // block b-1 consumed; M(b) visible
        issue(b + kDepth - 1);
        store_m(b + 1, int((b + 1) & 1));  // values loaded one stage ago
        load_m(b + 2);                     // next gather in flight during this stage
        const uint32_t q = seq + uint32_t(b);
        tma::wait(&mybar[q % kDepth], (q / kDepth) & 1u);
        const T* srow = myring + size_t(q % kDepth) * kRows * W + t * KT;
        const T* mrow = mym + size_t(b & 1) * kRows * RC;
        const int nrows = int(j1 - (j0 + b * kRows) < kRows ? j1 - (j0 + b * kRows) : kRows);
        if (kvalid) {
#pragma unroll
          for (int rr = 0; rr < kRows; ++rr) {
            if (rr >= nrows) break;
            A sv[KT / AW];
            *reinterpret_cast<typename VecT<T, KT>::type*>(sv) =
                *reinterpret_cast<const typename VecT<T, KT>::type*>(srow + size_t(rr) * W);
#pragma unroll
            for (int r = 0; r < RC; r += 4) {
              T m4[4];
              if constexpr (sizeof(T) == 4) {
                *reinterpret_cast<float4*>(m4) = *reinterpret_cast<const float4*>(mrow + rr * RC + r);
              } else {
                *reinterpret_cast<double2*>(m4) = *reinterpret_cast<const double2*>(mrow + rr * RC + r);
                *reinterpret_cast<double2*>(m4 + 2) = *reinterpret_cast<const double2*>(mrow + rr * RC + r + 2);
              }
#pragma unroll
              for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int h = 0; h < KT / AW; ++h) g[r + c][h] = acc_fma<A>(sv[h], m4[c], g[r + c][h]);
            }
          }
        }
      }
      seq += uint32_t(nblk);

      const T* gp = reinterpret_cast<const T*>(&g[0][0]);  // gp[r * KT + kk] = G(k0 + kk, r)
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
            for (int kk = 0; kk < KT; ++kk) v += double(gp[r * KT + kk]) * p.lastfac[s][(k0 + kk) * p.R + p.r0 + r];
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

// ---------------------------------------------------------------------------
// K2/K5: reconstruction + weights + objective with bulk-copied X rows.

template <typename T, int RP, int KT>
struct R3Smem {
  static constexpr int TPB = 128;
  static constexpr int W = TPB * KT;
  static constexpr size_t ring = size_t(kDepth) * kRows * W * sizeof(T);
  static constexpr size_t bars = size_t(kDepth) * sizeof(uint64_t);
  static constexpr size_t total = ring + bars;
};

// Tensor-core flavour of the weights tail, one beta kind per instantiation:
// P~/Q~ straight into the bf16 hi/lo planes, and the objective in its
// "model part" form -- the x-only part of d_beta (x^b / (b (b-1)) for
// b not in {0, 1}) is a per-tensor constant summed once in fp64
// (xconst_kernel) and added by objective_finalize_kernel, so each entry
// costs a couple of FMAs on top of the weights it shares Q with.
struct TailConst {
  float e, b, b1, b2, ib;  // eps, beta, beta-1, beta-2, 1/(beta(beta-1))
};

// c >= eps > 0 here; the .ftz approximation skips the denormal scaling
// rsqrtf() carries (an fp32 eps below FLT_MIN is not representable anyway)
__device__ __forceinline__ float rsqrt_ftz(float c) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(c));
  return r;
}

template <int BK>
__device__ __forceinline__ void tc_weights(float x, float y, const TailConst& k, float& pv, float& qv,
                                           bool obj, float& oacc, unsigned& bad) {
  const float c = y < k.e ? k.e : y;  // std::max(xhat, eps)
  // same formulas as weights_entry(float, ...) (identical results for normal c)
  if constexpr (BK == kBeta1) {
    pv = __fdividef(x, c);
    qv = 1.f;
  } else if constexpr (BK == kBetaHalf) {
    const float rs = rsqrt_ftz(c);
    qv = rs;
    pv = x * __fdividef(rs, c);
  } else if constexpr (BK == kBeta3Half) {
    const float rs = rsqrt_ftz(c);
    qv = c * rs;
    pv = x * rs;
  } else if constexpr (BK == kBeta0) {
    const float ic = __fdividef(1.f, c);
    qv = ic;
    pv = x * ic * ic;
  } else {
    const float lg = __log2f(c);
    qv = exp2f(k.b1 * lg);
    pv = x * exp2f(k.b2 * lg);
  }
  if (!obj) return;
  if (!(y > 0.f)) bad |= 1u;
  if (x < 0.f) bad |= 2u;
  const bool clamped = y < k.e;  // rare: the objective needs xhat itself
  float t;
  if constexpr (BK == kBeta1) {
    t = (x > 0.f ? x * __logf(clamped ? __fdividef(x, y) : pv) : 0.f) - x + y;
  } else if constexpr (BK == kBeta0) {
    const float r = clamped ? __fdividef(x, y) : x * qv;
    t = x == 0.f ? __int_as_float(0x7f800000) : r - __logf(r) - 1.f;
  } else if constexpr (BK == kBetaHalf) {  // -4 sqrt(x) + 2 y^-.5 (x + y)
    const float q = clamped ? rsqrtf(y) : qv;
    t = 2.f * q * (x + y);
  } else if constexpr (BK == kBeta3Half) {  // x^1.5 / .75 + y^.5 (2y/3 - 2x)
    const float q = clamped ? y * rsqrtf(y) : qv;
    t = q * (y * (2.f / 3.f) - 2.f * x);
  } else {  // x^b / (b (b-1)) + y^(b-1) ((b-1) y - b x) / (b (b-1))
    const float q = clamped ? exp2f(k.b1 * __log2f(y)) : qv;
    t = q * (k.b1 * y - k.b * x) * k.ib;
  }
  oacc += t;
}

// bf16 hi/lo stores of KT consecutive weights
template <int KT>
__device__ __forceinline__ void store_planes(const float* w, __nv_bfloat16* hi, __nv_bfloat16* lo) {
  if constexpr (KT == 1) {
    bf16_split_stable(w[0], hi[0], lo[0]);
  } else {
    uint32_t h[KT / 2], l[KT / 2];
#pragma unroll
    for (int j = 0; j < KT / 2; ++j) bf16_split_pair(w[2 * j], w[2 * j + 1], h[j], l[j]);
    if constexpr (KT == 2) {
      *reinterpret_cast<uint32_t*>(hi) = h[0];
      *reinterpret_cast<uint32_t*>(lo) = l[0];
    } else {
      *reinterpret_cast<uint2*>(hi) = make_uint2(h[0], h[1]);
      *reinterpret_cast<uint2*>(lo) = make_uint2(l[0], l[1]);
    }
  }
}

// BK = -1: any output set, beta kind at run time.  BK >= 0 (fp32 only):
// tensor-core planes output for that beta kind, objective optional.
template <typename T, int RP, int KT, int BK = -1>
static __global__ void __launch_bounds__(128) recon3_kernel(const ReconParams<T> p) {
  using L = R3Smem<T, RP, KT>;
  using A = typename Acc<T, KT>::type;
  constexpr int AW = Acc<T, KT>::W;
  constexpr int TPB = L::TPB, W = L::W;
  constexpr int ITEMS = (kRows * RP + TPB - 1) / TPB;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* ring = reinterpret_cast<T*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + L::ring);
  __shared__ __align__(16) T hs[2][kRows][RP];
  __shared__ double red[TPB / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t K = p.g.K;
  const int nprefix = p.g.order - 1;
  const int kt = int(blockIdx.x % p.ktiles);
  const int64_t rb_stride = gridDim.x / p.ktiles;
  const int64_t row_blocks = (p.g.rows + kRows - 1) / kRows;
  const int64_t kbase = int64_t(kt) * W;
  const int64_t seg = (K - kbase < W ? K - kbase : W);
  const int64_t k0 = kbase + int64_t(tid) * KT;
  const bool kvalid = k0 < K;

  if (tid == 0)
    for (int d = 0; d < kDepth; ++d) tma::mbar_init(&bars[d], 1);
  tma::fence_barrier_init();
  __syncthreads();

  // last-factor columns of this thread, packed like the accumulators
  A a[RP][KT / AW];
#pragma unroll
  for (int r = 0; r < RP; ++r)
#pragma unroll
    for (int h = 0; h < KT / AW; ++h) {
      T tmp[AW];
#pragma unroll
      for (int w = 0; w < AW; ++w) tmp[w] = kvalid ? __ldg(p.alast + (k0 + h * AW + w) * RP + r) : T(0);
      a[r][h] = *reinterpret_cast<const A*>(tmp);
    }

  const int64_t rb0 = blockIdx.x / p.ktiles;
  const int64_t nmine = rb0 < row_blocks ? (row_blocks - rb0 + rb_stride - 1) / rb_stride : 0;
  auto issue = [&](int64_t i) {
    if (warp != 0 || i >= nmine) return;
    const int64_t row0 = (rb0 + i * rb_stride) * kRows;
    const int nrows = int(p.g.rows - row0 < kRows ? p.g.rows - row0 : kRows);
    T* dst = ring + size_t(i % kDepth) * kRows * W;
    if (lane == 0) {
      tma::fence_proxy_async();
      tma::expect_tx(&bars[i % kDepth], unsigned(nrows * seg * sizeof(T)));
    }
    __syncwarp();
    if (lane < nrows)
      tma::bulk_g2s(dst + size_t(lane) * W, p.x + (row0 + lane) * K + kbase, unsigned(seg * sizeof(T)),
                    &bars[i % kDepth]);
  };
  RowPrefetch<ITEMS> pre;
  auto load_h = [&](int64_t i) {
    const int64_t rb = rb0 + i * rb_stride;
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
      const int idx = tid + it * TPB;
      const int rr = idx / RP, r = idx % RP;
      const int64_t row = rb * kRows + rr;
      pre.v[it][0] = 0.0;
      pre.v[it][1] = 1.0;
      pre.v[it][2] = 1.0;
      if (idx < kRows * RP && i < nmine && r < p.R && row < p.g.rows) {
        if (p.htab) {
          pre.v[it][0] = p.htab[row * p.R + r];
        } else {
          pre.v[it][0] = 1.0;
#pragma unroll
          for (int c = 0; c < kPre; ++c)
            if (c < nprefix) pre.v[it][c] = p.fac[c][p.g.coord(row, c) * p.R + r];
        }
      }
    }
  };
  auto store_h = [&](int64_t i, int slot) {
    const int64_t rb = rb0 + i * rb_stride;
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
      const int idx = tid + it * TPB;
      if (idx >= kRows * RP) continue;
      const int rr = idx / RP, r = idx % RP;
      double h = pre.v[it][0] * pre.v[it][1] * pre.v[it][2];
      if (!p.htab && nprefix > kPre) {
        const int64_t row = rb * kRows + rr;
        if (i < nmine && r < p.R && row < p.g.rows)
          for (int c = kPre; c < nprefix; ++c) h *= p.fac[c][p.g.coord(row, c) * p.R + r];
      }
      hs[slot][rr][r] = T(h);
    }
  };

  double obj = 0.0;
  unsigned bad = 0;
  TailConst tk;
  tk.e = float(p.eps);
  tk.b = float(p.beta);
  tk.b1 = float(p.beta - 1.0);
  tk.b2 = float(p.beta - 2.0);
  tk.ib = float(1.0 / (p.beta * (p.beta - 1.0)));
  const bool want_obj = p.obj != nullptr;
  for (int d = 0; d < kDepth - 1; ++d) issue(d);
  load_h(0);
  store_h(0, 0);
  load_h(1);
#pragma unroll 1
  for (int64_t i = 0; i < nmine; ++i) {
    __syncthreads();
    issue(i + kDepth - 1);
    store_h(i + 1, int((i + 1) & 1));
    load_h(i + 2);
    tma::wait(&bars[i % kDepth], unsigned((i / kDepth) & 1));
    const int64_t row0 = (rb0 + i * rb_stride) * kRows;
    const T* xrow = ring + size_t(i % kDepth) * kRows * W + tid * KT;
    // plane element offset of (row0, k0); rows advance by K (tensor-core flavour)
    const int64_t off0 = row0 * K + k0;
    __nv_bfloat16* const pl0 = static_cast<__nv_bfloat16*>(p.planes[0]) + off0;
    __nv_bfloat16* const pl1 = static_cast<__nv_bfloat16*>(p.planes[1]) + off0;
    __nv_bfloat16* const pl2 = static_cast<__nv_bfloat16*>(p.planes[2]) + off0;
    __nv_bfloat16* const pl3 = static_cast<__nv_bfloat16*>(p.planes[3]) + off0;
#pragma unroll
    for (int rr = 0; rr < kRows; ++rr) {
      const int64_t row = row0 + rr;
      if (row >= p.g.rows) break;
      A xh[KT / AW];
#pragma unroll
      for (int h = 0; h < KT / AW; ++h) xh[h] = A{};
#pragma unroll
      for (int r = 0; r < RP; r += 4) {
        T h4[4];
        if constexpr (sizeof(T) == 4) {
          *reinterpret_cast<float4*>(h4) = *reinterpret_cast<const float4*>(&hs[i & 1][rr][r]);
        } else {
          *reinterpret_cast<double2*>(h4) = *reinterpret_cast<const double2*>(&hs[i & 1][rr][r]);
          *reinterpret_cast<double2*>(h4 + 2) = *reinterpret_cast<const double2*>(&hs[i & 1][rr][r + 2]);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int h = 0; h < KT / AW; ++h) xh[h] = acc_fma<A>(a[r + c][h], h4[c], xh[h]);
      }
      if (!kvalid) continue;
      const T* xhp = reinterpret_cast<const T*>(xh);
      T xv[KT];
      *reinterpret_cast<typename VecT<T, KT>::type*>(xv) =
          *reinterpret_cast<const typename VecT<T, KT>::type*>(xrow + size_t(rr) * W);
      if constexpr (BK >= 0 && sizeof(T) == 4) {
        float pw[KT], qw[KT];
        float oacc = 0.f;
#pragma unroll
        for (int kk = 0; kk < KT; ++kk)
          tc_weights<BK>(float(xv[kk]), float(xhp[kk]), tk, pw[kk], qw[kk], want_obj, oacc, bad);
        if (want_obj) obj += double(oacc);
        const int ro = rr * int(K);  // < 2^31: rows of one block
        store_planes<KT>(pw, pl0 + ro, pl1 + ro);
        if constexpr (BK != kBeta1) store_planes<KT>(qw, pl2 + ro, pl3 + ro);
        continue;
      }
      T pw[KT], qw[KT];
#pragma unroll
      for (int kk = 0; kk < KT; ++kk) {
        if (p.xhout) p.xhout[row * K + k0 + kk] = xhp[kk];
        if (p.pout || p.planes[0]) weights_entry(xv[kk], xhp[kk], p.bk, p.beta, p.eps, pw[kk], qw[kk]);
        if (p.obj) obj += objective_term<T>(xv[kk], xhp[kk], p.bk, p.beta, bad);
      }
      if (p.planes[0]) {  // tensor-core storage: bf16 hi/lo planes of P and Q
        __nv_bfloat16* ph = static_cast<__nv_bfloat16*>(p.planes[0]) + row * K + k0;
        __nv_bfloat16* pl = static_cast<__nv_bfloat16*>(p.planes[1]) + row * K + k0;
        __nv_bfloat16* qh = static_cast<__nv_bfloat16*>(p.planes[2]) + row * K + k0;
        __nv_bfloat16* ql = static_cast<__nv_bfloat16*>(p.planes[3]) + row * K + k0;
#pragma unroll
        for (int kk = 0; kk < KT; ++kk) {
          bf16_split_stable(float(pw[kk]), ph[kk], pl[kk]);
          if (p.planes[2]) bf16_split_stable(float(qw[kk]), qh[kk], ql[kk]);
        }
      } else if (p.pout) {
        *reinterpret_cast<typename VecT<T, KT>::type*>(p.pout + row * K + k0) =
            *reinterpret_cast<const typename VecT<T, KT>::type*>(pw);
        if (p.qout)
          *reinterpret_cast<typename VecT<T, KT>::type*>(p.qout + row * K + k0) =
              *reinterpret_cast<const typename VecT<T, KT>::type*>(qw);
      }
    }
  }
  if (p.obj) {
    obj = warp_sum(obj);
    if (lane == 0) red[warp] = obj;
    __syncthreads();
    if (tid == 0) {
      double sacc = 0.0;
      for (int w = 0; w < TPB / 32; ++w) sacc += red[w];
      p.obj[blockIdx.x] = sacc;
    }
  }
  if (bad && p.flags) atomicOr(p.flags, bad);
}

}  // namespace ntfg
