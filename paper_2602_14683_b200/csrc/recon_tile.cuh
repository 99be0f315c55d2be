// K2/K5 on the tensor-core (fp32) path: reconstruction + weights + objective
// as a register-tiled outer product.
//
//   Xhat(row, k) = sum_r H(row, r) A_last(k, r),   H(row, r) = prod_{m<N-1} A_m(i_m(row), r)
//
// A CTA owns one 128-column k tile of the last factor (transposed into shared
// memory once) and walks 32-row tiles of X.  Each thread computes a 4 row x
// 4 column block: per rank step one broadcast LDS.128 of H, one LDS.128 of
// A_last and 8 FFMA2 -- 16 independent accumulation chains instead of recon3's
// one chain per row, and no per-row register copy of A_last, so R = 64 runs at
// the same per-entry cost as R = 32.  Each accumulator sums r = 0..R-1 in
// order with fmaf, exactly like recon3_kernel, so Xhat, P~ and Q~ are bitwise
// unchanged.  X tiles are prefetched one tile ahead into registers (coalesced
// 512-byte rows per warp); the next tile's H rows are gathered (fp64 factor
// rows, product in the reference order) while the current tile computes.
//
// The weights tail (tc_weights formulas) writes P~/Q~ as bf16 hi/lo planes
// with 8-byte stores.  The objective uses the tensor-core "model part"
// (xconst_kernel supplies the x-only term); the per-entry domain checks of
// tc_weights are replaced by a per-tile min/sum screen, and a tile that trips
// it (xhat < eps, NaN/Inf, x < 0 -- rare) is re-evaluated entry by entry with
// tc_weights itself, so flags and clamped terms are exactly the old ones.
#pragma once
#include "stream3_kernels.cuh"

namespace ntfg {

constexpr int kRtRows = 32;      // rows per tile
constexpr int kRtCols = 128;     // k columns per CTA
constexpr int kRtThreads = 256;  // 8 warps x (4 rows) ; 32 lanes x (4 columns)

template <int RP>
struct RtSmem {
  static constexpr int HS = kRtRows + 4;  // padded H row stride (floats), keeps 16-byte alignment
  static constexpr size_t as = size_t(RP) * kRtCols * 4;
  static constexpr size_t hs = size_t(2) * RP * HS * 4;
  static constexpr size_t total = as + hs;
};

// fast (unclamped) weights + objective model term: same p/q formulas as
// tc_weights.  `t` is accumulated with one FMA; rt_obj_scale folds the
// constant factor back in per tile (exact: a power of two or 1).  NaN/Inf
// models reach the tile sum through y itself, except at beta = 0 whose
// clamp is the NaN-propagating select of tc_weights.
// 1 / c for c >= eps (a normal fp32): the bare SFU reciprocal; __fdividef's
// range scaling (five more instructions per entry) is for denormal divisors
__device__ __forceinline__ float rcp_ftz(float c) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(c));
  return r;
}

template <int BK>
__device__ __forceinline__ void rt_weights(float x, float y, const TailConst& k, float& pv, float& qv, float& tacc) {
  if constexpr (BK == kBeta1) {
    const float c = fmaxf(y, k.e);
    pv = x * rcp_ftz(c);
    qv = 1.f;
    tacc += (x > 0.f ? x * __logf(pv) : 0.f) - x + y;
  } else if constexpr (BK == kBetaHalf) {  // q = c^-1/2, p = x c^-3/2 = x q^3; t = 2 q (x + y)
    const float c = fmaxf(y, k.e);
    const float rs = rsqrt_ftz(c);
    qv = rs;
    pv = (x * rs) * (rs * rs);
    tacc = fmaf(qv, x + y, tacc);
  } else if constexpr (BK == kBeta3Half) {
    const float c = fmaxf(y, k.e);
    const float rs = rsqrt_ftz(c);
    qv = c * rs;
    pv = x * rs;
    tacc = fmaf(qv, y * (2.f / 3.f) - 2.f * x, tacc);
  } else if constexpr (BK == kBeta0) {
    const float c = y < k.e ? k.e : y;
    const float ic = rcp_ftz(c);
    qv = ic;
    pv = x * ic * ic;
    const float r = x * qv;
    tacc += x == 0.f ? __int_as_float(0x7f800000) : r - __logf(r) - 1.f;
  } else {
    const float c = fmaxf(y, k.e);
    const float lg = __log2f(c);
    qv = exp2f(k.b1 * lg);
    pv = x * exp2f(k.b2 * lg);
    tacc = fmaf(qv, k.b1 * y - k.b * x, tacc);
  }
}
template <int BK>
__device__ __forceinline__ float rt_obj_scale(const TailConst& k) {
  if constexpr (BK == kBetaHalf) return 2.f;
  else if constexpr (BK == kBetaGeneric) return k.ib;
  else return 1.f;
}

// stable hi/lo split of two values (same pairs as bf16_split_pair) with the
// round-trip check done by one packed bf16 add
__device__ __forceinline__ void rt_split_pair(float a, float b, uint32_t& hi, uint32_t& lo) {
  const uint32_t hu = bf16x2_bits(__floats2bfloat162_rn(a, b));
  uint32_t lu = bf16x2_bits(__floats2bfloat162_rn(a - bf16_lo_f(hu), b - bf16_hi_f(hu)));
  const __nv_bfloat162 s2 = __hadd2(*reinterpret_cast<const __nv_bfloat162*>(&hu),
                                    *reinterpret_cast<const __nv_bfloat162*>(&lu));
  if (bf16x2_bits(s2) != hu) {  // rare tie: the full routine applies the round-toward-zero fixup
    bf16_split_pair(a, b, hi, lo);
  } else {
    hi = hu;
    lo = lu;
  }
}

// the same split without the tie test: `tie` collects (hi + lo as bf16) ^ hi so
// that a block of entries is tested with ONE branch; a block with a tie is
// redone with rt_split_pair (rare: ~2^-8 per entry)
__device__ __forceinline__ void rt_split_pair_nocheck(float a, float b, uint32_t& hi, uint32_t& lo, uint32_t& tie) {
  hi = bf16x2_bits(__floats2bfloat162_rn(a, b));
  lo = bf16x2_bits(__floats2bfloat162_rn(a - bf16_lo_f(hi), b - bf16_hi_f(hi)));
  const __nv_bfloat162 s2 = __hadd2(*reinterpret_cast<const __nv_bfloat162*>(&hi),
                                    *reinterpret_cast<const __nv_bfloat162*>(&lo));
  tie |= bf16x2_bits(s2) ^ hi;
}

// NPRE: number of row (prefix) modes when 1..3 and the fastest one has 32 | I
// (a tile's 32 rows then share the slower coordinates: H = G(r) * A_f rows,
// G = product of the slower modes' rows, computed once per tile); 0 = generic.
template <int RP, int BK, int NPRE>
static __global__ void __launch_bounds__(kRtThreads, 3) recon_tile_kernel(const ReconParams<float> p) {
  using L = RtSmem<RP>;
  constexpr int HS = L::HS;
  constexpr int HI = RP * kRtRows / kRtThreads;  // H items per thread per tile (same r for all)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* as = reinterpret_cast<float*>(smem_raw);              // [RP][128]
  float* hs = reinterpret_cast<float*>(smem_raw + L::as);      // [2][RP][HS]
  __shared__ double red[kRtThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t K = p.g.K;
  const int64_t rows = p.g.rows;
  const int R = p.R;
  const int ktiles = p.ktiles;
  const int kt = int(blockIdx.x % ktiles);
  const int64_t tstride = gridDim.x / ktiles;
  const int64_t ntiles = (rows + kRtRows - 1) / kRtRows;
  const int64_t kbase = int64_t(kt) * kRtCols;
  const int64_t kcol = kbase + lane * 4;
  const int hr = tid % RP;          // this thread's H column
  const int hrr0 = tid / RP;        // first H row; rows hrr0 + it * (256 / RP)

  // last-factor tile, transposed (k contiguous); alast is [K][RP]
  for (int i = tid; i < RP * kRtCols; i += kRtThreads) {
    const int kk = i / RP, r = i % RP;
    as[r * kRtCols + kk] = p.alast[(kbase + kk) * RP + r];
  }

  float hv[HI];
  auto load_h = [&](int64_t tile) {
    const int64_t row0 = tile * kRtRows;
    if (tile >= ntiles || hr >= R) {
#pragma unroll
      for (int it = 0; it < HI; ++it) hv[it] = 0.f;
      return;
    }
    if constexpr (NPRE >= 1) {
      // row0 -> (c_0, .., c_{NPRE-1}) with NPRE - 1 divisions (row < 2^31 on this path)
      int64_t c[3] = {0, 0, 0};
      int64_t q = row0;
      if constexpr (NPRE == 3) {
        const int64_t t = p.g.fd[2].div(q);
        c[2] = q - t * p.g.dims[2];
        c[0] = p.g.fd[1].div(t);
        c[1] = t - c[0] * p.g.dims[1];
      } else if constexpr (NPRE == 2) {
        c[0] = p.g.fd[1].div(q);
        c[1] = q - c[0] * p.g.dims[1];
      } else {
        c[0] = q;
      }
      double g = 1.0;
      if constexpr (NPRE >= 2) g = p.fac[0][c[0] * R + hr];
      if constexpr (NPRE >= 3) g *= p.fac[1][c[1] * R + hr];
      const double* fr = p.fac[NPRE - 1] + (c[NPRE - 1] + hrr0) * R + hr;
#pragma unroll
      for (int it = 0; it < HI; ++it) {
        const double v = fr[int64_t(it) * (kRtThreads / RP) * R];
        hv[it] = float(NPRE >= 2 ? g * v : v);  // ((f0 * f1) * f2): the reference product order
      }
    } else {
      const int nprefix = p.g.order - 1;
#pragma unroll
      for (int it = 0; it < HI; ++it) {
        const int64_t row = row0 + hrr0 + it * (kRtThreads / RP);
        double h = 0.0;
        if (row < rows) {
          for (int m = 0; m < nprefix; ++m) {
            const double v = p.fac[m][p.g.coord(row, m) * R + hr];
            h = m == 0 ? v : h * v;
          }
        }
        hv[it] = float(h);
      }
    }
  };
  auto store_h = [&](int buf) {
#pragma unroll
    for (int it = 0; it < HI; ++it) hs[(size_t(buf) * RP + hr) * HS + hrr0 + it * (kRtThreads / RP)] = hv[it];
  };
  auto load_x = [&](int64_t tile, float4 (&xv)[4]) {
    const int64_t row = tile * kRtRows + warp * 4;
    const float* xb = p.x + row * K + kcol;
    if (row + 4 <= rows) {  // every row of a full tile (tile < ntiles implied)
#pragma unroll
      for (int i = 0; i < 4; ++i) xv[i] = __ldg(reinterpret_cast<const float4*>(xb + i * K));
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        xv[i] = (tile < ntiles && row + i < rows) ? __ldg(reinterpret_cast<const float4*>(xb + i * K))
                                                  : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };

  TailConst tk;
  tk.e = float(p.eps);
  tk.b = float(p.beta);
  tk.b1 = float(p.beta - 1.0);
  tk.b2 = float(p.beta - 2.0);
  tk.ib = float(1.0 / (p.beta * (p.beta - 1.0)));
  const float oscale = rt_obj_scale<BK>(tk);
  const bool want_obj = p.obj != nullptr;
  const bool store = p.planes[0] != nullptr;
  __nv_bfloat16* const pl0 = static_cast<__nv_bfloat16*>(p.planes[0]);
  __nv_bfloat16* const pl1 = static_cast<__nv_bfloat16*>(p.planes[1]);
  __nv_bfloat16* const pl2 = static_cast<__nv_bfloat16*>(p.planes[2]);
  __nv_bfloat16* const pl3 = static_cast<__nv_bfloat16*>(p.planes[3]);
  double obj = 0.0;
  unsigned bad = 0;

  int64_t tile = blockIdx.x / ktiles;
  load_h(tile);
  store_h(0);
  float4 xn[4];
  load_x(tile, xn);
  __syncthreads();
  for (int buf = 0; tile < ntiles; tile += tstride, buf ^= 1) {
    const int64_t nxt = tile + tstride;
    float4 xc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) xc[i] = xn[i];
    load_h(nxt);
    load_x(nxt, xn);

    float2 acc[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = make_float2(0.f, 0.f);
    const float* hb = hs + size_t(buf) * RP * HS + warp * 4;
    const float* ab = as + lane * 4;
#pragma unroll 8
    for (int r = 0; r < RP; ++r) {
      const float4 h = *reinterpret_cast<const float4*>(hb + r * HS);
      const float4 a = *reinterpret_cast<const float4*>(ab + r * kRtCols);
      const float2 a01 = make_float2(a.x, a.y), a23 = make_float2(a.z, a.w);
      acc[0][0] = __ffma2_rn(a01, make_float2(h.x, h.x), acc[0][0]);
      acc[0][1] = __ffma2_rn(a23, make_float2(h.x, h.x), acc[0][1]);
      acc[1][0] = __ffma2_rn(a01, make_float2(h.y, h.y), acc[1][0]);
      acc[1][1] = __ffma2_rn(a23, make_float2(h.y, h.y), acc[1][1]);
      acc[2][0] = __ffma2_rn(a01, make_float2(h.z, h.z), acc[2][0]);
      acc[2][1] = __ffma2_rn(a23, make_float2(h.z, h.z), acc[2][1]);
      acc[3][0] = __ffma2_rn(a01, make_float2(h.w, h.w), acc[3][0]);
      acc[3][1] = __ffma2_rn(a23, make_float2(h.w, h.w), acc[3][1]);
    }

    const int64_t row0 = tile * kRtRows + warp * 4;
    const int nrow = rows - row0 >= 4 ? 4 : int(rows - row0 > 0 ? rows - row0 : 0);
    const int64_t off0 = row0 * K + kcol;
    float tacc = 0.f, ymin = __int_as_float(0x7f800000), xmin = ymin;
    if (nrow == 4) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float xv[4] = {xc[i].x, xc[i].y, xc[i].z, xc[i].w};
        const float yv[4] = {acc[i][0].x, acc[i][0].y, acc[i][1].x, acc[i][1].y};
        float pw[4], qw[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          rt_weights<BK>(xv[j], yv[j], tk, pw[j], qw[j], tacc);
          ymin = fminf(ymin, yv[j]);
          xmin = fminf(xmin, xv[j]);
        }
        if (store) {
          const int64_t off = off0 + i * K;
          uint32_t h0, l0, h1, l1;
          rt_split_pair(pw[0], pw[1], h0, l0);
          rt_split_pair(pw[2], pw[3], h1, l1);
          *reinterpret_cast<uint2*>(pl0 + off) = make_uint2(h0, h1);
          *reinterpret_cast<uint2*>(pl1 + off) = make_uint2(l0, l1);
          if constexpr (BK != kBeta1) {
            rt_split_pair(qw[0], qw[1], h0, l0);
            rt_split_pair(qw[2], qw[3], h1, l1);
            *reinterpret_cast<uint2*>(pl2 + off) = make_uint2(h0, h1);
            *reinterpret_cast<uint2*>(pl3 + off) = make_uint2(l0, l1);
          }
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {  // ragged last tile
        if (i >= nrow) break;
        const float xv[4] = {xc[i].x, xc[i].y, xc[i].z, xc[i].w};
        const float yv[4] = {acc[i][0].x, acc[i][0].y, acc[i][1].x, acc[i][1].y};
        float pw[4], qw[4];
        for (int j = 0; j < 4; ++j) {
          rt_weights<BK>(xv[j], yv[j], tk, pw[j], qw[j], tacc);
          ymin = fminf(ymin, yv[j]);
          xmin = fminf(xmin, xv[j]);
        }
        if (store) {
          const int64_t off = off0 + i * K;
          uint32_t h0, l0, h1, l1;
          rt_split_pair(pw[0], pw[1], h0, l0);
          rt_split_pair(pw[2], pw[3], h1, l1);
          *reinterpret_cast<uint2*>(pl0 + off) = make_uint2(h0, h1);
          *reinterpret_cast<uint2*>(pl1 + off) = make_uint2(l0, l1);
          if constexpr (BK != kBeta1) {
            rt_split_pair(qw[0], qw[1], h0, l0);
            rt_split_pair(qw[2], qw[3], h1, l1);
            *reinterpret_cast<uint2*>(pl2 + off) = make_uint2(h0, h1);
            *reinterpret_cast<uint2*>(pl3 + off) = make_uint2(l0, l1);
          }
        }
      }
    }
    if (want_obj) {
      if (!(ymin >= tk.e) || !(xmin >= 0.f)) {
        // rare: clamped / non-positive model or negative data -- the exact
        // per-entry path (tc_weights), including the domain flags
        tacc = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (i >= nrow) break;
          const float xv[4] = {xc[i].x, xc[i].y, xc[i].z, xc[i].w};
          const float yv[4] = {acc[i][0].x, acc[i][0].y, acc[i][1].x, acc[i][1].y};
          for (int j = 0; j < 4; ++j) {
            float pv, qv;
            tc_weights<BK>(xv[j], yv[j], tk, pv, qv, true, tacc, bad);
          }
        }
        obj += double(tacc);
      } else {
        obj += double(tacc * oscale);
      }
    }
    store_h(buf ^ 1);
    __syncthreads();
  }
  if (want_obj) {
    obj = warp_sum(obj);
    if (lane == 0) red[warp] = obj;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < kRtThreads / 32; ++w) s += red[w];
      p.obj[blockIdx.x] = s;
    }
  }
  if (bad && p.flags) atomicOr(p.flags, bad);
}

}  // namespace ntfg
