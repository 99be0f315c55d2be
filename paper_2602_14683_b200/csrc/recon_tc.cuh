// K2/K5 on the 5th-gen tensor cores (fp32 build): reconstruction + weights +
// objective with Xhat as a UMMA (reference cp_reconstruct cp.cpp:26-76 fused
// with weight_entries kernels.hpp:30-66 and d_beta divergence.cpp:16-44).
//
//   Xhat(row, k) = sum_r H(row, r) A_last(k, r),   H(row, r) = prod_{m<N-1} A_m(i_m(row), r)
//
// D[M = 128 k-columns (TMEM lanes)] x [N = 128 rows (TMEM columns)] =
// A_last tile (128 x R, K-major) * H tile^T (128 x R, K-major), K = R.
// fp32 accuracy from three kind::tf32 MMAs per 8 ranks: both operands are
// split into tf32 hi + lo (hi = RN_tf32(v), lo = RN_tf32(v - hi)) and
// hi*hi + hi*lo + lo*hi is accumulated in the fp32 TMEM accumulator: the
// dropped lo*lo term and the lo roundings are ~2^-22 relative, the same size as
// the rounding of a 64-term fp32 FMA chain.
//
// One persistent CTA per SM owns one 128-column tile of the last factor (its
// tf32 planes stay in shared memory) and walks 128-row tiles of X:
//   warps 16-18  build the H tile of the next row tile (fp64 product in the
//                reference order, then tf32 hi/lo planes in the no-swizzle
//                K-major core-matrix layout), two stages;
//   warp 19      TMEM allocator + MMA issuer (converged warp, elected lane);
//   warps 0-15   epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31 (its k
//                columns) and accumulator columns 32 (w / 4) .. +31 (32 rows),
//                so every global access of a warp is one contiguous run along
//                k: X is read with 128-byte requests (prefetched one tile
//                ahead in registers) and the four bf16 hi/lo planes of P~/Q~
//                are written with 64-byte requests.  Weights, bf16 splits and
//                the objective term are recon_tile.cuh's (identical formulas).
// The accumulator is double-buffered (2 x 128 TMEM columns), so the MMAs of
// tile i+1 overlap the epilogue of tile i.
//
// Eligible when the fastest row mode has 128 | I (a tile's rows then share the
// slower coordinates and run over 128 consecutive rows of that factor: one
// contiguous block) and K is a multiple of 128 up to 512; everything else
// stays on recon_tile_kernel.  With a row table (p.htab, the Tucker partial
// chain Y(row, j), tensor.cpp:408-419) H is that table and 128 | rows suffices.
// Outputs: bf16 hi/lo planes (tensor-core K3), fp32 P/Q arrays (CUDA-core
// contraction paths and the Tucker engine), or the objective only.
#pragma once
#include "recon_tile.cuh"
#include "tc_common.cuh"

namespace ntfg {

constexpr int kRcRows = 128;      // X rows per tile (UMMA N)
constexpr int kRcCols = 128;      // k columns per CTA (UMMA M)
constexpr int kRcEpiWarps = 16;
constexpr int kRcProdWarps = 3;       // 20 warps in all: 96 registers per thread
constexpr int kRcThreads = (kRcEpiWarps + kRcProdWarps + 1) * 32;  // 640
// bytes between K-adjacent core matrices (8 rows x 16 B): 128 + 16 so the
// scalar H stores of a warp (consecutive ranks) spread over all banks
constexpr int kRcLbo = 144;

__host__ __device__ inline uint32_t rc_sbo(int RP) { return uint32_t(RP / 4) * kRcLbo; }      // between 8-row groups
__host__ __device__ inline uint32_t rc_plane(int RP) { return 16u * rc_sbo(RP); }             // one 128 x RP tf32 plane
constexpr int kRcMaxStages = 4;
// H stages (2..4) that fit next to the A planes: 2 at R = 64, 4 below (a deeper ring absorbs the
// producers' latency jitter; the accumulator stays double-buffered)
inline int rc_stages(int RP) {
  const int planes = int((size_t(232448) - 1536 - 128) / rc_plane(RP));
  const int nh = (planes - 2) / 2;
  return nh < 2 ? 2 : nh > kRcMaxStages ? kRcMaxStages : nh;
}
inline size_t rc_smem(int RP) { return size_t(2 + 2 * rc_stages(RP)) * rc_plane(RP) + 128; }  // A hi/lo + NH stages of H hi/lo

// the launcher lives in recon_tc.cu (own translation unit)
void recon_tc_launch(int grid, cudaStream_t stream, const ReconParams<float>& p, int RP, int bk);

#ifdef NTFG_RECON_TC_IMPL

__device__ __forceinline__ uint32_t tf32_rna(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         bool accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(uint32_t(accumulate)));
}
// instruction descriptor kind::tf32: D f32, A/B tf32, both K-major, N>>3, M>>4
__host__ __device__ constexpr uint32_t idesc_tf32_f32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ void sts_b32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.b32 [%0], %1;\n" ::"r"(a), "r"(v) : "memory");
}

// HV: H source of the producers -- 0 scalar fp64 (R % 4 != 0), 1 fp64 rows in 32-byte chunks,
// 2 fp32 staged rows in 16-byte chunks.  A template parameter (like BK, KC) so an instance carries
// one variant: this kernel is sensitive to its code size (a run-time choice between two split
// routines in the unrolled epilogue cost 10%).
template <int BK, int KC, int HV>
static __global__ void __launch_bounds__(kRcThreads, 1) recon_tc_kernel(const ReconParams<float> p, const int RP,
                                                                        const int NH) {
  constexpr int64_t K = int64_t(KC) * kRcCols;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  __shared__ uint64_t h_full[kRcMaxStages], h_empty[kRcMaxStages], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(16) double gs[2][64];
  __shared__ double red[kRcEpiWarps];

  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);  // warp-uniform role branches
  const int R = p.R;
  const uint32_t sbo = rc_sbo(RP), plane = rc_plane(RP);
  const int kt = int(blockIdx.x % KC);
  const int64_t tstride = gridDim.x / KC;
  const int64_t ntiles = p.g.rows / kRcRows;  // exact on this path (128 | I of the fastest row mode)
  const int64_t kbase = int64_t(kt) * kRcCols;
  const int64_t tile0 = blockIdx.x / KC;

  if (tid == 0) {
    for (int b = 0; b < kRcMaxStages; ++b) {
      tc::mbar_init(&h_full[b], kRcProdWarps);  // one arrival per warp
      tc::mbar_init(&h_empty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&acc_full[b], 1);
      tc::mbar_init(&acc_empty[b], kRcEpiWarps);
    }
  }
  tc::fence_barrier_init();
  if (warp == kRcEpiWarps + kRcProdWarps) tc::tmem_alloc(&tmem_base, 256);
  {
    // last-factor tile as tf32 hi/lo planes; H stages zeroed (rank padding
    // columns r >= R are never written again and must contribute 0)
    const uint32_t a_hi = tc::saddr(smem), a_lo = a_hi + plane;
    int rsh = 3;
    while ((1 << rsh) < RP) ++rsh;
    for (int i = tid; i < kRcCols * RP; i += kRcThreads) {
      const int kk = i >> rsh, r = i & (RP - 1);
      const float v = p.alast[(kbase + kk) * RP + r];
      const uint32_t hi = tf32_rna(v);
      const uint32_t lo = tf32_rna(v - __uint_as_float(hi));
      const uint32_t off = uint32_t(kk >> 3) * sbo + uint32_t(r >> 2) * kRcLbo + uint32_t(kk & 7) * 16u + uint32_t(r & 3) * 4u;
      sts_b32(a_hi + off, hi);
      sts_b32(a_lo + off, lo);
    }
    uint4* hz = reinterpret_cast<uint4*>(smem + 2 * size_t(plane));
    for (int i = tid; i < int(2 * NH * plane / 16); i += kRcThreads) hz[i] = make_uint4(0u, 0u, 0u, 0u);
    tc::fence_proxy_async();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_base;

  double obj = 0.0;
  unsigned bad = 0;

  if (warp == kRcEpiWarps + kRcProdWarps) {
    // ================= MMA issuer (converged warp, uniform operands) =================
    const uint32_t idesc = idesc_tf32_f32(kRcCols, kRcRows);
    const uint64_t a_hi = tc::desc_k_interleave(smem, kRcLbo, sbo);
    const uint64_t a_lo = a_hi + (plane >> 4);
    const uint64_t h0 = tc::desc_k_interleave(smem + 2 * size_t(plane), kRcLbo, sbo);
    const int ksteps = RP / 8;
    uint32_t i = 0;
    int hs = 0;        // H stage ring position / parity
    uint32_t hph = 0;
    for (int64_t tile = tile0; tile < ntiles; tile += tstride, ++i) {
      const uint32_t st = i & 1u, ph = (i >> 1) & 1u;  // accumulator buffer / parity
      tc::wait(&h_full[hs], hph);
      tc::wait(&acc_empty[st], ph ^ 1u);
      tc::fence_after_sync();
      const uint64_t b_hi = h0 + uint64_t(hs) * (2u * plane >> 4);
      const uint64_t b_lo = b_hi + (plane >> 4);
      const uint32_t d = tmem + st * uint32_t(kRcRows);
      if (tc::elect_one()) {
        for (int ks = 0; ks < ksteps; ++ks) {
          const uint64_t ko = uint64_t(ks) * (2u * kRcLbo >> 4);
          mma_tf32(d, a_hi + ko, b_hi + ko, idesc, ks > 0);
          mma_tf32(d, a_hi + ko, b_lo + ko, idesc, true);
          mma_tf32(d, a_lo + ko, b_hi + ko, idesc, true);
        }
        tc::commit(&h_empty[hs]);
        tc::commit(&acc_full[st]);
      }
      __syncwarp();
      if (++hs == NH) {
        hs = 0;
        hph ^= 1u;
      }
    }
  } else if (warp >= kRcEpiWarps) {
    // ================= H producers =================
    constexpr int PT = kRcProdWarps * 32;
    const int pt = tid - kRcEpiWarps * 32;  // 0..PT-1
    const int npre = p.htab ? 1 : p.g.order - 1;  // row table: H is read as is
    const int f = p.g.order - 2;                    // fastest row mode
    const int rstep = PT % R, rowstep = PT / R;
    const int nel = kRcRows * R;
    const uint32_t hbase = tc::saddr(smem) + 2u * plane;
    uint32_t i = 0;
    int hs = 0;
    uint32_t hph = 1;  // producer parity: the first pass over the ring finds every stage free
    for (int64_t tile = tile0; tile < ntiles; tile += tstride, ++i) {
      const uint32_t st = i & 1u;  // G buffer (guarded by the per-tile producer barrier)
      tc::wait(&h_empty[hs], hph);
      const int64_t row0 = tile * kRcRows;
      if (npre >= 2 && pt < R) {  // product of the slower modes' rows, reference order
        double g = p.fac[0][p.g.coord(row0, 0) * R + pt];
        for (int m = 1; m < f; ++m) g *= p.fac[m][p.g.coord(row0, m) * R + pt];
        gs[st][pt] = g;
      }
      named_sync(2, kRcProdWarps * 32);
      // H rows of the tile: 128 consecutive rows of the fastest row mode's
      // factor, or (Tucker partial chain) of the row table itself
      const double* hsrc = p.htab ? p.htab + row0 * R : p.fac[f] + p.g.coord(row0, f) * R;
      const uint32_t hhi = hbase + uint32_t(hs) * 2u * plane, hlo = hhi + plane;
      if constexpr (HV == 2) {
        // fp32 staged factor: one 16-byte load per item, fp32 product with the
        // (fp64-accumulated, then rounded) slower-mode product G
        const int R4 = R >> 2;
        const int kstep = PT % R4, rowstep4 = PT / R4, nchunk = kRcRows * R4;
        const float4* fr = reinterpret_cast<const float4*>(p.hfac32 + p.g.coord(row0, f) * R);
        int row = pt / R4, kc = pt - row * R4;
#pragma unroll 4
        for (int c = pt; c < nchunk; c += PT) {
          const float4 v4 = __ldg(fr + c);
          float v[4] = {v4.x, v4.y, v4.z, v4.w};
          if (npre >= 2) {
            const double2 g01 = *reinterpret_cast<const double2*>(&gs[st][4 * kc]);
            const double2 g23 = *reinterpret_cast<const double2*>(&gs[st][4 * kc + 2]);
            v[0] *= float(g01.x); v[1] *= float(g01.y); v[2] *= float(g23.x); v[3] *= float(g23.y);
          }
          uint32_t hi[4], lo[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            hi[e] = tf32_rna(v[e]);
            lo[e] = tf32_rna(v[e] - __uint_as_float(hi[e]));
          }
          const uint32_t off = uint32_t(row >> 3) * sbo + uint32_t(kc) * kRcLbo + uint32_t(row & 7) * 16u;
          tc::sts_v4(hhi + off, make_uint4(hi[0], hi[1], hi[2], hi[3]));
          tc::sts_v4(hlo + off, make_uint4(lo[0], lo[1], lo[2], lo[3]));
          kc += kstep;
          row += rowstep4;
          if (kc >= R4) {
            kc -= R4;
            ++row;
          }
        }
      } else if constexpr (HV == 1) {
        // four consecutive ranks of one row per item: 32-byte loads (a warp
        // reads 1 KB contiguous), one 16-byte store per plane (conflict-free
        // with the 144-byte core-matrix stride), one address per four values
        const int R4 = R >> 2;
        const int kstep = PT % R4, rowstep4 = PT / R4, nchunk = kRcRows * R4;
        const double2* fr = reinterpret_cast<const double2*>(hsrc);
        int row = pt / R4, kc = pt - row * R4;
#pragma unroll 4
        for (int c = pt; c < nchunk; c += PT) {
          const double2 v01 = __ldg(fr + 2 * c), v23 = __ldg(fr + 2 * c + 1);
          double v[4] = {v01.x, v01.y, v23.x, v23.y};
          if (npre >= 2) {
            const double2 g01 = *reinterpret_cast<const double2*>(&gs[st][4 * kc]);
            const double2 g23 = *reinterpret_cast<const double2*>(&gs[st][4 * kc + 2]);
            v[0] *= g01.x; v[1] *= g01.y; v[2] *= g23.x; v[3] *= g23.y;
          }
          uint32_t hi[4], lo[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float h = float(v[e]);
            hi[e] = tf32_rna(h);
            lo[e] = tf32_rna(h - __uint_as_float(hi[e]));
          }
          const uint32_t off = uint32_t(row >> 3) * sbo + uint32_t(kc) * kRcLbo + uint32_t(row & 7) * 16u;
          tc::sts_v4(hhi + off, make_uint4(hi[0], hi[1], hi[2], hi[3]));
          tc::sts_v4(hlo + off, make_uint4(lo[0], lo[1], lo[2], lo[3]));
          kc += kstep;
          row += rowstep4;
          if (kc >= R4) {
            kc -= R4;
            ++row;
          }
        }
      } else {
        const double* fr = hsrc + pt;
        int row = pt / R, r = pt - row * R;
#pragma unroll 8
        for (int e = pt; e < nel; e += PT) {
          const double v = fr[e - pt];
          const float h = float(npre >= 2 ? gs[st][r] * v : v);
          const uint32_t hi = tf32_rna(h);
          const uint32_t lo = tf32_rna(h - __uint_as_float(hi));
          const uint32_t off = uint32_t(row >> 3) * sbo + uint32_t(r >> 2) * kRcLbo + uint32_t(row & 7) * 16u + uint32_t(r & 3) * 4u;
          sts_b32(hhi + off, hi);
          sts_b32(hlo + off, lo);
          r += rstep;
          row += rowstep;
          if (r >= R) {
            r -= R;
            ++row;
          }
        }
      }
      tc::fence_proxy_async();
      tc::warp_arrive(&h_full[hs], lane);
      if (++hs == NH) {
        hs = 0;
        hph ^= 1u;
      }
    }
  } else {
    // ================= epilogue =================
    const int quarter = warp & 3, chunk = warp >> 2;
    TailConst tk;
    tk.e = float(p.eps);
    tk.b = float(p.beta);
    tk.b1 = float(p.beta - 1.0);
    tk.b2 = float(p.beta - 2.0);
    tk.ib = float(1.0 / (p.beta * (p.beta - 1.0)));
    const float oscale = rt_obj_scale<BK>(tk);
    const bool want_obj = p.obj != nullptr;
    const bool store = p.planes[0] != nullptr;
    float* const pout32 = p.pout;
    float* const qout32 = p.qout;
    unsigned short* const pl0 = static_cast<unsigned short*>(p.planes[0]);
    unsigned short* const pl1 = static_cast<unsigned short*>(p.planes[1]);
    unsigned short* const pl2 = static_cast<unsigned short*>(p.planes[2]);
    unsigned short* const pl3 = static_cast<unsigned short*>(p.planes[3]);
    const int64_t tile_step = tstride * kRcRows * K;
    int64_t ob = (tile0 * kRcRows + chunk * 32) * K + kbase + quarter * 32 + lane;  // (row, k) of this thread's first entry
    float xr[32];
    if (tile0 < ntiles) {
#pragma unroll
      for (int j = 0; j < 32; ++j) xr[j] = __ldg(p.x + ob + j * K);
    }
    uint32_t i = 0;
    for (int64_t tile = tile0; tile < ntiles; tile += tstride, ++i, ob += tile_step) {
      const uint32_t st = i & 1u;
      const bool hasn = tile + tstride < ntiles;
      const float* xn = p.x + ob + tile_step;
      tc::wait(&acc_full[st], (i >> 1) & 1u);
      tc::fence_after_sync();
      const uint32_t taddr = tmem + (uint32_t(quarter * 32) << 16) + st * uint32_t(kRcRows) + uint32_t(chunk * 32);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t yv[16];
        tc::tmem_ld16_nowait(taddr + uint32_t(half * 16), yv);
        tc::tmem_ld_wait();
        if (half == 1) {  // accumulator read: the MMAs of tile i + 2 may overwrite it
          tc::fence_before_sync();
          tc::warp_arrive(&acc_empty[st], lane);
        }
#pragma unroll
        for (int sub = 0; sub < 2; ++sub) {
          const int j0 = half * 16 + sub * 8;
          float pw[8], qw[8];
          float tacc = 0.f, ymin = __int_as_float(0x7f800000), xmin = ymin;
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            const float x = xr[j0 + jj], y = __uint_as_float(yv[sub * 8 + jj]);
            rt_weights<BK>(x, y, tk, pw[jj], qw[jj], tacc);
            ymin = fminf(ymin, y);
            xmin = fminf(xmin, x);
          }
          if (pout32) {  // fp32 P/Q arrays (CUDA-core contraction paths, Tucker): 128-byte rows per warp
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              const int64_t o = ob + (j0 + jj) * K;
              pout32[o] = pw[jj];
              if (qout32) qout32[o] = qw[jj];
            }
          }
          if (store) {
#pragma unroll
            for (int jj = 0; jj < 8; jj += 2) {
              const int64_t o0 = ob + (j0 + jj) * K, o1 = o0 + K;
              uint32_t h, l;
              rt_split_pair(pw[jj], pw[jj + 1], h, l);
              pl0[o0] = (unsigned short)(h & 0xffffu);
              pl0[o1] = (unsigned short)(h >> 16);
              pl1[o0] = (unsigned short)(l & 0xffffu);
              pl1[o1] = (unsigned short)(l >> 16);
              if constexpr (BK != kBeta1) {
                rt_split_pair(qw[jj], qw[jj + 1], h, l);
                pl2[o0] = (unsigned short)(h & 0xffffu);
                pl2[o1] = (unsigned short)(h >> 16);
                pl3[o0] = (unsigned short)(l & 0xffffu);
                pl3[o1] = (unsigned short)(l >> 16);
              }
            }
          }
          if (want_obj) {
            if (!(ymin >= tk.e) || !(xmin >= 0.f)) {
              // rare: clamped / non-positive model or negative data -- the exact
              // per-entry path (tc_weights), including the domain flags
              tacc = 0.f;
#pragma unroll
              for (int jj = 0; jj < 8; ++jj) {
                float pv, qv;
                tc_weights<BK>(xr[j0 + jj], __uint_as_float(yv[sub * 8 + jj]), tk, pv, qv, true, tacc, bad);
              }
              obj += double(tacc);
            } else {
              obj += double(tacc * oscale);
            }
          }
          if (hasn) {  // this tile's x values are consumed: prefetch the next tile's into the same registers
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) xr[j0 + jj] = __ldg(xn + (j0 + jj) * K);
          }
        }
      }
    }
    if (want_obj) {
      obj = warp_sum(obj);
      if (lane == 0) red[warp] = obj;
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (tid == 0 && p.obj != nullptr) {
    double s = 0.0;
    for (int w = 0; w < kRcEpiWarps; ++w) s += red[w];
    p.obj[blockIdx.x] = s;
  }
  if (bad && p.flags) atomicOr(p.flags, bad);
  if (warp == kRcEpiWarps + kRcProdWarps) tc::tmem_dealloc(tmem, 256);
}

#endif  // NTFG_RECON_TC_IMPL

}  // namespace ntfg
