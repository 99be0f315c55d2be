// K3 on the 5th-gen tensor cores (fp32 build): the mode-n contraction
//   G(k, r) = sum_{rows of unit} S(row, k) M(row, r)
// as a UMMA with A = S^T (M-dim = 128 columns k, K-dim = 16 rows, MN-major,
// TMA-loaded with the 128-byte swizzle straight from the row-major data),
// B = M (K-dim = 16 rows, N = rank, K-major, written by producer warps) and
// the fp32 accumulator in TMEM.
//
// Precision: the weight tensors P~/Q~ are stored by the reconstruction pass
// as two bf16 planes (hi = bf16(p), lo = bf16(p - hi), ~2^-17 relative) and
// M likewise, so three kind::f16 MMAs per tile (hi*hi + hi*lo + lo*hi)
// reproduce the fp32 products to ~1e-5 relative per term, unbiased; all
// cross-unit reductions stay fp64 (hard part 2).  Same 8 bytes
// per entry per pass as fp32 P~/Q~.
//
// Warp roles (320 threads): 0-3 build the B tiles (M rows, fp64 factor
// gathers one stage ahead), 4-7 epilogue (tcgen05.ld -> partials), 8 TMA
// producer, 9 TMEM allocator + single-thread MMA issuer.  Stages of 16 rows
// cycle through a 3-deep smem ring guarded by mbarriers (TMA tx, B-tile
// arrivals, tcgen05.commit); the TMEM accumulator is double-buffered across
// units when it fits so the epilogue of one unit overlaps the next.
#pragma once
#include <cuda_bf16.h>

#include "cp_kernels.cuh"
#include "stream3_kernels.cuh"
#include "tc_common.cuh"

namespace ntfg {

constexpr int kTcRows = 16;   // UMMA K for 16-bit inputs
constexpr int kTcStages = 3;

struct TcParams {
  Geom g;
  int n, R, RP, N;       // target mode, rank, partial stride, UMMA N (16/32/64)
  int ns, mt;            // streams, 128-column m-tiles (K / 128)
  int caseA;
  int64_t units, S, An, Bn;
  int64_t chunk;         // rows per unit (multiple of 16, case A) / j per split (case B)
  int boxB, boxA;        // TMA box for the 16 rows of a stage
  FastDiv fB;
  const double* mfac[2][kMaxOrder];
  const float* lastfac[2];   // case B: last-mode factor as [K][N] fp32, zero padded past R (G itself
                             // is an fp32 MMA result, so fp32 F adds ~6e-8 per term)
  float* partA;          // [ns][units][K][RP]
  double* partB;         // [ns][In][S][RP]
  int tmem_cols, dbuf;   // allocation, double-buffered accumulator?
  int ablate;            // perf experiments (NTFG_TC_ABLATE): 1 no B work, 2 no MMAs, 4 no epilogue work
  unsigned long long* trace;  // perf experiments: [cta][16 unit iterations][8] clock64 events (nullable)
};

struct TcMaps {
  CUtensorMap m[2][2];  // [stream][hi, lo]
};

template <int NMAX>
struct TcSmem {
  static constexpr size_t a_stream = size_t(2) * 4 * 2 * 2048;  // hi/lo x 4 m-tiles x 2 ko blocks (max)
  static constexpr size_t a_stage = 2 * a_stream;                // two streams
  static constexpr size_t b_tile = size_t(NMAX) * kTcRows * 2;   // one bf16 B tile
  static constexpr size_t b_stage = 2 * 2 * b_tile;               // [stream][hi, lo]
  static constexpr size_t stage = a_stage + b_stage;
  static constexpr size_t total = kTcStages * stage + 1024;       // + alignment slack
};

__device__ __forceinline__ void bf16_split(double v, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  const float f = float(v);
  hi = __float2bfloat16_rn(f);
  lo = __float2bfloat16_rn(f - __bfloat162float(hi));
}

template <int NMAX>
static __global__ void __launch_bounds__(320, 1)
    tc_contract_kernel(const __grid_constant__ TcMaps maps, const TcParams p) {
  using L = TcSmem<NMAX>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t a_full[kTcStages], b_full[kTcStages], empty[kTcStages], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;
  __shared__ double red[4][64];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t K = p.g.K;
  const int64_t In = p.g.dims[p.n];
  constexpr int N = NMAX;  // UMMA N (host launches the instance matching the rank)

  if (tid == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      tc::mbar_init(&a_full[s], 1);
      tc::mbar_init(&b_full[s], 128);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&acc_full[b], 1);
      tc::mbar_init(&acc_empty[b], 128);
    }
  }
  tc::fence_barrier_init();
  if (warp == 9) tc::tmem_alloc(&tmem_base, uint32_t(p.tmem_cols));
  if (warp == 8 && lane == 0)
    for (int s = 0; s < p.ns; ++s) {
      tc::prefetch_map(&maps.m[s][0]);
      tc::prefetch_map(&maps.m[s][1]);
    }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_base;
  const int cols_per_buf = p.ns * p.mt * N;

  auto unit_range = [&](int64_t u, int64_t& j0, int64_t& j1, int64_t& itgt, int64_t& split) {
    if (p.caseA) {
      itgt = 0;
      split = u;
      j0 = u * p.chunk;
      j1 = j0 + p.chunk < p.g.rows ? j0 + p.chunk : p.g.rows;
    } else {
      itgt = u / p.S;
      split = u % p.S;
      const int64_t tot = p.An * p.Bn;
      j0 = split * p.chunk;
      j1 = j0 + p.chunk < tot ? j0 + p.chunk : tot;
    }
  };
  auto row_of = [&](int64_t j, int64_t itgt) -> int64_t {
    if (p.caseA) return j;
    const int64_t aa = p.g.small_rows ? p.fB.div(j) : j / p.Bn;
    return aa * (In * p.Bn) + itgt * p.Bn + (j - aa * p.Bn);
  };
  auto stage_a = [&](int slot, int s, int plane) -> unsigned char* {
    return smem + size_t(slot) * L::stage + size_t(s) * L::a_stream + size_t(plane) * (L::a_stream / 2);
  };
  auto stage_b = [&](int slot, int s, int plane) -> unsigned char* {
    return smem + size_t(slot) * L::stage + L::a_stage + (size_t(s) * 2 + plane) * L::b_tile;
  };

  if (warp == 8) {
    // ================= TMA producer =================
    if (lane == 0) {
      uint32_t q = 0;
      const unsigned bytes = unsigned(p.ns) * 2u * unsigned(K / 64) * 2048u;
      for (int64_t u = blockIdx.x; u < p.units; u += gridDim.x) {
        int64_t j0, j1, itgt, split;
        unit_range(u, j0, j1, itgt, split);
        for (int64_t j = j0; j < j1; j += kTcRows, ++q) {
          const int slot = int(q % kTcStages);
          tc::wait(&empty[slot], ((q / kTcStages) & 1u) ^ 1u);
          tc::expect_tx(&a_full[slot], bytes);
          int c2, c3, c4;
          if (p.caseA) {
            c2 = int(j); c3 = 0; c4 = 0;
          } else {
            const int64_t aa = p.g.small_rows ? p.fB.div(j) : j / p.Bn;
            c2 = int(j - aa * p.Bn); c3 = int(itgt); c4 = int(aa);
          }
          for (int s = 0; s < p.ns; ++s)
            for (int plane = 0; plane < 2; ++plane)
              tc::tma_load_5d(stage_a(slot, s, plane), &maps.m[s][plane], 0, c2, c3, c4, 0, &a_full[slot]);
        }
      }
    }
  } else if (warp == 9) {
    // ================= MMA issuer =================
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_bf16_f32(128, N, true, false);
      uint32_t q = 0, it = 0;
      for (int64_t u = blockIdx.x; u < p.units; u += gridDim.x, ++it) {
        int64_t j0, j1, itgt, split;
        unit_range(u, j0, j1, itgt, split);
        const uint32_t tb = p.dbuf ? (it & 1u) : 0u;
        const uint32_t use = p.dbuf ? (it >> 1) : it;  // uses of this accumulator buffer so far
        unsigned long long* tr = (p.trace && it < 16) ? p.trace + (size_t(blockIdx.x) * 16 + it) * 8 : nullptr;
        if (tr) tr[2] = clock64();
        tc::wait(&acc_empty[tb], (use & 1u) ^ 1u);
        tc::fence_after_sync();
        if (tr) tr[3] = clock64();
        unsigned long long wa = 0, wb = 0;
        bool first = true;
        for (int64_t j = j0; j < j1; j += kTcRows, ++q) {
          const int slot = int(q % kTcStages);
          const uint32_t ph = (q / kTcStages) & 1u;
          unsigned long long t0 = tr ? clock64() : 0;
          tc::wait(&a_full[slot], ph);
          unsigned long long t1 = tr ? clock64() : 0;
          tc::wait(&b_full[slot], ph);
          if (tr) {
            wa += t1 - t0;
            wb += clock64() - t1;
          }
          tc::fence_after_sync();
          for (int s = 0; s < p.ns && !(p.ablate & 2); ++s) {
            const uint64_t bh = tc::desc_k_interleave(stage_b(slot, s, 0), 128, 256);
            const uint64_t bl = tc::desc_k_interleave(stage_b(slot, s, 1), 128, 256);
            for (int m = 0; m < p.mt; ++m) {
              const uint32_t d = tmem + tb * uint32_t(cols_per_buf) + uint32_t((s * p.mt + m) * N);
              const uint64_t ah = tc::desc_mn_sw128(stage_a(slot, s, 0) + size_t(m) * 4096, 2048, 1024);
              const uint64_t al = tc::desc_mn_sw128(stage_a(slot, s, 1) + size_t(m) * 4096, 2048, 1024);
              tc::mma_bf16(d, ah, bh, idesc, !first);
              tc::mma_bf16(d, ah, bl, idesc, true);
              tc::mma_bf16(d, al, bh, idesc, true);
            }
          }
          tc::commit(&empty[slot]);
          first = false;
        }
        tc::commit(&acc_full[tb]);
        if (tr) {
          tr[4] = wa;
          tr[5] = wb;
          tr[7] = clock64();
        }
      }
    }
  } else if (warp < 4) {
    // ================= B-tile (M rows) producers =================
    // thread t owns stage row k = t / 8 and rank columns [c*W, c*W + W),
    // c = t % 8: the row's coordinates are decoded once and each factor row
    // segment is a contiguous fp64 load; the gathers for the next stage are
    // issued before this stage's MMAs wait on them (one stage of slack).
    constexpr int W = N / 8;
    const int k = tid >> 3, r0 = (tid & 7) * W;
    const int nrm = p.g.order - 1;
    int mm[kMaxOrder];
    int nmm = 0;
    for (int m = 0; m < nrm; ++m)
      if (m != p.n) mm[nmm++] = m;
    double pv[2][3][W];
    auto gather = [&](int64_t j, int64_t j1, int64_t itgt) {
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int c2 = 0; c2 < 3; ++c2)
#pragma unroll
          for (int w = 0; w < W; ++w) pv[s][c2][w] = (c2 == 0 && j >= j1) ? 0.0 : 1.0;
      if (j >= j1) return;
      const int64_t row = row_of(j, itgt);
#pragma unroll
      for (int c2 = 0; c2 < 3; ++c2) {
        if (c2 >= nmm) break;
        const int64_t crd = p.g.coord(row, mm[c2]);
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          if (s >= p.ns) break;
          const double* f = p.mfac[s][mm[c2]] + crd * p.R + r0;
#pragma unroll
          for (int w = 0; w < W; ++w) pv[s][c2][w] = (r0 + w < p.R) ? __ldg(f + w) : 0.0;
        }
      }
    };
    uint32_t q = 0;
    for (int64_t u = blockIdx.x; u < p.units; u += gridDim.x) {
      int64_t j0, j1, itgt, split;
      unit_range(u, j0, j1, itgt, split);
      if (!(p.ablate & 1)) gather(j0 + k, j1, itgt);
      for (int64_t jb = j0; jb < j1; jb += kTcRows, ++q) {
        const int slot = int(q % kTcStages);
        tc::wait(&empty[slot], ((q / kTcStages) & 1u) ^ 1u);
        if (p.ablate & 1) {
          tc::arrive(&b_full[slot]);
          continue;
        }
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          if (s >= p.ns) break;
#pragma unroll
          for (int w = 0; w < W; ++w) {
            double v = pv[s][0][w] * pv[s][1][w] * pv[s][2][w];
            if (nmm > 3 && jb + k < j1 && r0 + w < p.R) {  // order > 5: remaining modes here
              const int64_t row = row_of(jb + k, itgt);
              for (int c2 = 3; c2 < nmm; ++c2) v *= p.mfac[s][mm[c2]][p.g.coord(row, mm[c2]) * p.R + r0 + w];
            }
            __nv_bfloat16 hi, lo;
            bf16_split(v, hi, lo);
            const int r = r0 + w;
            const size_t off = size_t(r / 8) * 256 + size_t(k / 8) * 128 + size_t(r % 8) * 16 + size_t(k % 8) * 2;
            *reinterpret_cast<__nv_bfloat16*>(stage_b(slot, s, 0) + off) = hi;
            *reinterpret_cast<__nv_bfloat16*>(stage_b(slot, s, 1) + off) = lo;
          }
        }
        tc::fence_proxy_async();
        tc::arrive(&b_full[slot]);
        if (jb + kTcRows < j1) gather(jb + kTcRows + k, j1, itgt);
      }
    }
  } else {
    // ================= epilogue (warps 4..7: TMEM lane quarter = warp % 4) =================
    const int quarter = warp & 3;
    const int et = tid - 128;  // 0..127
    // case B: out(r) = sum_k F_last(k, r) G(k, r) over this thread's k = m*128 +
    // 32*quarter + lane, in steps (stream s, column chunk c, m-tile m).  The
    // F_last values of a step do not depend on the accumulator, so they are
    // loaded one step ahead (16-byte loads of the padded [K][N] fp32 copy) and
    // the L2 round trip overlaps the previous step's TMEM read + FMAs.
    constexpr int CW = N < 32 ? N : 32;
    constexpr int NC = N / CW;
    constexpr int V4 = CW / 4;
    const int nsteps = p.ns * NC * p.mt;
    float4 cur[V4], nxt[V4];
    auto load_lf = [&](int step, float4(&dst)[V4]) {
      const int m = step % p.mt;
      const int c = (step / p.mt) % NC;
      const int s = step / (p.mt * NC);
      const int64_t k = int64_t(m) * 128 + quarter * 32 + lane;
      const float4* src = reinterpret_cast<const float4*>((s ? p.lastfac[1] : p.lastfac[0]) + k * N + c * CW);
#pragma unroll
      for (int j = 0; j < V4; ++j) dst[j] = __ldg(src + j);
    };
    if (!p.caseA) load_lf(0, cur);
    uint32_t it = 0;
    for (int64_t u = blockIdx.x; u < p.units; u += gridDim.x, ++it) {
      int64_t j0, j1, itgt, split;
      unit_range(u, j0, j1, itgt, split);
      const uint32_t tb = p.dbuf ? (it & 1u) : 0u;
      const uint32_t use = p.dbuf ? (it >> 1) : it;
      tc::wait(&acc_full[tb], use & 1u);
      tc::fence_after_sync();
      unsigned long long* tr = (p.trace && it < 16 && et == 0) ? p.trace + (size_t(blockIdx.x) * 16 + it) * 8 : nullptr;
      if (tr) tr[0] = clock64();
      const uint32_t tbase = tmem + (uint32_t(quarter * 32) << 16) + tb * uint32_t(cols_per_buf);
      if (p.ablate & 4) {
      } else if (p.caseA) {
        for (int s = 0; s < p.ns; ++s) {
          for (int m = 0; m < p.mt; ++m) {
            const int64_t k = int64_t(m) * 128 + quarter * 32 + lane;
#pragma unroll
            for (int c0 = 0; c0 < N; c0 += 32) {
              uint32_t v[32];
              tc::tmem_ld32(tbase + uint32_t((s * p.mt + m) * N + c0), v);
              // one 128-byte row segment per thread, 16-byte stores (columns
              // R..RP-1 carry the zero B columns' G = 0)
              float4* dst = reinterpret_cast<float4*>(p.partA + ((int64_t(s) * p.units + u) * K + k) * p.RP + c0);
#pragma unroll
              for (int r = 0; r < 32; r += 4)
                if (c0 + r < p.RP)
                  dst[r / 4] = make_float4(__uint_as_float(v[r]), __uint_as_float(v[r + 1]),
                                           __uint_as_float(v[r + 2]), __uint_as_float(v[r + 3]));
            }
          }
        }
      } else {
        float acc[CW];
        for (int step = 0; step < nsteps; ++step) {
          const int m = step % p.mt;
          const int c = (step / p.mt) % NC;
          const int s = step / (p.mt * NC);
          load_lf(step + 1 < nsteps ? step + 1 : 0, nxt);  // next step, or the next unit's first
          if (m == 0) {
#pragma unroll
            for (int r = 0; r < CW; ++r) acc[r] = 0.f;
          }
          uint32_t v[32];
          tc::tmem_ld32(tbase + uint32_t((s * p.mt + m) * N + c * CW), v);
          const float* f = reinterpret_cast<const float*>(cur);
          // fp32 over the <= 4 m-tiles of one k residue (G is an fp32 MMA
          // result; the cross-k and cross-unit sums below are fp64)
#pragma unroll
          for (int r = 0; r < CW; ++r) acc[r] = fmaf(__uint_as_float(v[r]), f[r], acc[r]);
          if (m == p.mt - 1) {
#pragma unroll
            for (int r = 0; r < CW; ++r) {
              const double w = warp_sum(double(acc[r]));
              if (lane == 0) red[quarter][c * CW + r] = w;
            }
            if (c == NC - 1) {
              named_sync(1, 128);
              if (et < p.R)
                p.partB[((int64_t(s) * In + itgt) * p.S + split) * p.RP + et] =
                    red[0][et] + red[1][et] + red[2][et] + red[3][et];
              named_sync(1, 128);
            }
          }
#pragma unroll
          for (int j = 0; j < V4; ++j) cur[j] = nxt[j];
        }
      }
      if (tr) tr[1] = clock64();
      tc::fence_before_sync();
      tc::arrive(&acc_empty[tb]);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 9) tc::tmem_dealloc(tmem, uint32_t(p.tmem_cols));
}

// [K][R] fp64 -> [K][N] fp32 zero padded, for the case-B epilogue's 16-byte loads
static __global__ void pad_last_kernel(const double* src, int64_t K, int R, int N, float* dst) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= K * N) return;
  const int64_t k = i / N;
  const int r = int(i % N);
  dst[i] = r < R ? float(src[k * R + r]) : 0.f;
}

// host P~/Q~ (fp64) -> bf16 hi/lo planes (step-level uploads).  The split is
// done in fp64 so that values produced as hi + lo by join_planes_kernel map
// back to the same (hi, lo) pair.
static __global__ void split_planes_kernel(const double* src, int64_t n, __nv_bfloat16* hi, __nv_bfloat16* lo) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    bf16_split_stable(float(src[i]), hi[i], lo[i]);
  }
}

static __global__ void join_planes_kernel(const __nv_bfloat16* hi, const __nv_bfloat16* lo, int64_t n, double* dst) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = double(__bfloat162float(hi[i])) + double(__bfloat162float(lo[i]));
}

}  // namespace ntfg
