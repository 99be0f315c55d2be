// K3 on the 5th-gen tensor cores (fp32 build): the mode-n contraction
//   G(k, r) = sum_{rows of unit} S(row, k) M(row, r)
// as a UMMA with A = S^T (M-dim = 128 columns k, K-dim = 16 rows, MN-major,
// TMA-loaded with the 128-byte swizzle straight from the row-major data),
// B = M (K-dim = 16 rows, N = rank, K-major) and the fp32 accumulator in TMEM.
//
// Precision: the weight tensors P~/Q~ are stored by the reconstruction pass
// as two bf16 planes (hi = bf16(p), lo = bf16(p - hi), ~2^-17 relative) and
// M likewise, so three kind::f16 MMAs per tile (hi*hi + hi*lo + lo*hi)
// reproduce the fp32 products to ~1e-5 relative per term, unbiased; all
// cross-unit reductions stay fp64 (hard part 2).  Same 8 bytes
// per entry per pass as fp32 P~/Q~.
//
// Two instances per rank width N (template flag SB):
//
// * SB = true, static B tiles (fast shapes: the fastest off-mode f has 128 | I_f).
//   M(row, r) = g(r) * A_f(c_f, r), with g (the slower off-modes' rows) constant
//   over a run of I_f rows.  The B operand of a stage is the bf16 hi/lo split of
//   16 rows of A_f alone, built once per launch in global memory in the tile
//   layout (stage_btiles_kernel) and bulk-copied per stage by the TMA warp; g
//   scales each finished accumulation segment in the epilogue (segments end at
//   run boundaries).  No per-stage producer work.
// * SB = false, generic: producer warps multiply the fp32 factor rows a gather
//   warp fetched with bulk async copies (`gdepth` stages ahead) and write the
//   hi/lo tiles per stage (272-byte stride between 8-column core-matrix groups,
//   so a warp's stores are conflict-free).
//
// Warp roles: [0, kB) B producers (SB: extra drain groups), kB..kB+3 epilogue
// (TMEM lane quarter = warp % 4), then TMA producer, MMA issuer (+ TMEM
// allocator), gather warp, second issuer (N <= 32).  The TMA and MMA warps run
// converged with warp-uniform operands and an elected lane (a single divergent
// issuing lane costs 150-350 cycles per MMA in compiler-generated operand
// marshalling, tools/mma_probe.cu).  Stages of 16 rows cycle through a smem
// ring (3-6 deep by budget) guarded by mbarriers (TMA tx, B arrivals,
// tcgen05.commit).
//
// Accumulation is segmented: a tile's TMEM accumulator restarts every p.seg
// stages and the epilogue adds the finished segment into running sums in a
// second TMEM region with CUDA-core FMAs -- long fp32 chains inside the tensor
// core truncate and drift (see the issuer).  One segment buffer, per-tile
// full/empty barriers; in SB mode the tiles of a segment are drained by
// several warp groups in parallel.
#pragma once
#include <cuda_bf16.h>

#include "cp_kernels.cuh"
#include "stream3_kernels.cuh"
#include "tc_common.cuh"

namespace ntfg {

constexpr int kTcRows = 16;     // UMMA K for 16-bit inputs
constexpr int kTcMaxStages = 6;
constexpr int kTcMaxGather = 6;
constexpr int kTcMaxTiles = 8;   // accumulator tiles per work item: ns * mtw
// MMA-issuing warps (9, and 11 when 2): one issuing thread was the stage-rate
// limit at N <= 32 (C2 K3 0.198 -> 0.189 ms); at N = 64 a second issuer gains
// nothing and its registers push the kernel into spills, so it stays at one
template <int N> __host__ __device__ constexpr int tc_issuers() { return N <= 32 ? 2 : 1; }
// B-producer warps: one (stream, k-group, rank) item per thread per stage at
// N = 64 (256 items).  A single warp per scheduler runs the ~300-instruction
// stage body at ~0.2 IPC (1300 of the 1456 cycles a C5 stage may take at HBM
// speed); two warps per scheduler hide each other's latencies.
template <int N> __host__ __device__ constexpr int tc_bwarps() { return N > 32 ? 8 : 4; }
template <int N> __host__ __device__ constexpr int tc_threads() { return 32 * (tc_bwarps<N>() + 7 + (tc_issuers<N>() - 1)); }
constexpr int kTcBSbo = 272;    // bytes between 8-column groups of a B tile (256 + 16: bank spread)
constexpr int kTcGModes = 3;    // factor modes gathered through the cp.async ring (more: direct fp64)
constexpr size_t kTcSmemMax = 227 * 1024 - 5120;  // dynamic budget (static smem 4.4 KB + 1 KB alignment slack)

// runtime shared-memory layout (host-computed, tc_layout)
struct TcLayout {
  uint32_t a_stream, a_stage;  // bytes of one stream's A planes / all streams (multiple of 1024)
  uint32_t b_tile;             // bytes of one bf16 B tile
  uint32_t b_off, ring_off;    // region offsets
  int nst, gdepth, gmodes;     // stages, gather ring depth, gathered modes
  uint32_t g_stream, g_slot;   // bytes of one stream's gather regions / one gather slot (all streams)

  uint32_t total;
};

struct TcParams {
  Geom g;
  int n, R, RP, N;       // target mode, rank, partial stride, UMMA N (16/32/64)
  int ns, mt;            // streams, 128-column m-tiles (K / 128)
  int mtw, G;            // m-tiles per work item, m-tile groups (mt = mtw * G)
  int seg;               // stages per TMEM accumulation segment
  int caseA;
  int64_t units, S, An, Bn;
  int64_t items;         // work items = units * G
  int64_t chunk;         // rows per unit (multiple of 16, case A) / j per split (case B)
  int boxB, boxA;        // TMA box for the 16 rows of a stage
  FastDiv fB;
  const double* mfac[2][kMaxOrder];
  const float* lastfac[2];   // case B: last-mode factor as [K][N] fp32, zero padded past R (G itself
                             // is an fp32 MMA result, so fp32 F adds ~6e-8 per term)
  const float* fac32[2][kMaxOrder];  // every factor as [I_m][N] fp32, zero padded (B operand gathers)
  int gfast;                          // stage rows = 16 consecutive rows of the fastest off-mode
  // static B tiles (sb): the B operand of a stage is the bf16 hi/lo split of 16 rows of the
  // fastest off-mode's factor alone -- built ONCE per launch in global memory in the tile
  // layout and bulk-copied per stage -- and the product g(r) of the other off-modes' rows,
  // constant over a run of I_f rows, scales the finished segment in the epilogue
  // (segments end at run boundaries).  No B-producer or gather work per stage.
  int sb, sb_runst, fmode;            // enabled, stages per run (I_f / 16), fastest off-mode
  unsigned char* btiles;              // [ns][I_f / 16][hi, lo][b_tile] (engine scratch)
  TcLayout lay;
  float* partA;          // [ns][units][K][RP]
  double* partB;         // [ns][In][S][RP]
  int tmem_cols;         // allocation (two segment buffers of ns * mtw * N columns)
  int ablate;            // perf experiments (NTFG_TC_ABLATE): 1 no B work, 2 no MMAs, 4 no epilogue work
  unsigned long long* trace;  // perf experiments: [cta][16 unit iterations][8] clock64 events (nullable)
};

struct TcMaps {
  CUtensorMap m[2][2];  // [stream][hi, lo]
};

// two values -> packed bf16 hi and lo (element a in the low half)
__device__ __forceinline__ void bf16_split_pair_fast(float a, float b, uint32_t& hi, uint32_t& lo) {
  hi = bf16x2_bits(__floats2bfloat162_rn(a, b));
  lo = bf16x2_bits(__floats2bfloat162_rn(a - bf16_lo_f(hi), b - bf16_hi_f(hi)));
}

__device__ __forceinline__ void bf16_split(double v, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  const float f = float(v);
  hi = __float2bfloat16_rn(f);
  lo = __float2bfloat16_rn(f - __bfloat162float(hi));
}

// every factor of every stream, [I_m][R] fp64 -> [I_m][N] fp32 zero padded:
// the B-operand gathers and the case-B epilogue's last factor (16-byte loads)
struct F32Stage {
  const double* src[2][kMaxOrder];
  float* dst[2][kMaxOrder];
  int64_t off[kMaxOrder + 1];  // cumulative I_m * N
  int order, ns, R, N;
};

// The kernel lives in its own translation unit (tc_contract.cu); the engine
// launches it through this entry point: ONE staging launch (fp32 factor copies
// and, in static-B mode, the B tiles), then the contraction.
void tc_contract_launch(int grid, cudaStream_t stream, const TcMaps& maps, const TcParams& p, const F32Stage& fs);

#ifdef NTFG_TC_CONTRACT_IMPL
// SB: static-B mode (TcParams::sb) as a compile-time flag, so each instance carries only its own
// roles' code (the generic producers / gather warp, or the TMA B copies and the drain groups)
template <int NMAX, bool SB>
static __global__ void __launch_bounds__(tc_threads<NMAX>(), 1)
    tc_contract_kernel(const __grid_constant__ TcMaps maps, const TcParams p) {
  // role wait counters (tools/tc_wstats.py): compiled in only with -DNTFG_TC_TRACE_BUILD, the
  // kernel is sensitive to its code size
#ifdef NTFG_TC_TRACE_BUILD
  const bool kTrace = p.trace != nullptr;
#else
  constexpr bool kTrace = false;
#endif
  const TcLayout& L = p.lay;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t a_full[kTcMaxStages], b_full[kTcMaxStages], empty[kTcMaxStages];
  __shared__ uint64_t acc_full[kTcMaxTiles], acc_empty[kTcMaxTiles];  // per accumulator tile (stream, m-tile)
  __shared__ uint64_t g_full[kTcMaxGather], g_empty[kTcMaxGather];
  __shared__ uint32_t tmem_base;
  __shared__ double red[4][128];
  // static-B mode: run scale g per (stream, rank), double-buffered by segment.  Aliases the start of
  // `red`: red is only touched in the per-item readout, which the drain groups' item barriers keep
  // apart from every segment drain (the only readers/writers of gsm).
  float (*gsm)[128] = reinterpret_cast<float (*)[128]>(&red[0][0]);

  // warp index through a shuffle: the compiler then treats the role branches
  // (and everything computed inside them from uniform inputs) as warp-uniform
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int64_t K = p.g.K;
  const int64_t In = p.g.dims[p.n];
  constexpr int N = NMAX;  // UMMA N (host launches the instance matching the rank)
  // warp roles: [0, kB) B producers, kB..kB+3 epilogue (TMEM lane quarter = warp % 4),
  // then TMA producer, MMA issuer (+ TMEM allocator), gather warp, second issuer
  constexpr int kB = tc_bwarps<NMAX>();
  constexpr int kWTma = kB + 4, kWMma = kB + 5, kWGather = kB + 6, kWMma2 = kB + 7;

  if (tid == 0) {
    for (int s = 0; s < L.nst; ++s) {
      tc::mbar_init(&a_full[s], 1);
      tc::mbar_init(&b_full[s], kB);    // one arrival per B-producer warp
      tc::mbar_init(&empty[s], tc_issuers<NMAX>());
    }
    for (int g = 0; g < L.gdepth; ++g) {
      tc::mbar_init(&g_full[g], 1);
      tc::mbar_init(&g_empty[g], kB);
    }
    for (int t = 0; t < kTcMaxTiles; ++t) {
      tc::mbar_init(&acc_full[t], 1);     // committed by the tile's issuer
      tc::mbar_init(&acc_empty[t], 4);  // drained by the epilogue warps
    }
  }
  tc::fence_barrier_init();
  if (warp == kWMma) tc::tmem_alloc(&tmem_base, uint32_t(p.tmem_cols));
  if (warp == kWTma && lane == 0)
    for (int s = 0; s < p.ns; ++s) {
      tc::prefetch_map(&maps.m[s][0]);
      tc::prefetch_map(&maps.m[s][1]);
    }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_base;
  const int cols_per_buf = p.ns * p.mtw * N;  // segment accumulators (<= 256 columns); the running sums follow

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
    return smem + size_t(slot) * L.a_stage + size_t(s) * L.a_stream + size_t(plane) * (L.a_stream / 2);
  };
  auto stage_b = [&](int slot, int s, int plane) -> unsigned char* {
    return smem + L.b_off + ((size_t(slot) * 2 + s) * 2 + plane) * L.b_tile;
  };

  unsigned long long ew_out = 0, ed_out = 0;
  // Drain groups (static-B mode): the idle B-producer warps form kB / 4 extra
  // groups of four warps (one per TMEM lane quarter) next to the epilogue
  // warps; group q drains the segment tiles t = q, q + ngroups, ...  A tile's
  // drain is ~1200 cycles of TMEM round trips, and the issuer cannot start a
  // tile's next segment before it is drained: draining the tiles in parallel
  // cut the issuer's wait from 14% of the launch.
  const int ngroups = SB ? 1 + kB / 4 : 1;
  const int ntile_all = p.ns * p.mtw;
  const uint32_t cols_run = uint32_t(cols_per_buf);
  // one segment tile into the running sums: run = (sg ? run : 0) + seg * g
  auto drain_tile = [&](int t, bool first, bool has_g, const float* gcur, uint32_t lanes_) {
    const uint32_t sbuf_ = tmem + lanes_, run_ = tmem + lanes_ + cols_run;
    const int gbase = (t / p.mtw) * N - t * N;  // column c * 16 + j of tile t -> entry (stream, rank)
    constexpr int CW = (N == 64) ? 32 : 16;  // columns per TMEM round trip (x32 only paid at N = 64, measured)
    for (int c = t * (N / CW); c < (t + 1) * (N / CW); ++c) {
      uint32_t v[CW], r[CW];
      if constexpr (CW == 32) {
        tc::tmem_ld32_nowait(sbuf_ + uint32_t(c * CW), v);
        if (!first) tc::tmem_ld32_nowait(run_ + uint32_t(c * CW), r);
      } else {
        tc::tmem_ld16_nowait(sbuf_ + uint32_t(c * CW), v);
        if (!first) tc::tmem_ld16_nowait(run_ + uint32_t(c * CW), r);
      }
      tc::tmem_ld_wait();
      if (has_g) {
        const float* gp = gcur + gbase + c * CW;
#pragma unroll
        for (int j = 0; j < CW; ++j)
          v[j] = __float_as_uint(!first ? fmaf(__uint_as_float(v[j]), gp[j], __uint_as_float(r[j]))
                                        : __uint_as_float(v[j]) * gp[j]);
      } else if (!first) {
#pragma unroll
        for (int j = 0; j < CW; ++j) v[j] = __float_as_uint(__uint_as_float(r[j]) + __uint_as_float(v[j]));
      }
      if constexpr (CW == 32) tc::tmem_st32(run_ + uint32_t(c * CW), v);
      else tc::tmem_st16(run_ + uint32_t(c * CW), v);
    }
  };
  if (warp == kWTma) {
    // ================= TMA producer =================
    // converged warp, one elected lane issues (uniform operands: no per-lane
    // operand marshalling around the TMA instructions)
    {
      int slot = 0;
      uint32_t sph = 1;  // producer parity: the first pass over the ring finds every slot free
      const unsigned bytes = unsigned(p.ns) * 2u * unsigned(2 * p.mtw) * 2048u;
      unsigned long long tw = 0, t00 = kTrace ? clock64() : 0;
      for (int64_t w = blockIdx.x; w < p.items; w += gridDim.x) {
        const int64_t u = w / p.G;
        const int blk0 = int(w % p.G) * 2 * p.mtw;  // first 64-column block of this item's m-tiles
        int64_t j0, j1, itgt, split;
        unit_range(u, j0, j1, itgt, split);
        int rblk = SB ? int((j0 / kTcRows) % p.sb_runst) : 0;  // 16-row block of the fastest off-mode
        for (int64_t j = j0; j < j1; j += kTcRows) {
          const unsigned long long tq = kTrace ? clock64() : 0;
          tc::wait(&empty[slot], sph);
          if (kTrace) tw += clock64() - tq;
          int c2, c3, c4;
          if (p.caseA) {
            c2 = int(j); c3 = 0; c4 = 0;
          } else {
            const int64_t aa = p.g.small_rows ? p.fB.div(j) : j / p.Bn;
            c2 = int(j - aa * p.Bn); c3 = int(itgt); c4 = int(aa);
          }
          if (tc::elect_one()) {
            tc::expect_tx(&a_full[slot], bytes + (SB ? unsigned(p.ns) * 2u * L.b_tile : 0u));
            for (int s = 0; s < p.ns; ++s)
              for (int plane = 0; plane < 2; ++plane)
                tc::tma_load_5d(stage_a(slot, s, plane), &maps.m[s][plane], 0, c2, c3, c4, blk0, &a_full[slot]);
            if constexpr (SB)  // this stage's 16 factor rows as ready-made hi/lo B tiles (adjacent in smem)
              for (int s = 0; s < p.ns; ++s)
                tma::bulk_g2s(stage_b(slot, s, 0), p.btiles + size_t((s * p.sb_runst + rblk) * 2) * L.b_tile,
                              2u * L.b_tile, &a_full[slot]);
          }
          __syncwarp();
          if (++rblk == p.sb_runst) rblk = 0;
          if (++slot == L.nst) {
            slot = 0;
            sph ^= 1u;
          }
        }
      }
      if (kTrace && lane == 0) {
        p.trace[size_t(gridDim.x) * 128 + blockIdx.x * 8 + 5] = tw;
        p.trace[size_t(gridDim.x) * 128 + blockIdx.x * 8 + 6] = clock64() - t00;
      }
    }
  } else if (warp == kWMma || (warp == kWMma2 && tc_issuers<NMAX>() > 1)) {
    // ================= MMA issuers =================
    // issuer i (first MMA warp: 0, second: 1) owns the accumulator tiles t = s * mtw + m
    // with t % 2 == i.  The accumulator of a tile restarts from zero every
    // p.seg stages (a "segment"); the epilogue adds each finished segment into
    // running sums (a second TMEM region) on the CUDA cores: long fp32
    // accumulation chains inside the tensor core drift low (measured: C2
    // beta = 1 factors 1.3e-3 off the fp64 build after 100 outer iterations
    // with 111-stage chains, 3.5e-5 with 16-stage chains), the CUDA-core sums
    // round to nearest.  One segment buffer: tile t's drain overlaps the last
    // stage's MMAs of tiles t+1.. (per-tile full/empty barriers).
    //
    // The whole warp runs this loop converged and every operand is a
    // warp-uniform value (kernel parameters, loop counters, the smem base), so
    // the MMAs issue from uniform registers; a single-lane (divergent) issuer
    // makes the compiler wrap every tcgen05.mma in an elect/R2UR loop, which
    // cost ~150 cycles per MMA against the 43 + N/2 the tensor pipe needs
    // (tools/mma_probe.cu).
    const int issuer = warp == kWMma ? 0 : 1;
    const uint32_t idesc = tc::idesc_bf16_f32(128, N, true, false);
    const int ntile = p.ns * p.mtw;
    const uint64_t a_desc0 = tc::desc_mn_sw128(smem, 2048, 1024);
    const uint64_t b_desc0 = tc::desc_k_interleave(smem + L.b_off, 128, kTcBSbo);
    const uint32_t a_plane16 = (L.a_stream / 2) >> 4, b_tile16 = L.b_tile >> 4;
    int slot = 0;
    uint32_t sph = 0, sc = 0;
    unsigned long long iw = 0;  // trace: cycles this issuer waited for segment drains
    for (int64_t w = blockIdx.x; w < p.items; w += gridDim.x) {
      int64_t j0, j1, itgt, split;
      unit_range(w / p.G, j0, j1, itgt, split);
      const int nstage = int((j1 - j0 + kTcRows - 1) / kTcRows);
      int qi = 0;
      int rblk = SB ? int((j0 / kTcRows) % p.sb_runst) : 0;
      for (int stg = 0; stg < nstage; ++stg) {
        const bool seg_first = qi == 0;
        const bool seg_last = qi == p.seg - 1 || stg == nstage - 1 || (SB && rblk == p.sb_runst - 1);
        if (++rblk == p.sb_runst) rblk = 0;
        tc::wait(&a_full[slot], sph);
        if constexpr (!SB) tc::wait(&b_full[slot], sph);
        tc::fence_after_sync();
        for (int t = issuer; t < ntile; t += tc_issuers<NMAX>()) {
          const int s = t >= p.mtw ? 1 : 0, m = t - s * p.mtw;
          if (seg_first) {  // the epilogue drained this tile's previous segment
            const unsigned long long tq = kTrace ? clock64() : 0;
            tc::wait(&acc_empty[t], (sc & 1u) ^ 1u);
            if (kTrace) iw += clock64() - tq;
            tc::fence_after_sync();
          }
          const uint32_t aoff = uint32_t(slot) * L.a_stage + uint32_t(s) * L.a_stream + uint32_t(m) * 4096u;
          const uint32_t boff = uint32_t((slot * 2 + s) * 2) * L.b_tile;
          const uint64_t ah = a_desc0 + (aoff >> 4), al = ah + a_plane16;
          const uint64_t bh = b_desc0 + (boff >> 4), bl = bh + b_tile16;
          const uint32_t d = tmem + uint32_t(t * N);
          if (tc::elect_one()) {
            if (!(p.ablate & 2)) {
              tc::mma_bf16(d, ah, bh, idesc, !seg_first);
              tc::mma_bf16(d, ah, bl, idesc, true);
              tc::mma_bf16(d, al, bh, idesc, true);
            }
            if (seg_last) tc::commit(&acc_full[t]);
          }
          __syncwarp();
        }
        if (tc::elect_one()) tc::commit(&empty[slot]);
        __syncwarp();
        if (++slot == L.nst) {
          slot = 0;
          sph ^= 1u;
        }
        if (seg_last) {
          ++sc;
          qi = 0;
        } else {
          ++qi;
        }
      }
    }
    if (kTrace && SB && lane == 0 && issuer == 0) p.trace[size_t(gridDim.x) * 128 + blockIdx.x * 8 + 2] = iw;
  } else if (warp == kWGather) {
    // ================= factor-row gathers (bulk async copies) =================
    // gather slot q % gdepth holds, per stream, gm regions of [16][N] floats.
    // Fast path (p.gfast: the fastest off-mode f has 16 | I_f, so a stage's 16
    // rows share every other coordinate and run over 16 consecutive rows of
    // A_f): region 0 = those 16 rows (one contiguous copy), region mi > 0 =
    // the single row of the mi-th other mode.  Otherwise one copy per
    // (row, mode); rows past the unit end copy the unit's last row (the B
    // threads zero them).
    const int nrm = p.g.order - 1;
    int mm[kMaxOrder];
    int nmm = 0;
    for (int m = 0; m < nrm; ++m)
      if (m != p.n) mm[nmm++] = m;
    const int gm = nmm < kTcGModes ? nmm : kTcGModes;
    const int fm = nmm > 0 ? mm[nmm - 1] : 0;  // fastest off-mode (highest index)
    const unsigned rowb = unsigned(N * 4);
    const unsigned regb = 16u * rowb;
    const unsigned bytes = p.gfast ? unsigned(p.ns) * (regb + unsigned(gm - 1) * rowb)
                                   : unsigned(16 * gm * p.ns) * rowb;
    unsigned char* ring = smem + L.ring_off;
    int gs = 0;
    uint32_t gph = 1;  // producer parity: the first pass finds every gather slot free
    unsigned long long gw = 0, g00 = kTrace ? clock64() : 0;
    if constexpr (!SB) if (gm > 0 && !(p.ablate & 1)) {
      for (int64_t w = blockIdx.x; w < p.items; w += gridDim.x) {
        int64_t j0, j1, itgt, split;
        unit_range(w / p.G, j0, j1, itgt, split);
        for (int64_t jb = j0; jb < j1; jb += kTcRows) {
          const unsigned long long tq = kTrace ? clock64() : 0;
          tc::wait(&g_empty[gs], gph);
          if (kTrace) gw += clock64() - tq;
          if (lane == 0) tc::expect_tx(&g_full[gs], bytes);
          __syncwarp();
          if (p.gfast) {
            if (lane < gm * p.ns) {
              const int mi = lane % gm, st = lane / gm;
              const int64_t row = row_of(jb, itgt);
              // compact fast-path slot: [16][N] rows of the fastest off-mode, then one row per other mode
              unsigned char* dst = ring + size_t(gs) * L.g_slot + size_t(st) * L.g_stream +
                                   (mi == 0 ? 0u : regb + unsigned(mi - 1) * rowb);
              if (mi == 0)
                tma::bulk_g2s(dst, p.fac32[st][fm] + p.g.coord(row, fm) * N, regb, &g_full[gs]);
              else
                tma::bulk_g2s(dst, p.fac32[st][mm[mi - 1]] + p.g.coord(row, mm[mi - 1]) * N, rowb, &g_full[gs]);
            }
          } else {
            for (int c = lane; c < 16 * gm * p.ns; c += 32) {
              const int kk = c & 15, mi = (c >> 4) % gm, st = (c >> 4) / gm;
              const int64_t j = jb + kk < j1 ? jb + kk : j1 - 1;
              const int64_t crd = p.g.coord(row_of(j, itgt), mm[mi]);
              unsigned char* dst = ring + size_t(gs) * L.g_slot + size_t(st) * L.g_stream + (size_t(mi) * 16 + kk) * rowb;
              tma::bulk_g2s(dst, p.fac32[st][mm[mi]] + crd * N, rowb, &g_full[gs]);
            }
          }
          if (++gs == L.gdepth) {
            gs = 0;
            gph ^= 1u;
          }
        }
      }
    }
    if (kTrace && lane == 0) {
      p.trace[size_t(gridDim.x) * 128 + blockIdx.x * 8 + 3] = gw;
      p.trace[size_t(gridDim.x) * 128 + blockIdx.x * 8 + 4] = clock64() - g00;
    }
  } else if (warp < kB) {
    // ================= B-tile (M rows) producers =================
    // work item = (stream s, k group kg of 8 stage rows, rank column r): the
    // 8 products M(8kg..8kg+7, r) are one 16-byte core-matrix row of the
    // K-major B tile, written as one st.shared.v4 per plane.  A warp covers
    // 32 consecutive r: ring reads and tile stores are conflict-free.  The
    // factor rows come from the gather ring (warp 10).
    const int nrm = p.g.order - 1;
    int mm[kMaxOrder];
    int nmm = 0;
    for (int m = 0; m < nrm; ++m)
      if (m != p.n) mm[nmm++] = m;
    const int gm = nmm < kTcGModes ? nmm : kTcGModes;
    const uint32_t ring = tc::saddr(smem + L.ring_off);
    const uint32_t btiles = tc::saddr(smem + L.b_off);
    const int nitems = p.ns * 2 * N;
    constexpr int kBT = kB * 32;                                  // B-producer threads
    constexpr int kMaxItems = (4 * N + kBT - 1) / kBT;            // ns * 2 * N items per stage
    int slot = -1, gs = -1;           // ring positions (advanced at the top of every stage)
    uint32_t sph = 0, gph = 1;        // sph: parity the slot's "empty" wait uses (ph ^ 1 trick); gph: gather "full" parity
    unsigned long long bw0 = 0, bw1 = 0, b00 = kTrace ? clock64() : 0;
    if constexpr (!SB) for (int64_t w = blockIdx.x; w < p.items; w += gridDim.x) {
      int64_t j0, j1, itgt, split;
      unit_range(w / p.G, j0, j1, itgt, split);
      for (int64_t jb = j0; jb < j1; jb += kTcRows) {
        if (++slot == L.nst) slot = 0;
        if (slot == 0) sph ^= 1u;    // first pass: 1 (slots start free)
        if (++gs == L.gdepth) gs = 0;
        if (gs == 0) gph ^= 1u;      // first pass: 0
        if (p.ablate & 1) {
          tc::wait(&empty[slot], sph);
          tc::warp_arrive(&b_full[slot], lane);
          continue;
        }
        const int nvalid = int(j1 - jb < kTcRows ? j1 - jb : kTcRows);
        unsigned long long tq = kTrace ? clock64() : 0;
        if (gm > 0) tc::wait(&g_full[gs], gph);
        if (kTrace) { bw0 += clock64() - tq; }
        uint4 hv[kMaxItems], lv[kMaxItems];
#pragma unroll
        for (int it = 0; it < kMaxItems; ++it) {
          const int i = tid + it * kBT;
          if (i >= nitems) break;
          const int r = i % N, kg = (i / N) & 1, st = i / (2 * N);
          float v[8];
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) v[kk] = 1.f;
          const uint32_t reg0 = ring + uint32_t(gs) * L.g_slot + uint32_t(st) * L.g_stream + uint32_t(r) * 4;
          if (p.gfast && gm > 0) {  // v = (prod of the other modes' rows, ascending) * A_f rows
            float g = 1.f;
            for (int mi = 1; mi < gm; ++mi) {
              const float f = tc::lds_f32(reg0 + 16u * uint32_t(N * 4) + uint32_t(mi - 1) * uint32_t(N * 4));
              g = mi == 1 ? f : g * f;
            }
            const uint32_t base = reg0 + uint32_t(kg * 8) * uint32_t(N * 4);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const float f = tc::lds_f32(base + uint32_t(kk) * uint32_t(N * 4));
              v[kk] = gm > 1 ? g * f : f;
            }
          } else {
            for (int mi = 0; mi < gm; ++mi) {
              const uint32_t base = reg0 + uint32_t(mi * 16 + kg * 8) * uint32_t(N * 4);
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) v[kk] *= tc::lds_f32(base + uint32_t(kk) * uint32_t(N * 4));
            }
          }
          if (nmm > kTcGModes) {  // order > 5: remaining modes straight from the fp64 factors
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              if (kg * 8 + kk >= nvalid) continue;
              const int64_t row = row_of(jb + kg * 8 + kk, itgt);
              for (int c2 = kTcGModes; c2 < nmm; ++c2)
                v[kk] = r < p.R ? float(double(v[kk]) * p.mfac[st][mm[c2]][p.g.coord(row, mm[c2]) * p.R + r]) : 0.f;
            }
          }
          if (nvalid < kTcRows) {  // last stage of a unit: rows past its end contribute nothing
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              if (kg * 8 + kk >= nvalid) v[kk] = 0.f;
          }
          uint32_t h[4], l[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) bf16_split_pair_fast(v[2 * e], v[2 * e + 1], h[e], l[e]);
          hv[it] = make_uint4(h[0], h[1], h[2], h[3]);
          lv[it] = make_uint4(l[0], l[1], l[2], l[3]);
        }
        if (gm > 0) tc::warp_arrive(&g_empty[gs], lane);
        tq = kTrace ? clock64() : 0;
        tc::wait(&empty[slot], sph);
        if (kTrace) { bw1 += clock64() - tq; }
#pragma unroll
        for (int it = 0; it < kMaxItems; ++it) {
          const int i = tid + it * kBT;
          if (i >= nitems) break;
          const int r = i % N, kg = (i / N) & 1, st = i / (2 * N);
          const uint32_t off = uint32_t(r / 8) * kTcBSbo + uint32_t(kg) * 128 + uint32_t(r % 8) * 16;
          const uint32_t tile = btiles + uint32_t((slot * 2 + st) * 2) * L.b_tile;
          tc::sts_v4(tile + off, hv[it]);
          tc::sts_v4(tile + L.b_tile + off, lv[it]);
        }
        tc::fence_proxy_async();
        tc::warp_arrive(&b_full[slot], lane);
      }
    }
    if constexpr (SB) {
      // ---- helper drain group (see drain_tile): warps 4q .. 4q+3 are group q + 1
      const int grp = 1 + warp / 4;
      const uint32_t lanes_ = uint32_t((warp & 3) * 32) << 16;
      int om_n = 0;
      for (int m = 0; m < nrm; ++m)
        if (m != p.n && m != p.fmode) ++om_n;
      const bool has_g = om_n > 0;
      uint32_t sc = 0;
      for (int64_t w = blockIdx.x; w < p.items; w += gridDim.x) {
        int64_t j0, j1, itgt, split;
        unit_range(w / p.G, j0, j1, itgt, split);
        const int nstage = int((j1 - j0 + kTcRows - 1) / kTcRows);
        int qi = 0, sg = 0;
        int rblk = int((j0 / kTcRows) % p.sb_runst);
        for (int stg = 0; stg < nstage; ++stg) {
          const bool seg_last = qi == p.seg - 1 || stg == nstage - 1 || rblk == p.sb_runst - 1;
          if (++rblk == p.sb_runst) rblk = 0;
          if (!seg_last) {
            ++qi;
            continue;
          }
          qi = 0;
          if (has_g) named_sync(3, 128 * ngroups);  // the epilogue group published this segment's g
          for (int t = grp; t < ntile_all; t += ngroups) {
            tc::wait(&acc_full[t], sc & 1u);
            tc::fence_after_sync();
            drain_tile(t, sg == 0, has_g, gsm[sc & 1u], lanes_);
            tc::fence_before_sync();
            tc::warp_arrive(&acc_empty[t], lane);
          }
          tc::tmem_st_wait();
          ++sc;
          ++sg;
        }
        // the epilogue group reads the running sums of every tile: after every group's
        // last drain (first barrier), and before anyone overwrites them (second barrier)
        tc::fence_before_sync();
        named_sync(3, 128 * ngroups);
        named_sync(3, 128 * ngroups);
        tc::fence_after_sync();
      }
    }
    if (kTrace && !SB && tid == 0) {
      p.trace[size_t(gridDim.x) * 128 + blockIdx.x * 8 + 0] = bw0;
      p.trace[size_t(gridDim.x) * 128 + blockIdx.x * 8 + 1] = bw1;
      p.trace[size_t(gridDim.x) * 128 + blockIdx.x * 8 + 2] = clock64() - b00;
    }
  } else {
    // ================= epilogue (warps 4..7: TMEM lane quarter = warp % 4) =================
    // Per segment: this thread's k row (lane) of the segment buffer is added
    // into a running-sum region of TMEM (columns cols_per_buf ..) with
    // CUDA-core fp32 adds (round to nearest; tcgen05.ld -> FADD -> tcgen05.st).
    // Per work item: case A writes the [K][RP] partial of its m-tile group;
    // case B dots G with the last-mode factor over k: out(r) = sum_k
    // F_last(k, r) G(k, r) (fp64 across k, m-tiles and units).
    const int quarter = warp & 3;
    const int et = tid - kB * 32;  // 0..127
    const int ntile = p.ns * p.mtw;
    const uint32_t lanes = uint32_t(quarter * 32) << 16;
    const uint32_t run = tmem + lanes + uint32_t(cols_per_buf);
    const uint32_t sbuf = tmem + lanes;
    // static-B mode: g(r) = product of the other off-modes' rows (ascending,
    // fp32) for the run a segment belongs to; thread et owns entry
    // (stream et / N, rank et % N), prefetched one segment ahead
    const int nrm = p.g.order - 1;
    int om[kMaxOrder];
    int nom = 0;  // off-modes other than the fastest one
    for (int m = 0; m < nrm; ++m)
      if (m != p.n && m != p.fmode) om[nom++] = m;
    const bool has_g = SB && nom > 0;
    auto g_of = [&](int64_t j, int64_t itgt) -> float {
      if (!has_g || et >= p.ns * N) return 1.f;
      const int s = et / N, r = et - s * N;
      const int64_t row = row_of(j, itgt);
      float gv = __ldg(p.fac32[s][om[0]] + p.g.coord(row, om[0]) * N + r);
      for (int q = 1; q < nom; ++q) gv *= __ldg(p.fac32[s][om[q]] + p.g.coord(row, om[q]) * N + r);
      return gv;
    };
    uint32_t sc = 0;
    unsigned long long ew = 0, ed = 0;  // trace: cycles waiting for a finished segment tile / draining it
    for (int64_t w = blockIdx.x; w < p.items; w += gridDim.x) {
      const int64_t u = w / p.G;
      const int g = int(w % p.G);
      int64_t j0, j1, itgt, split;
      unit_range(u, j0, j1, itgt, split);
      const int nstage = int((j1 - j0 + kTcRows - 1) / kTcRows);
      int qi = 0, sg = 0;
      int rblk = SB ? int((j0 / kTcRows) % p.sb_runst) : 0;
      float gnext = g_of(j0, itgt);
      for (int stg = 0; stg < nstage; ++stg) {
        const bool seg_last = qi == p.seg - 1 || stg == nstage - 1 || (SB && rblk == p.sb_runst - 1);
        if (++rblk == p.sb_runst) rblk = 0;
        if (!seg_last) {
          ++qi;
          continue;
        }
        qi = 0;
        const float* gcur = gsm[sc & 1u];
        if (has_g) {
          gsm[sc & 1u][et] = gnext;
          if (stg + 1 < nstage) gnext = g_of(j0 + int64_t(stg + 1) * kTcRows, itgt);  // next segment's run
          named_sync(ngroups > 1 ? 3 : 1, 128 * ngroups);
        }
        for (int t = 0; t < ntile; t += ngroups) {
          const unsigned long long tq0 = kTrace ? clock64() : 0;
          tc::wait(&acc_full[t], sc & 1u);
          tc::fence_after_sync();
          if (kTrace) {
            const unsigned long long tq1 = clock64();
            ew += tq1 - tq0;
            ed -= tq1;
          }
          if (!(p.ablate & 4)) drain_tile(t, sg == 0, has_g, gcur, lanes);
          tc::fence_before_sync();
          tc::warp_arrive(&acc_empty[t], lane);  // the segment tile is read: its next segment may start
          if (kTrace) ed += clock64();
        }
        tc::tmem_st_wait();
        ew_out = ew;
        ed_out = ed;
        ++sc;
        ++sg;
      }
      if (ngroups > 1) {  // every group's last drain of this item is in the running sums
        tc::fence_before_sync();
        named_sync(3, 128 * ngroups);
        tc::fence_after_sync();
      }
      if (p.ablate & 4) {
        if (ngroups > 1) named_sync(3, 128 * ngroups);
        continue;
      }
      if (p.caseA) {
        for (int t = 0; t < ntile; ++t) {
          const int s = t / p.mtw, m = t - s * p.mtw;
          const int64_t k = int64_t(g * p.mtw + m) * 128 + quarter * 32 + lane;
          // one row segment per thread, 16-byte stores (columns R..RP-1 carry
          // the zero B columns' G = 0)
          float4* dst = reinterpret_cast<float4*>(p.partA + ((int64_t(s) * p.units + u) * K + k) * p.RP);
          for (int c = 0; c < N; c += 16) {
            if (c >= p.RP) break;
            uint32_t v[16];
            tc::tmem_ld16_nowait(run + uint32_t(t * N + c), v);
            tc::tmem_ld_wait();
#pragma unroll
            for (int r = 0; r < 16; r += 4)
              if (c + r < p.RP)
                dst[(c + r) / 4] = make_float4(__uint_as_float(v[r]), __uint_as_float(v[r + 1]),
                                               __uint_as_float(v[r + 2]), __uint_as_float(v[r + 3]));
          }
        }
      } else {
        // per (stream, 16-column chunk): fp32 dot over this thread's k rows of
        // the item's m-tiles, then a transposing butterfly over the 32 lanes
        // (16 shuffles for 16 columns); lane l ends with column col(l)
        const int col = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
        for (int s = 0; s < p.ns; ++s) {
          for (int c = 0; c < N; c += 16) {
            float a[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) a[j] = 0.f;
            for (int m = 0; m < p.mtw; ++m) {
              const int t = s * p.mtw + m;
              const int64_t k = int64_t(g * p.mtw + m) * 128 + quarter * 32 + lane;
              const float4* f4 = reinterpret_cast<const float4*>((s ? p.lastfac[1] : p.lastfac[0]) + k * N + c);
              uint32_t v[16];
              tc::tmem_ld16_nowait(run + uint32_t(t * N + c), v);
              float f[16];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float4 q4 = __ldg(f4 + j);
                f[4 * j] = q4.x; f[4 * j + 1] = q4.y; f[4 * j + 2] = q4.z; f[4 * j + 3] = q4.w;
              }
              tc::tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 16; ++j) a[j] = fmaf(__uint_as_float(v[j]), f[j], a[j]);
            }
#pragma unroll
            for (int lvl = 0; lvl < 4; ++lvl) {
              const int msk = 16 >> lvl, half = 8 >> lvl;
              const bool upper = (lane & msk) != 0;
#pragma unroll
              for (int i = 0; i < half; ++i) {
                const float send = upper ? a[i] : a[i + half];
                const float keep = upper ? a[i + half] : a[i];
                a[i] = keep + __shfl_xor_sync(0xffffffffu, send, msk);
              }
            }
            a[0] += __shfl_xor_sync(0xffffffffu, a[0], 1);
            if ((lane & 1) == 0) red[quarter][s * N + c + col] = double(a[0]);
          }
        }
        named_sync(1, 128);
        if (et < p.ns * N) {
          const int s = et / N, r = et - s * N;
          if (r < p.R)
            p.partB[((int64_t(s) * In + itgt) * (p.S * p.G) + split * p.G + g) * p.RP + r] =
                red[0][et] + red[1][et] + red[2][et] + red[3][et];
        }
        named_sync(1, 128);
      }
      if (ngroups > 1) {  // running sums read: the groups may start the next item's first segment
        tc::fence_before_sync();
        named_sync(3, 128 * ngroups);
      }
    }
  }
  if (kTrace && SB && tid == kB * 32) {  // static-B mode: the B counters' slots carry the epilogue's
    p.trace[size_t(gridDim.x) * 128 + blockIdx.x * 8 + 0] = ew_out;
    p.trace[size_t(gridDim.x) * 128 + blockIdx.x * 8 + 1] = ed_out;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == kWMma) tc::tmem_dealloc(tmem, uint32_t(p.tmem_cols));
}

#endif  // NTFG_TC_CONTRACT_IMPL

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
