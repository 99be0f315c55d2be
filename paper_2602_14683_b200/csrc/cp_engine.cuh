// CP engine: device state of one CP problem and the B-CoMM / J-CoMM steps.
//
// Reference call stacks:
//   bcomm_block_update  cp.cpp:109-129  = recon(P,Q) -> contract -> finalize
//   make_jcomm_reference cp.cpp:202-208 = recon(P~,Q~) (+ fused objective)
//   jcomm_inner_update  cp.cpp:210-229  = contract(P~ chi1, Q~ chi2) -> finalize
// The whole outer iteration is enqueued on one stream and (optionally)
// captured once into a CUDA graph by the fit driver.
#pragma once
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "coo_ingest.cuh"
#include "coo_kernels.cuh"
#include "cp_kernels.cuh"
#include "engine.cuh"
#include "nccl_comm.cuh"
#include "stream3_kernels.cuh"
#include "recon_tile.cuh"
#include "recon_tc.cuh"
#include "tc_contract.cuh"

namespace ntfg {

template <typename T>
class CpEngine {
 public:
  // dims: this rank's extents (dims[0] = slab rows when sharded).
  CpEngine(Context& c, uint32_t order, const uint64_t* dims, int64_t rank, double beta,
           double eps, const ntfg_shard* shard)
      : c_(c), N_(int(order)), R_(rank), beta_(beta), eps_(eps) {
    if (order < 1 || order > uint32_t(kMaxOrder))
      throw Error(NTFG_ERR_SHAPE, "tensor order must be in [1, 8]");
    if (rank < 1) throw Error(NTFG_ERR_DOMAIN, "rank must be >= 1");
    RP_ = pad_rank(rank);
    gamma_ = gamma_of(beta);
    bk_ = beta_kind_of(beta);
    g_.order = N_;
    E_ = 1;
    for (int m = 0; m < N_; ++m) {
      if (dims[m] < 1) throw Error(NTFG_ERR_SHAPE, "tensor dimensions must be >= 1");
      g_.dims[m] = int64_t(dims[m]);
      E_ *= g_.dims[m];
    }
    g_.K = g_.dims[N_ - 1];
    g_.rows = E_ / g_.K;
    int64_t st = 1;
    for (int m = N_ - 2; m >= 0; --m) {
      g_.rstride[m] = st;
      st *= g_.dims[m];
    }
    g_.rstride[N_ - 1] = 1;
    g_.init_fast();
    E_global_ = E_;
    if (shard) {
      if (shard->slab_begin + dims[0] > shard->global_dim0)
        throw Error(NTFG_ERR_SHAPE, "shard slab exceeds the global mode-0 extent");
      E_global_ = E_ / g_.dims[0] * int64_t(shard->global_dim0);
      sharded_ = c_.has_comm();
    }
    off_.resize(N_ + 1, 0);
    for (int m = 0; m < N_; ++m) off_[m + 1] = off_[m] + g_.dims[m] * R_;
    const size_t F = size_t(off_[N_]);
    A_ = c_.buf<double>("cp.A", F);
    Aref_ = c_.buf<double>("cp.Aref", F);
    chi1_ = c_.buf<double>("cp.chi1", F);
    chi2_ = c_.buf<double>("cp.chi2", F);
    anch_ = c_.buf<double>("cp.anchor", F);
    stage_ = c_.buf<T>("cp.stage", size_t(g_.K) * RP_);
    stage_anchor_ = c_.buf<T>("cp.stage_anchor", size_t(g_.K) * RP_);
    colsum_ = c_.buf<double>("cp.colsum", size_t(N_) * R_ + 1);
    colprod_ = c_.buf<double>("cp.colprod", size_t(R_));
    flags_ = c_.buf<unsigned>("cp.flags", 1);
    counter_ = c_.buf<int>("cp.counter", 1);
    colsum_done_ = c_.buf<int>("cp.colsum_done", 1);
    NTFG_CUDA(cudaMemsetAsync(colsum_done_, 0, sizeof(int), c_.stream));
    raw_ = c_.buf<double>("cp.raw", 1);
    numden_ = c_.buf<double>("cp.numden", size_t(2) * max_dim() * R_);
    // objective partials: one per recon CTA (grid depends on the kernel variant)
    objpart_ = c_.buf<double>("cp.objpart", size_t(std::max({recon_grid(false), recon_grid(true), c_.sm_count * 8})));
    tc_ = decide_tc();
    if (sizeof(T) == 4 && N_ >= 2) hstage_ = c_.buf<float>("cp.hstage", size_t(g_.dims[N_ - 2]) * size_t(R_));
  }

  int order() const { return N_; }
  int64_t entries() const { return E_; }
  int64_t entries_global() const { return E_global_; }
  int64_t dim(int m) const { return g_.dims[m]; }
  size_t factor_doubles() const { return size_t(off_[N_]); }
  double* A(int m) const { return A_ + off_[m]; }
  double* A_all() const { return A_; }

  // ---- data & parameters ---------------------------------------------------
  void set_x(const void* x, int dtype, int location) {
    const bool want_f32 = sizeof(T) == 4;
    if (location == NTFG_DEVICE && ((dtype == 1) == want_f32)) {
      x_ = static_cast<const T*>(x);
      compute_xconst();
      return;
    }
    T* dst = c_.buf<T>("cp.x", size_t(E_));
    upload_convert(dst, x, dtype, location, E_);
    x_ = dst;
    compute_xconst();
  }

  // x-only objective constant for the tensor-core recon (see xconst_kernel);
  // computed when the data arrives, outside any captured graph.
  bool split_objective() const { return tc_ && (bk_ == kBetaHalf || bk_ == kBeta3Half || bk_ == kBetaGeneric); }
  // the tile / tcgen05 reconstructions evaluate the model part of d_beta only
  bool rt_objective() const { return bk_ == kBetaHalf || bk_ == kBeta3Half || bk_ == kBetaGeneric; }
  void compute_xconst() {
    if (!(split_objective() || (rt_objective() && (recon_tc_ok(true) || recon_tc_ok(false))))) return;
    if (!xconst_) xconst_ = c_.buf<double>("cp.xconst", 1 + kXconstGrid);
    xconst_kernel<T><<<kXconstGrid, 256, 0, c_.stream>>>(x_, E_, beta_, xconst_ + 1);
    NTFG_LAUNCHED(c_);
    xconst_finish_kernel<<<1, 256, 0, c_.stream>>>(xconst_ + 1, kXconstGrid, 1.0 / (beta_ * (beta_ - 1.0)), xconst_);
    NTFG_LAUNCHED(c_);
  }

  void upload_convert(T* dst, const void* src, int dtype, int location, int64_t n) {
    const bool same = (dtype == 1) == (sizeof(T) == 4);
    const cudaMemcpyKind kind = location == NTFG_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (same) {
      NTFG_CUDA(cudaMemcpyAsync(dst, src, size_t(n) * sizeof(T), kind, c_.stream));
      return;
    }
    // convert in chunks through a device staging buffer
    const int64_t chunk = int64_t(1) << 26;
    const size_t esz = dtype == 1 ? 4 : 8;
    void* tmp = c_.bufs.get("cp.xstage", size_t(std::min(n, chunk)) * esz);
    for (int64_t b = 0; b < n; b += chunk) {
      const int64_t len = std::min(chunk, n - b);
      NTFG_CUDA(cudaMemcpyAsync(tmp, static_cast<const char*>(src) + b * esz, size_t(len) * esz, kind, c_.stream));
      const int grid = int(std::min<int64_t>(ceil_div(len, 256), 4096));
      if (dtype == 1)
        convert_kernel<T, float><<<grid, 256, 0, c_.stream>>>(static_cast<const float*>(tmp), len, dst + b);
      else
        convert_kernel<T, double><<<grid, 256, 0, c_.stream>>>(static_cast<const double*>(tmp), len, dst + b);
      NTFG_LAUNCHED(c_);
    }
  }

  void set_factors_host(const double* f) {
    c_.h2d(A_, f, factor_doubles() * sizeof(double));
    stage(A(N_ - 1), stage_);
  }
  void get_factors_host(double* f) { c_.d2h(f, A_, factor_doubles() * sizeof(double)); }
  void restage() { stage(A(N_ - 1), stage_); }

  // ---- scratch for P / Q -----------------------------------------------------
  void ensure_pq() {
    if (tc_) {
      if (!planes_[0]) {
        planes_[0] = c_.bufs.get("cp.ph", size_t(E_) * 2);
        planes_[1] = c_.bufs.get("cp.pl", size_t(E_) * 2);
      }
      if (!planes_[2] && beta_ != 1.0) {
        planes_[2] = c_.bufs.get("cp.qh", size_t(E_) * 2);
        planes_[3] = c_.bufs.get("cp.ql", size_t(E_) * 2);
      }
      return;
    }
    if (!p_) p_ = c_.buf<T>("cp.p", size_t(E_));
    if (!q_ && beta_ != 1.0) q_ = c_.buf<T>("cp.q", size_t(E_));
  }

  // weights of the model `fac` into the P/Q storage of this engine
  // (fp32/fp64 arrays, or bf16 hi/lo planes on the tensor-core path)
  void recon_pq(const double* const* fac, const T* alast, bool write_q, bool objective) {
    ensure_pq();
    if (tc_) {
      planes_out_ = true;
      recon(fac, alast, nullptr, nullptr, objective);
      planes_out_ = false;
    } else {
      recon(fac, alast, p_, write_q ? q_ : nullptr, objective);
    }
  }
  T* p() { ensure_pq(); return p_; }
  // Q buffer even at beta = 1 (the Tucker path contracts Q == 1 densely, as
  // the reference does, tucker.cpp:52,72)
  T* q_always() {
    ensure_pq();
    if (!q_) q_ = c_.buf<T>("cp.q", size_t(E_));
    return q_;
  }
  T* q() { ensure_pq(); return q_; }
  void set_pq_external(T* p, T* q) { p_ = p; q_ = q; }

  // ---- loss bookkeeping ----------------------------------------------------------
  void bind_losses(double* losses) { losses_ = losses; }
  void reset_counter() { NTFG_CUDA(cudaMemsetAsync(counter_, 0, sizeof(int), c_.stream)); }
  void reset_flags() { NTFG_CUDA(cudaMemsetAsync(flags_, 0, sizeof(unsigned), c_.stream)); }
  unsigned* flags() const { return flags_; }

  // ---- kernels -----------------------------------------------------------------------
  void stage(const double* src, T* dst) {
    const int64_t n = g_.K * RP_;
    stage_kernel<T><<<int(ceil_div(n, 256)), 256, 0, c_.stream>>>(src, g_.K, int(R_), RP_, dst);
    NTFG_LAUNCHED(c_);
  }

  int64_t recon_work() const {
    return ceil_div(g_.rows, kRows) * ceil_div(g_.K, int64_t(recon_tpb()) * recon_kt());
  }
  // v2: two columns per thread (packed loads, FFMA2) when the row length allows
  int recon_kt() const { return (sizeof(T) == 4 && RP_ <= 32 && g_.K % 2 == 0) ? 2 : 1; }
  int recon_tpb() const { return g_.K > 128 * recon_kt() ? 256 : 128; }
  // v3 (bulk-copy staging): rows must be 16-byte multiples
  bool rows_tma_ok(const void* base) const {
    return (g_.K * int64_t(sizeof(T))) % 16 == 0 && (reinterpret_cast<uintptr_t>(base) % 16) == 0;
  }
  int recon_kt3() const {
    if (sizeof(T) == 4) return RP_ <= 16 ? 4 : RP_ <= 32 ? 2 : 1;
    return RP_ <= 16 ? 2 : 1;
  }
  int recon_grid(bool v3) const {
    const int64_t w = v3 ? int64_t(128) * recon_kt3() : int64_t(recon_tpb()) * recon_kt();
    const int64_t kts = ceil_div(g_.K, w);
    const int64_t per = std::max<int64_t>(1, std::min<int64_t>(ceil_div(g_.rows, kRows),
                                                               ceil_div(int64_t(c_.sm_count) * (v3 ? 3 : 2), kts)));
    return int(kts * per);
  }

  // Xhat of the model `fac` (prefix modes) with staged last factor `alast`;
  // writes P/Q (nullable) and/or the objective into losses[counter].
  void recon(const double* const* fac, const T* alast, T* pout, T* qout, bool objective,
             T* xhout = nullptr, const double* htab = nullptr) {
    ReconParams<T> p{};
    p.g = g_;
    p.R = int(R_);
    for (int m = 0; m < N_; ++m) p.fac[m] = fac[m];
    p.alast = alast;
    p.x = x_;
    p.pout = pout;
    p.qout = qout;
    p.xhout = xhout;
    p.htab = htab;
    if (planes_out_)
      for (int i = 0; i < 4; ++i) p.planes[i] = planes_[i];
    p.obj = objective ? objpart_ : nullptr;
    p.flags = flags_;
    p.beta = beta_;
    p.eps = eps_;
    p.bk = bk_;
    // tensor-core path (fp32, K % 128 == 0): the register-tiled kernel for the
    // planes pass and for objective-only passes
    const bool tile = tc_ && sizeof(T) == 4 && !htab && !xhout && !pout && !qout && rows_tma_ok(x_) &&
                      g_.K % kRtCols == 0 && RP_ <= 64 && !tile_disabled();
    // tcgen05 reconstruction: also with fp32 P/Q outputs and with a row table
    const bool rtc = sizeof(T) == 4 && !xhout && rows_tma_ok(x_) && RP_ <= 64 && !tile_disabled() &&
                     recon_tc_ok(htab != nullptr) && (tile || htab || pout || !tc_);
    obj_split_ = (tile || rtc) ? rt_objective() : (planes_out_ && split_objective());
    if (rtc) {
      // Xhat on the tensor cores (recon_tc.cuh): one persistent CTA per SM,
      // grid a multiple of the k tiles
      p.ktiles = int(g_.K / kRcCols);
      const int64_t ntiles = g_.rows / kRcRows;
      const int64_t per = std::max<int64_t>(1, std::min<int64_t>(ntiles, int64_t(c_.sm_count) / p.ktiles));
      recon_grid_ = int(per * p.ktiles);
      if constexpr (sizeof(T) == 4) {
        // fp32 copy of the fastest row mode's factor for the H producers: pays at R = 64 (C5 K2 12.3 ->
        // 11.8 ms, half the L2 bytes per tile), not at R = 32 (C2 0.327 -> 0.361 ms), measured
        if (!htab && hstage_ && (R_ & 3) == 0 && R_ > 32) {
          const int64_t n = g_.dims[N_ - 2] * R_;
          stage_kernel<float><<<int(ceil_div(n, 256)), 256, 0, c_.stream>>>(fac[N_ - 2], g_.dims[N_ - 2], int(R_),
                                                                            int(R_), hstage_);
          NTFG_LAUNCHED(c_);
          p.hfac32 = hstage_;
        }
      }
      const int ph = c_.prof_begin(0);
      if constexpr (sizeof(T) == 4) {
        recon_tc_launch(recon_grid_, c_.stream, p, RP_, bk_);
        NTFG_LAUNCHED(c_);
      }
      c_.prof_end(ph);
      if (objective) finish_objective();
      return;
    }
    if (tile) {
      p.ktiles = int(g_.K / kRtCols);
      const int ph = c_.prof_begin(0);
      if constexpr (sizeof(T) == 4) {
        switch (RP_) {
          case 8: launch_tile<8>(p); break;
          case 16: launch_tile<16>(p); break;
          case 32: launch_tile<32>(p); break;
          default: launch_tile<64>(p); break;
        }
      }
      c_.prof_end(ph);
      if (objective) finish_objective();
      return;
    }
    const bool v3 = (rows_tma_ok(x_) && (!pout || rows_tma_ok(pout)) && (!qout || rows_tma_ok(qout))) || planes_out_;
    recon_grid_ = recon_grid(v3);
    recon_v3_ = v3;
    p.ktiles = int(ceil_div(g_.K, v3 ? int64_t(128) * recon_kt3() : int64_t(recon_tpb()) * recon_kt()));
    p.work = recon_work();
    const int ph = c_.prof_begin(0);
    switch (RP_) {
      case 8: launch_recon<8>(p); break;
      case 16: launch_recon<16>(p); break;
      case 32: launch_recon<32>(p); break;
      default: launch_recon<64>(p); break;
    }
    c_.prof_end(ph);
    if (objective) finish_objective();
  }

  void finish_objective() {
    const double inv = 1.0 / double(E_global_);
    if (sharded_) {
      objective_finalize_kernel<<<1, 256, 0, c_.stream>>>(objpart_, recon_grid_, inv, losses_, counter_, raw_,
                                                           obj_split_ ? xconst_ : nullptr);
      NTFG_LAUNCHED(c_);
      allreduce(raw_, 1);
      objective_scale_kernel<<<1, 1, 0, c_.stream>>>(raw_, inv, losses_, counter_);
      NTFG_LAUNCHED(c_);
    } else {
      objective_finalize_kernel<<<1, 256, 0, c_.stream>>>(objpart_, recon_grid_, inv, losses_, counter_, nullptr,
                                                           obj_split_ ? xconst_ : nullptr);
      NTFG_LAUNCHED(c_);
    }
  }

  // Mode-n contraction of one or two streams (reference cp_contract,
  // tensor.cpp:372-406) into per-unit partials, then the fp64 second stage
  // + MU step.  mfac[s][m] are the factors multiplied in for stream s.
  struct Stream {
    const T* src;
    const double* fac[kMaxOrder];
    const double* mtab = nullptr;  // case A row table (Tucker partial reconstruction)
    int plane = -1;                // tensor-core path: 0 = P planes, 1 = Q planes
  };

  // ---- tensor-core K3 (tc_contract.cuh) -------------------------------------------
  // Eligible: fp32 build, K a multiple of 128 up to 512, rank <= 64 with the
  // double-buffered accumulator fitting TMEM, 16-row TMA boxes for every mode.
  bool decide_tc() const {
    if (sizeof(T) != 4 || !tc_allowed_) return false;
    if (const char* e = std::getenv("NTFG_DISABLE_TC")) if (e[0] == '1') return false;
    if (g_.K % 128 != 0 || g_.K > 512 || R_ > 64 || g_.rows >= (int64_t(1) << 31)) return false;
    for (int n = 0; n < N_ - 1; ++n) {
      int64_t Bn = 1;
      for (int m = n + 1; m < N_ - 1; ++m) Bn *= g_.dims[m];
      if (!(Bn % 16 == 0 || Bn == 1 || Bn == 2 || Bn == 4 || Bn == 8)) return false;
    }
    return true;
  }
  int tc_n() const { return R_ <= 16 ? 16 : R_ <= 32 ? 32 : 64; }
  // shared-memory plan of one contraction launch: A stages (1024-aligned),
  // B tiles, then the B producers' cp.async gather ring.  Deeper gathers first
  // (they hide the L2 latency of the factor rows), then more stages.
  // m-tiles per work item: ns * mtw * N segment accumulator columns plus as
  // many running-sum columns must fit the 512 TMEM columns
  int tc_mtw(int ns) const {
    const int mt = int(g_.K / 128), N = tc_n();
    int w = mt;
    while (w > 1 && (ns * w * N > 256 || mt % w != 0)) --w;
    return w;
  }
  TcLayout tc_layout(int ns, int N, int nmm, bool gfast) const {
    TcLayout L{};
    L.a_stream = uint32_t(2 * (2 * tc_mtw(ns)) * 2048);
    L.a_stage = uint32_t(ns) * L.a_stream;
    L.b_tile = uint32_t(N / 8 * kTcBSbo);
    L.gmodes = std::max(1, std::min(nmm, kTcGModes));
    // gather slot: per stream gm regions of [16][N] floats, or (fast path) one
    // [16][N] region plus one row per other mode
    L.g_stream = gfast ? uint32_t(16 + L.gmodes - 1) * uint32_t(N * 4) : uint32_t(L.gmodes) * 16u * uint32_t(N * 4);
    L.g_slot = uint32_t(ns) * L.g_stream;
    auto total = [&](int nst, int gd) {
      return size_t(nst) * L.a_stage + size_t(nst) * 4 * L.b_tile + size_t(gd) * L.g_slot + 1024;
    };
    // Stages first: the A stages are the HBM bytes in flight (a C5 stage is
    // 32 KB; three of them per SM are below the ~90 KB the bandwidth-latency
    // product asks for), then gather depth (L2 latency of the factor rows).
    static const int env_nst = [] { const char* e = std::getenv("NTFG_TC_NST"); return e ? std::atoi(e) : 0; }();
    static const int env_gd = [] { const char* e = std::getenv("NTFG_TC_GD"); return e ? std::atoi(e) : 0; }();
    int gd = 2, nst = 2;
    while (nst < kTcMaxStages && total(nst + 1, gd) <= kTcSmemMax) ++nst;
    // give one stage back for gather depth only when more than four stages fit
    while (gd < 4 && total(nst, gd + 1) <= kTcSmemMax) ++gd;
    if (gd < 3 && nst > 4 && total(nst - 1, 3) <= kTcSmemMax) {
      --nst;
      gd = 3;
      while (gd < 4 && total(nst, gd + 1) <= kTcSmemMax) ++gd;
    }
    if (env_nst > 0) nst = std::min(env_nst, kTcMaxStages);
    if (env_gd > 0) gd = std::min(env_gd, kTcMaxGather);
    if (total(nst, gd) > kTcSmemMax) throw Error(NTFG_ERR_SHAPE, "tensor-core contraction: shared memory plan");
    L.nst = nst;
    L.gdepth = gd;
    L.b_off = uint32_t(nst) * L.a_stage;
    L.ring_off = L.b_off + uint32_t(nst) * 4 * L.b_tile;
    L.total = uint32_t(total(nst, gd));
    return L;
  }
  bool tc() const { return tc_; }
  void disable_tc() { tc_allowed_ = false; tc_ = false; }
  void* plane(int i) { ensure_pq(); return planes_[i]; }

  // work split of one tensor-core contraction: case A (last mode) = row
  // chunks, case B = (target index, split) pairs; chunk = rows per unit
  // stages (of 16 rows) per TMEM accumulation segment (tc_contract.cuh, MMA issuers)
  static int tc_seg_stages() {
    static const int v = [] { const char* e = std::getenv("NTFG_TC_SEG"); return e ? std::max(1, std::atoi(e)) : 16; }();
    return v;
  }
  static int64_t tc_unit_rows_cap() {  // experiments: NTFG_TC_UNIT_ROWS caps the TMEM accumulation length
    static const int64_t v = [] { const char* e = std::getenv("NTFG_TC_UNIT_ROWS"); return e ? std::atoll(e) : 0; }();
    return v;
  }
  void tc_units(int n, int64_t& units, int64_t& S, int64_t& chunk) const {
    const int64_t cap = tc_unit_rows_cap();
    if (n == N_ - 1) {
      const int64_t target = std::min<int64_t>(ceil_div(g_.rows, kTcRows), int64_t(c_.sm_count));
      chunk = ceil_div(ceil_div(g_.rows, target), kTcRows) * kTcRows;
      if (cap > 0) chunk = std::min(chunk, ceil_div(cap, kTcRows) * kTcRows);
      units = ceil_div(g_.rows, chunk);
      S = 1;
      return;
    }
    const int64_t In = g_.dims[n];
    int64_t An = 1, Bn = 1;
    for (int m = 0; m < n; ++m) An *= g_.dims[m];
    for (int m = n + 1; m < N_ - 1; ++m) Bn *= g_.dims[m];
    const int64_t tot = An * Bn;
    int64_t S0 = std::max<int64_t>(1, std::min<int64_t>(ceil_div(int64_t(4) * c_.sm_count, In), ceil_div(tot, kTcRows)));
    {
      // units are dealt round-robin to one CTA per SM: pick the split count in
      // [S0, S0 + 8] whose last wave is fullest (C5: S = 3 gives 768 units =
      // 5.19 waves, i.e. 6 -- 13% of the launch idle; S = 4 gives 6.92 -> 7)
      const int64_t smax = std::min<int64_t>(S0 + 8, std::max<int64_t>(S0, tot / (4 * kTcRows)));
      double best = 0.0;
      int64_t bestS = S0;
      for (int64_t s = S0; s <= smax; ++s) {
        const int64_t chunk_s = ceil_div(ceil_div(tot, s), kTcRows) * kTcRows;
        const int64_t units_s = In * ceil_div(tot, chunk_s);
        const double eff = double(units_s) / double(ceil_div(units_s, c_.sm_count) * c_.sm_count);
        if (eff > best + 0.01) {
          best = eff;
          bestS = s;
        }
      }
      S0 = bestS;
    }
    if (cap > 0) S0 = std::max(S0, ceil_div(tot, ceil_div(cap, kTcRows) * kTcRows));
    chunk = ceil_div(ceil_div(tot, S0), kTcRows) * kTcRows;
    S = ceil_div(tot, chunk);
    units = In * S;
  }

  void tc_contract(int n, int ns, const Stream* st, int64_t& units_out, int64_t& S_out) {
    const bool caseA = (n == N_ - 1);
    TcParams p{};
    p.g = g_;
    p.n = n;
    p.R = int(R_);
    p.RP = RP_;
    p.N = tc_n();
    p.ns = ns;
    p.mt = int(g_.K / 128);
    p.mtw = tc_mtw(ns);
    p.G = p.mt / p.mtw;
    p.seg = tc_seg_stages();
    p.caseA = caseA;
    const int64_t In = g_.dims[n];
    TcMaps maps{};
    int64_t mapB, mapI = 1, mapA = 1;
    if (caseA) {
      tc_units(n, p.units, p.S, p.chunk);
      p.An = 1;
      p.Bn = g_.rows;
      p.boxB = kTcRows;
      p.boxA = 1;
      mapB = g_.rows;
    } else {
      int64_t An = 1, Bn = 1;
      for (int m = 0; m < n; ++m) An *= g_.dims[m];
      for (int m = n + 1; m < N_ - 1; ++m) Bn *= g_.dims[m];
      tc_units(n, p.units, p.S, p.chunk);
      p.An = An;
      p.Bn = Bn;
      p.boxB = int(Bn >= kTcRows ? kTcRows : Bn);
      p.boxA = kTcRows / p.boxB;
      mapB = Bn;
      mapI = In;
      mapA = An;
    }
    p.fB.init(p.Bn);
    // fp32 zero-padded copies of every factor of every stream (B gathers, case-B epilogue)
    F32Stage fs{};
    fs.order = N_;
    fs.ns = ns;
    fs.R = int(R_);
    fs.N = p.N;
    for (int m = 0; m < N_; ++m) fs.off[m + 1] = fs.off[m] + g_.dims[m] * p.N;
    if (!lastT_) lastT_ = c_.buf<float>("cp.lastT", size_t(2) * fs.off[N_]);
    for (int s = 0; s < ns; ++s) {
      for (int m = 0; m < N_; ++m) {
        p.mfac[s][m] = st[s].fac[m];
        fs.src[s][m] = st[s].fac[m];
        fs.dst[s][m] = lastT_ + size_t(s) * fs.off[N_] + fs.off[m];
        p.fac32[s][m] = fs.dst[s][m];
      }
      p.lastfac[s] = p.fac32[s][N_ - 1];
      for (int h = 0; h < 2; ++h)
        if (!tc::make_plane_map(&maps.m[s][h], planes_[2 * st[s].plane + h], g_.K, mapB, mapI, mapA, p.boxB,
                                p.boxA, 2 * p.mtw))
          throw Error(NTFG_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    }
    int nmm = 0;
    for (int m = 0; m < N_ - 1; ++m) nmm += (m != n);
    {  // fast gathers: the fastest off-mode f (highest index != n among the row modes) has 16 | I_f
      int f = -1;
      for (int m = 0; m < N_ - 1; ++m)
        if (m != n) f = m;
      p.gfast = (f >= 0 && g_.dims[f] % kTcRows == 0) ? 1 : 0;
      const char* slow = std::getenv("NTFG_TC_SLOW_GATHER");  // tests: force the per-row gather path
      if (slow && slow[0] == '1') p.gfast = 0;
      p.fmode = f;
      p.btiles = btiles_;  // scratch for the static B tiles (decided by the launcher)
    }
    p.lay = tc_layout(ns, p.N, nmm, p.gfast != 0);
    p.partA = reinterpret_cast<float*>(partA_);
    p.partB = partB_;
    const int cols = ns * p.mtw * p.N;  // segment accumulators, then the running sums
    int alloc = 32;
    while (alloc < 2 * cols) alloc *= 2;
    p.tmem_cols = alloc;
    p.items = p.units * p.G;
    {  // perf experiments only (tools/): role ablation bits, results are wrong when set
      static const int dbg = [] { const char* e = std::getenv("NTFG_TC_ABLATE"); return e ? std::atoi(e) : 0; }();
      p.ablate = dbg;
    }
    const int grid = int(std::min<int64_t>(p.items, int64_t(c_.sm_count)));
    static const char* trace_path = std::getenv("NTFG_TC_TRACE");  // perf experiments (eager fits only)
    if (trace_path) {
      p.trace = reinterpret_cast<unsigned long long*>(c_.bufs.get("cp.tctrace", size_t(grid) * 17 * 8 * 8));
      NTFG_CUDA(cudaMemsetAsync(p.trace, 0, size_t(grid) * 17 * 8 * 8, c_.stream));
    }
    tc_contract_launch(grid, c_.stream, maps, p, fs);  // staging launch + contraction
    NTFG_LAUNCHED(c_);
    NTFG_LAUNCHED(c_);
    if (trace_path) {
      std::vector<unsigned long long> h(size_t(grid) * 17 * 8);
      NTFG_CUDA(cudaMemcpyAsync(h.data(), p.trace, h.size() * 8, cudaMemcpyDeviceToHost, c_.stream));
      NTFG_CUDA(cudaStreamSynchronize(c_.stream));
      if (FILE* f = std::fopen(trace_path, "a")) {
        std::fprintf(f, "launch n=%d units=%lld S=%lld grid=%d\n", n, (long long)p.units, (long long)p.S, grid);
        for (size_t i = 0; i < size_t(grid) * 128; i += 8)
          std::fprintf(f, "%zu %zu %llu %llu %llu %llu %llu %llu %llu %llu\n", i / 128, (i / 8) % 16, h[i], h[i + 1],
                       h[i + 2], h[i + 3], h[i + 4], h[i + 5], h[i + 6], h[i + 7]);
        for (size_t i = size_t(grid) * 128; i < h.size(); i += 8)  // per-CTA role wait totals
          std::fprintf(f, "wstats %llu %llu %llu %llu %llu %llu %llu\n", h[i], h[i + 1], h[i + 2], h[i + 3],
                       h[i + 4], h[i + 5], h[i + 6]);
        std::fclose(f);
      }
    }
    units_out = p.units;
    S_out = caseA ? p.S : p.S * p.G;  // case B partials: [ns][In][S * G][RP]
  }

  struct Plan {
    bool caseA, v3;
    int RC, KT, TPS, ktiles, grid;
    int64_t In, units, S, An, Bn;
  };

  Plan plan(int n, bool v3 = false) const {
    Plan pl{};
    pl.caseA = (n == N_ - 1);
    pl.v3 = v3;
    const int RCmax = sizeof(T) == 4 ? 64 : 32;
    pl.RC = R_ <= 8 ? 8 : R_ <= 16 ? 16 : R_ <= 32 ? 32 : RCmax;
    if (v3) {
      pl.KT = sizeof(T) == 4 ? (pl.RC <= 32 ? 4 : 1) : 2;
      pl.TPS = 128;
    } else {
      pl.KT = (sizeof(T) == 4 && pl.RC <= 32 && g_.K % 2 == 0) ? 2 : 1;
      pl.TPS = g_.K > 128 * pl.KT ? 256 : 128;
    }
    pl.ktiles = int(ceil_div(g_.K, int64_t(pl.TPS) * pl.KT));
    pl.In = g_.dims[n];
    pl.S = 1;
    pl.An = 1;
    pl.Bn = 1;
    if (pl.caseA) {
      pl.units = std::min<int64_t>(g_.rows, int64_t(c_.sm_count) * ((pl.TPS == 256 || v3) ? 1 : 2));
    } else {
      for (int m = 0; m < n; ++m) pl.An *= g_.dims[m];
      for (int m = n + 1; m < N_ - 1; ++m) pl.Bn *= g_.dims[m];
      const int64_t tot = pl.An * pl.Bn;
      pl.S = std::max<int64_t>(1, std::min<int64_t>(ceil_div(int64_t(4) * c_.sm_count, pl.In),
                                                    std::max<int64_t>(1, tot / 16)));
      pl.units = pl.In * pl.S;
    }
    const int ns_max = beta_ == 1.0 ? 1 : 2;  // one CTA per SM at 512 threads
    const int per_sm = v3 ? 1 : (pl.TPS * ns_max >= 512 ? 1 : 2);
    pl.grid = int(std::min<int64_t>(pl.units, int64_t(c_.sm_count) * per_sm));
    return pl;
  }

  // Allocate every buffer a fit can touch (no cudaMalloc during graph capture).
  void prealloc(int ns) {
    if (sparse_) {
      if (!n1num_) n1num_ = c_.buf<double>("cp.n1num", factor_doubles() + size_t(max_dim()) * R_);
      return;
    }
    size_t a = 0, b = 0;
    for (int n = 0; n < N_; ++n) {
      for (int v = 0; v < 2; ++v) {
        const Plan pl = plan(n, v == 1);
        if (pl.caseA) a = std::max(a, size_t(ns) * pl.units * g_.K * RP_);
        else b = std::max(b, size_t(ns) * pl.In * pl.S * RP_);
      }
    }
    if (tc_)
      for (int n = 0; n < N_; ++n) {
        int64_t units, S, chunk;
        tc_units(n, units, S, chunk);
        if (n == N_ - 1) a = std::max(a, size_t(ns) * units * g_.K * RP_);
        else b = std::max(b, size_t(ns) * units * (g_.K / 128) * RP_);  // x G m-tile groups
      }
    partA_ = c_.buf<T>("cp.partA", std::max<size_t>(a, 1));
    partB_ = c_.buf<double>("cp.partB", std::max<size_t>(b, 1));
    partAd_ = c_.buf<double>("cp.partAd", std::max<size_t>(a / 8 + size_t(ns) * g_.K * RP_, 1));
    if (beta_ == 1.0) n1num_ = c_.buf<double>("cp.n1num", factor_doubles() + size_t(max_dim()) * R_);
    if (tc_) {
      size_t fl = 0;
      for (int m = 0; m < N_; ++m) fl += size_t(g_.dims[m]) * 64;
      lastT_ = c_.buf<float>("cp.lastT", 2 * fl);
      // static B tiles: [2 streams][I_f / 16 blocks][hi, lo][(N / 8) * 272 B] for the largest row mode
      int64_t imax = 16;
      for (int m = 0; m < N_ - 1; ++m) imax = std::max<int64_t>(imax, g_.dims[m]);
      btiles_ = static_cast<unsigned char*>(c_.bufs.get("cp.btiles", size_t(2) * size_t(ceil_div(imax, 16)) * 2 *
                                                                       size_t(tc_n() / 8 * kTcBSbo)));
    }
    ensure_pq();
  }

  // raw contraction of stream 0 into numden[0:In*R] (cp_contract API)
  void contract_numden(int n, const Stream* st, double* scratch) {
    contract_and_update(n, 1, st, true, scratch, scratch, nullptr, nullptr, nullptr, nullptr, 1);
  }

  void contract_and_update(int n, int ns, const Stream* st, bool den_closed,
                           const double* anchor, double* out, const double* ref, double* c1,
                           double* c2, T* stage_out, int force_phase = -1) {
    if (!partA_) prealloc(2);
    bool v3 = true;
    for (int s2 = 0; s2 < ns; ++s2) v3 = v3 && rows_tma_ok(st[s2].src);
    const bool use_tc = tc_ && st[0].plane >= 0;
    const Plan pl = plan(n, v3);
    const bool caseA = pl.caseA;
    const int RC = pl.RC;
    const int ktiles = pl.ktiles;
    const int64_t In = pl.In, An = pl.An, Bn = pl.Bn;
    int64_t units = pl.units, S = pl.S;
    const int grid = pl.grid;
    T* partA = caseA ? partA_ : nullptr;
    double* partB = caseA ? nullptr : partB_;

    const int ph = c_.prof_begin(1);
    if (use_tc) tc_contract(n, ns, st, units, S);
    for (int r0 = 0; r0 < R_ && !use_tc; r0 += RC) {
      if (ns == 2) {
        ContractParams<T, 2> p{};
        fill_contract(p, n, r0, caseA, units, S, An, Bn, partA, partB, ktiles, st, 2);
        launch_contract<2>(p, pl, grid);
      } else {
        ContractParams<T, 1> p{};
        fill_contract(p, n, r0, caseA, units, S, An, Bn, partA, partB, ktiles, st, 1);
        launch_contract<1>(p, pl, grid);
      }
    }
    c_.prof_end(ph);

    FinalizeParams<T> f{};
    if (caseA && units > 16) {
      const int64_t per = 8, chunks = ceil_div(units, per), slice = In * RP_;
      const int64_t total = int64_t(ns) * chunks * slice;
      const int rgrid = int(std::min<int64_t>(ceil_div(total, 256), int64_t(c_.sm_count) * 8));
      reduce_units_kernel<T><<<rgrid, 256, 0, c_.stream>>>(partA, units, per, chunks, slice, ns, partAd_);
      NTFG_LAUNCHED(c_);
      f.partAd = partAd_;
      f.units = chunks;
    } else {
      f.units = units;
    }
    f.caseA = caseA;
    f.In = In;
    f.R = int(R_);
    f.RP = RP_;
    f.S = S;
    f.partA = partA;
    f.partB = partB;
    f.den_closed = den_closed;
    f.colprod = colprod_;
    f.numden = numden_;
    f.anchor = anchor;
    f.out = out;
    f.ref = ref;
    f.chi1 = c1;
    f.chi2 = c2;
    f.stage = stage_out;
    f.gamma = gamma_;
    f.eps = eps_;
    f.beta = beta_;
    f.flags = flags_;
    const int fgrid = int(ceil_div(In * RP_, 256));
    if (force_phase == 1) {
      f.phase = 1;
      finalize_kernel<T><<<fgrid, 256, 0, c_.stream>>>(f);
      NTFG_LAUNCHED(c_);
      return;
    }
    if (sharded_ && n != 0) {
      // data-parallel: local partial sums -> allreduce -> identical MU on all ranks
      f.phase = 1;
      finalize_kernel<T><<<fgrid, 256, 0, c_.stream>>>(f);
      NTFG_LAUNCHED(c_);
      allreduce(numden_, size_t(2) * In * R_);
      f.phase = 2;
    } else {
      f.phase = 0;
    }
    finalize_kernel<T><<<fgrid, 256, 0, c_.stream>>>(f);
    NTFG_LAUNCHED(c_);
  }

  // beta = 1 closed-form denominator prod_{m != skip} colsum(F_m)
  void colprod(const double* const* fac, int skip) {
    ColsumParams p{};
    p.order = N_;
    p.skip = skip;
    p.R = int(R_);
    for (int m = 0; m < N_; ++m) {
      p.rows[m] = g_.dims[m];
      p.fac[m] = fac[m];
    }
    p.out = colsum_;
    // two launches when the slab-local mode-0 column sums are allreduced in between, or when no
    // block takes part (order-1 tensors: the empty product)
    const bool split = (sharded_ && skip != 0) || N_ - ((skip >= 0 && skip < N_) ? 1 : 0) == 0;
    p.prod = split ? nullptr : colprod_;
    p.done = colsum_done_;
    colsum_kernel<<<N_, kColsumThreads, 0, c_.stream>>>(p);
    NTFG_LAUNCHED(c_);
    if (split) {
      allreduce(colsum_, size_t(R_));
      colprod_kernel<<<int(ceil_div(R_, 64)), 64, 0, c_.stream>>>(colsum_, N_, skip, int(R_), colprod_);
      NTFG_LAUNCHED(c_);
    }
  }

  // ---- solver steps ----------------------------------------------------------------------

  // cp_block_update_anchored (cp.cpp:109-123); anchor == A(n) for the plain path.
  void block_update(int n, const double* anchor, bool objective) {
    const double* fac[kMaxOrder];
    for (int m = 0; m < N_; ++m) fac[m] = (m == n) ? anchor : A(m);
    if (sparse_) {
      if (objective && n != 0) coo_objective(fac);
      coo_num(n, fac, numden_, objective && n == 0);
      if (sharded_ && n != 0) allreduce(numden_, size_t(g_.dims[n]) * R_);
      if (objective && n == 0) coo_finish_objective(fac);
      colprod(fac, n);
      coo_finalize(n, numden_, anchor, nullptr);
      return;
    }
    const T* alast = stage_;
    if (n == N_ - 1 && anchor != A(n)) {
      stage(anchor, stage_anchor_);
      alast = stage_anchor_;
    }
    recon_pq(fac, alast, beta_ != 1.0, objective);
    const bool closed = beta_ == 1.0;
    if (closed) colprod(fac, n);
    Stream st[2];
    st[0].src = p_;
    st[1].src = q_;
    if (tc_) {
      st[0].plane = 0;
      st[1].plane = 1;
    }
    for (int m = 0; m < N_; ++m) st[0].fac[m] = st[1].fac[m] = fac[m];
    contract_and_update(n, closed ? 1 : 2, st, closed, anchor, A(n), nullptr, nullptr, nullptr,
                        n == N_ - 1 ? stage_ : nullptr);
  }

  // bcomm_sweep (cp.cpp:131-135), objective of the incoming model fused into block 0
  void bcomm_sweep(bool fuse_objective) {
    for (int n = 0; n < N_; ++n) block_update(n, A(n), fuse_objective && n == 0);
  }

  void bcomm_sweep_anchored(const double* anchors) {
    for (int n = 0; n < N_; ++n) block_update(n, anchors + off_[n], false);
  }

  // make_jcomm_reference (cp.cpp:202-208): ref := A, chi := A (exact: chi(Z,Z) = Z)
  void jcomm_reference(bool objective) {
    const size_t bytes = factor_doubles() * sizeof(double);
    c_.d2d(Aref_, A_, bytes);
    c_.d2d(chi1_, A_, bytes);
    c_.d2d(chi2_, A_, bytes);
    const double* fac[kMaxOrder];
    for (int m = 0; m < N_; ++m) fac[m] = A(m);
    if (sparse_) {  // the objective rides on the mode-0 numerator pass (n1_numerators)
      coo_pending_obj_ = objective;
      return;
    }
    recon_pq(fac, stage_, beta_ != 1.0, objective);
  }

  // jcomm_inner_update (cp.cpp:210-229)
  void jcomm_inner(int n) {
    const bool closed = beta_ == 1.0;
    const double* c2[kMaxOrder];
    for (int m = 0; m < N_; ++m) c2[m] = chi2_ + off_[m];
    if (closed) colprod(c2, n);
    Stream st[2];
    st[0].src = p_;
    st[1].src = q_;
    if (tc_) {
      st[0].plane = 0;
      st[1].plane = 1;
    }
    for (int m = 0; m < N_; ++m) {
      st[0].fac[m] = chi1_ + off_[m];
      st[1].fac[m] = chi2_ + off_[m];
    }
    contract_and_update(n, closed ? 1 : 2, st, closed, Aref_ + off_[n], A(n), Aref_ + off_[n],
                        chi1_ + off_[n], chi2_ + off_[n], n == N_ - 1 ? stage_ : nullptr);
  }

  // beta = 1 (SURVEY.md 8(a) note N1): chi1(Z, Zref) == Zref exactly
  // (fast_pow(x, 0) == 1, kernels.hpp:13), so every inner numerator
  // cp_contract(P~, chi1(...)) depends only on P~ and the reference factors:
  // it is computed once per outer iteration (one P~ pass per mode) and reused
  // by all L sweeps; the denominator is the closed form of cp.cpp:224-225.
  void n1_numerators() {
    if (!n1num_) n1num_ = c_.buf<double>("cp.n1num", factor_doubles() + size_t(max_dim()) * R_);
    if (sparse_) {
      const double* fac[kMaxOrder];
      for (int m = 0; m < N_; ++m) fac[m] = Aref_ + off_[m];
      for (int n = 0; n < N_; ++n) {
        coo_num(n, fac, n1num_ + off_[n], n == 0 && coo_pending_obj_);
        if (sharded_ && n != 0) allreduce(n1num_ + off_[n], size_t(g_.dims[n]) * R_);
        if (n == 0 && coo_pending_obj_) coo_finish_objective(fac);
      }
      coo_pending_obj_ = false;
      return;
    }
    Stream st[2];
    st[0].src = p_;
    st[1].src = p_;
    if (tc_) st[0].plane = st[1].plane = 0;
    for (int m = 0; m < N_; ++m) st[0].fac[m] = st[1].fac[m] = Aref_ + off_[m];
    for (int n = 0; n < N_; ++n) {
      contract_and_update(n, 1, st, true, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 1);
      if (sharded_ && n != 0) allreduce(numden_, size_t(g_.dims[n]) * R_);
      c_.d2d(n1num_ + off_[n], numden_, size_t(g_.dims[n]) * R_ * sizeof(double));
    }
  }

  void jcomm_inner_n1(int n) {
    const double* c2[kMaxOrder];
    for (int m = 0; m < N_; ++m) c2[m] = chi2_ + off_[m];
    colprod(c2, n);
    FinalizeParams<T> f{};
    f.In = g_.dims[n];
    f.R = int(R_);
    f.RP = RP_;
    f.den_closed = 1;
    f.colprod = colprod_;
    f.phase = 2;
    f.numden = n1num_ + off_[n];
    f.anchor = Aref_ + off_[n];
    f.out = A(n);
    f.ref = Aref_ + off_[n];
    f.chi1 = chi1_ + off_[n];
    f.chi2 = chi2_ + off_[n];
    f.stage = n == N_ - 1 ? stage_ : nullptr;
    f.gamma = gamma_;
    f.eps = eps_;
    f.beta = beta_;
    f.flags = flags_;
    finalize_kernel<T><<<int(ceil_div(g_.dims[n] * RP_, 256)), 256, 0, c_.stream>>>(f);
    NTFG_LAUNCHED(c_);
  }

  // jcomm_outer_step (cp.cpp:231-240)
  void jcomm_outer(int inner_steps, bool fuse_objective) {
    jcomm_reference(fuse_objective);
    if (beta_ == 1.0 && (n1_enabled_ || sparse_)) {
      n1_numerators();
      for (int l = 0; l < inner_steps; ++l)
        for (int n = 0; n < N_; ++n) jcomm_inner_n1(n);
      return;
    }
    for (int l = 0; l < inner_steps; ++l)
      for (int n = 0; n < N_; ++n) jcomm_inner(n);
  }
  void set_n1(bool on) { n1_enabled_ = on; }

  const T* x() const { return x_; }
  unsigned* flag_ptr() const { return flags_; }
  double* chi1_all() const { return chi1_; }
  double* chi2_all() const { return chi2_; }
  T* stage_last() const { return stage_; }
  double* numden() const { return numden_; }

  // standalone objective of the current model
  void objective() {
    const double* fac[kMaxOrder];
    for (int m = 0; m < N_; ++m) fac[m] = A(m);
    if (sparse_) {
      coo_objective(fac);
      return;
    }
    recon(fac, stage_, nullptr, nullptr, true);
  }

  // ---- sparse COO data (K7, coo_kernels.cuh; beta = 1 only) -------------------------------
  // indices: [nnz][order] int32 row-major (host or device), values fp32/fp64;
  // in a data-parallel fit (shard) they are this rank's nonzeros with i_0
  // local to its mode-0 slab (dims[0] = slab rows), exactly like a dense slab.
  // Duplicates are summed in input order (as read_coo's dense +=, io.cpp:138);
  // one copy of the merged nonzeros per mode, stably sorted by that mode's
  // index (coo_ingest.cuh: keys, radix sorts and scans on the device).
  template <typename F>
  void cub_call(const char* what, F&& f) {
    size_t bytes = 0;
    NTFG_CUDA(f(nullptr, bytes));
    void* tmp = c_.bufs.get("coo.cubtmp", std::max<size_t>(bytes, 16));
    cuda_check(f(tmp, bytes), what);
  }
  void set_coo(uint64_t nnz, const int32_t* indices, const void* values, int dtype, int location) {
    if (beta_ != 1.0) throw Error(NTFG_ERR_DOMAIN, "sparse COO fits require beta = 1");
    if (R_ > 64) throw Error(NTFG_ERR_SHAPE, "sparse COO fits support rank <= 64");
    if (nnz >= (uint64_t(1) << 31)) throw Error(NTFG_ERR_SHAPE, "sparse COO fits support < 2^31 nonzeros");
    const int N = N_;
    const int64_t n = int64_t(nnz);
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), int64_t(c_.sm_count) * 8)));
    const size_t vbytes = dtype == 1 ? 4 : 8;
    const int32_t* didx = indices;
    const void* dval = values;
    if (location != NTFG_DEVICE) {
      int32_t* ti = c_.buf<int32_t>("coo.in_idx", std::max<size_t>(size_t(n) * N, 1));
      void* tv = c_.bufs.get("coo.in_val", std::max<size_t>(size_t(n) * vbytes, 8));
      c_.h2d(ti, indices, size_t(n) * N * sizeof(int32_t));
      c_.h2d(tv, values, size_t(n) * vbytes);
      didx = ti;
      dval = tv;
    }
    // 1. linear keys + stable sort -> merged nonzeros (lexicographic order)
    int64_t* key = c_.buf<int64_t>("coo.key", std::max<int64_t>(n, 1));
    int64_t* key2 = c_.buf<int64_t>("coo.key2", std::max<int64_t>(n, 1));
    int64_t* pos = c_.buf<int64_t>("coo.pos", std::max<int64_t>(n, 1));
    int64_t* pos2 = c_.buf<int64_t>("coo.pos2", std::max<int64_t>(n, 1));
    unsigned* bad = c_.buf<unsigned>("coo.bad", 1);
    NTFG_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned), c_.stream));
    CooKeyParams kp{};
    kp.order = N;
    for (int m = 0; m < N; ++m) kp.dims[m] = g_.dims[m];
    kp.nnz = n;
    kp.idx = didx;
    kp.key = key;
    kp.pos = pos;
    kp.bad = bad;
    coo_key_kernel<<<grid, 256, 0, c_.stream>>>(kp);
    NTFG_LAUNCHED(c_);
    unsigned hbad = 0;
    c_.d2h(&hbad, bad, sizeof(unsigned));
    c_.sync();
    if (hbad) throw Error(NTFG_ERR_SHAPE, "COO index out of range");
    const int kbits = bits_for(std::max<int64_t>(E_, 2) - 1);
    if (n > 0)
      cub_call("cub SortPairs (keys)", [&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortPairs(t, b, key, key2, pos, pos2, int(n), 0, kbits, c_.stream);
      });
    int32_t* head = c_.buf<int32_t>("coo.head", std::max<int64_t>(n, 1));
    int32_t* uid = c_.buf<int32_t>("coo.uid", std::max<int64_t>(n, 1) + 1);
    if (n > 0) {
      coo_head_kernel<<<grid, 256, 0, c_.stream>>>(key2, n, head);
      NTFG_LAUNCHED(c_);
      cub_call("cub ExclusiveSum (heads)", [&](void* t, size_t& b) {
        return cub::DeviceScan::ExclusiveSum(t, b, head, uid, int(n), c_.stream);
      });
    }
    int32_t last[2] = {0, 0};
    if (n > 0) {
      c_.d2h(&last[0], uid + (n - 1), sizeof(int32_t));
      c_.d2h(&last[1], head + (n - 1), sizeof(int32_t));
      c_.sync();
    }
    const int64_t M = n > 0 ? int64_t(last[0]) + last[1] : 0;
    coo_nnz_ = M;
    int32_t* midx[kMaxOrder] = {};
    for (int m = 0; m < N; ++m) midx[m] = c_.buf<int32_t>("coo.m.idx" + std::to_string(m), std::max<int64_t>(M, 1));
    double* mval = c_.buf<double>("coo.m.val", std::max<int64_t>(M, 1));
    if (n > 0) {
      CooMergeParams mp{};
      mp.order = N;
      mp.n = n;
      mp.key = key2;
      mp.pos = pos2;
      mp.head = head;
      mp.uid = uid;
      mp.idx = didx;
      mp.val = dval;
      mp.f32 = dtype == 1;
      for (int m = 0; m < N; ++m) mp.midx[m] = midx[m];
      mp.mval = mval;
      coo_merge_kernel<<<grid, 256, 0, c_.stream>>>(mp);
      NTFG_LAUNCHED(c_);
    }
    // 2. per mode: stable sort by i_n, gather, cut into pieces
    const int mgrid = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(M, 256), int64_t(c_.sm_count) * 8)));
    int32_t* iota = c_.buf<int32_t>("coo.iota", std::max<int64_t>(M, 1));
    int32_t* perm = c_.buf<int32_t>("coo.perm", std::max<int64_t>(M, 1));
    int32_t* skeys = c_.buf<int32_t>("coo.skeys", std::max<int64_t>(M, 1));
    coo_iota_kernel<<<mgrid, 256, 0, c_.stream>>>(M, iota);
    NTFG_LAUNCHED(c_);
    coo_.assign(size_t(N), CooMode{});
    int64_t max_pieces = 1;
    for (int md = 0; md < N; ++md) {
      const int64_t In = g_.dims[md];
      const std::string tag = "coo." + std::to_string(md) + ".";
      CooMode& cm = coo_[size_t(md)];
      if (M > 0)
        cub_call("cub SortPairs (mode)", [&](void* t, size_t& b) {
          return cub::DeviceRadixSort::SortPairs(t, b, midx[md], skeys, iota, perm, int(M), 0, bits_for(In),
                                                 c_.stream);
        });
      CooGatherParams gp{};
      gp.order = N;
      gp.n = M;
      gp.perm = perm;
      for (int m = 0; m < N; ++m) {
        gp.src_idx[m] = midx[m];
        cm.idx[m] = c_.buf<int32_t>(tag + "idx" + std::to_string(m), std::max<int64_t>(M, 1));
        gp.dst_idx[m] = cm.idx[m];
      }
      gp.src_val = mval;
      cm.val = c_.buf<double>(tag + "val", std::max<int64_t>(M, 1));
      gp.dst_val = cm.val;
      if (M > 0) {
        coo_gather_kernel<<<mgrid, 256, 0, c_.stream>>>(gp);
        NTFG_LAUNCHED(c_);
      }
      int32_t* cnt = c_.buf<int32_t>("coo.cnt", size_t(In) + 1);
      int64_t* cnt64 = c_.buf<int64_t>("coo.cnt64", size_t(In) + 1);
      int64_t* start = c_.buf<int64_t>("coo.start", size_t(In) + 1);
      int64_t* np = c_.buf<int64_t>("coo.np", size_t(In) + 1);
      cm.key_piece = c_.buf<int64_t>(tag + "kpiece", size_t(In) + 1);
      NTFG_CUDA(cudaMemsetAsync(cnt, 0, (size_t(In) + 1) * sizeof(int32_t), c_.stream));
      NTFG_CUDA(cudaMemsetAsync(np, 0, (size_t(In) + 1) * sizeof(int64_t), c_.stream));
      if (M > 0) {
        coo_count_kernel<<<mgrid, 256, 0, c_.stream>>>(cm.idx[md], M, cnt);
        NTFG_LAUNCHED(c_);
      }
      const int kgrid = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(In + 1, 256), int64_t(c_.sm_count) * 8)));
      widen_kernel<<<kgrid, 256, 0, c_.stream>>>(cnt, In + 1, cnt64);
      NTFG_LAUNCHED(c_);
      cub_call("cub ExclusiveSum (starts)", [&](void* t, size_t& b) {
        return cub::DeviceScan::ExclusiveSum(t, b, cnt64, start, int(In + 1), c_.stream);
      });
      coo_npieces_kernel<<<kgrid, 256, 0, c_.stream>>>(cnt, In, np);
      NTFG_LAUNCHED(c_);
      cub_call("cub ExclusiveSum (pieces)", [&](void* t, size_t& b) {
        return cub::DeviceScan::ExclusiveSum(t, b, np, cm.key_piece, int(In + 1), c_.stream);
      });
      int64_t total = 0;
      c_.d2h(&total, cm.key_piece + In, sizeof(int64_t));
      c_.sync();
      cm.npieces = total;
      max_pieces = std::max(max_pieces, total);
      cm.piece_start = c_.buf<int64_t>(tag + "pstart", size_t(total) + 1);
      coo_pieces_kernel<<<kgrid, 256, 0, c_.stream>>>(start, cnt, cm.key_piece, In, M, cm.piece_start);
      NTFG_LAUNCHED(c_);
    }
    coo_partial_ = c_.buf<double>("coo.partial", size_t(max_pieces) * size_t(R_));
    coo_obj_ = c_.buf<double>("coo.obj", size_t(max_pieces));
    coo_closed_ = c_.buf<double>("coo.closed", 1);
    c_.sync();
    sparse_ = true;
    tc_ = false;
  }
  int64_t coo_nnz() const { return coo_nnz_; }

 private:
  struct CooMode {
    int32_t* idx[kMaxOrder] = {};
    double* val = nullptr;
    int64_t* piece_start = nullptr;
    int64_t* key_piece = nullptr;
    int64_t npieces = 0;
  };

  // Num^(n) of the model `fac` into out[I_n][R]; with objective, the nnz part of
  // D_1 per mode-0 piece into coo_obj_ (n must be 0)
  void coo_num(int n, const double* const* fac, double* out, bool objective) {
    launch_coo_pieces(n, fac, true, objective);
    const int64_t In = g_.dims[n];
    const int grid = int(std::min<int64_t>(In, int64_t(c_.sm_count) * 8));
    coo_key_reduce_kernel<<<grid, 256, 0, c_.stream>>>(coo_partial_, coo_[size_t(n)].key_piece, In, int(R_), out);
    NTFG_LAUNCHED(c_);
  }
  void launch_coo_pieces(int n, const double* const* fac, bool partials, bool objective) {
    const CooMode& cm = coo_[size_t(n)];
    CooPieceParams pp{};
    pp.order = N_;
    pp.n = n;
    pp.R = int(R_);
    for (int m = 0; m < N_; ++m) {
      pp.idx[m] = cm.idx[m];
      pp.fac[m] = fac[m];
    }
    pp.val = cm.val;
    pp.piece_start = cm.piece_start;
    pp.npieces = cm.npieces;
    pp.eps = eps_;
    pp.partial = partials ? coo_partial_ : nullptr;
    pp.obj = objective ? coo_obj_ : nullptr;
    pp.flags = flags_;
    const int ph = c_.prof_begin(1);
    static const bool old_kernel = [] { const char* e = std::getenv("NTFG_COO_WARP_PER_NNZ"); return e && e[0] == '1'; }();
    if (old_kernel) {  // round-1 kernel (one warp per nonzero), kept for A/B timing
      const int grid = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(cm.npieces, 8), int64_t(c_.sm_count) * 16)));
      if (R_ <= 32) coo_piece_kernel<1><<<grid, 256, 0, c_.stream>>>(pp);
      else coo_piece_kernel<2><<<grid, 256, 0, c_.stream>>>(pp);
    } else {
      const size_t sm = coo_piece2_smem(int(R_));
      static size_t attr = 48 * 1024;
      if (sm > attr) {
        cuda_check(cudaFuncSetAttribute(coo_piece2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)),
                   "cudaFuncSetAttribute");
        attr = sm;
      }
      const int grid = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(cm.npieces, kCooWarps),
                                                                 int64_t(c_.sm_count) * 16)));
      coo_piece2_kernel<<<grid, kCooWarps * 32, sm, c_.stream>>>(pp);
    }
    NTFG_LAUNCHED(c_);
    c_.prof_end(ph);
  }
  // D_1 = [nnz part] + sum_r prod_m colsum(A_m)(r), mean over all entries
  void coo_finish_objective(const double* const* fac) {
    colprod(fac, -1);  // global column sums (the mode-0 part is allreduced when sharded)
    closed_sum_kernel<<<1, 32, 0, c_.stream>>>(colprod_, int(R_), coo_closed_);
    NTFG_LAUNCHED(c_);
    if (sharded_) {  // nnz part: local sum -> allreduce; the closed-form part once
      objective_finalize_kernel<<<1, 256, 0, c_.stream>>>(coo_obj_, int(coo_[0].npieces), 1.0, losses_, counter_,
                                                         raw_);
      NTFG_LAUNCHED(c_);
      allreduce(raw_, 1);
      objective_finalize_kernel<<<1, 32, 0, c_.stream>>>(raw_, 1, 1.0 / double(E_global_), losses_, counter_,
                                                        nullptr, coo_closed_);
      NTFG_LAUNCHED(c_);
      return;
    }
    objective_finalize_kernel<<<1, 256, 0, c_.stream>>>(coo_obj_, int(coo_[0].npieces), 1.0 / double(E_global_),
                                                       losses_, counter_, nullptr, coo_closed_);
    NTFG_LAUNCHED(c_);
  }
  void coo_objective(const double* const* fac) {
    launch_coo_pieces(0, fac, false, true);
    coo_finish_objective(fac);
  }
  // MU step of mode n from Num (numden layout, den closed form in colprod_)
  void coo_finalize(int n, double* num, const double* anchor, const double* ref) {
    FinalizeParams<T> f{};
    f.In = g_.dims[n];
    f.R = int(R_);
    f.RP = RP_;
    f.den_closed = 1;
    f.colprod = colprod_;
    f.phase = 2;
    f.numden = num;
    f.anchor = anchor;
    f.out = A(n);
    f.ref = ref;
    f.stage = n == N_ - 1 ? stage_ : nullptr;
    f.gamma = gamma_;
    f.eps = eps_;
    f.beta = beta_;
    f.flags = flags_;
    finalize_kernel<T><<<int(ceil_div(g_.dims[n] * RP_, 256)), 256, 0, c_.stream>>>(f);
    NTFG_LAUNCHED(c_);
  }
  std::vector<CooMode> coo_;
  bool sparse_ = false;
  bool coo_pending_obj_ = false;
  int64_t coo_nnz_ = 0;
  double* coo_partial_ = nullptr;
  double* coo_obj_ = nullptr;
  double* coo_closed_ = nullptr;

 public:

  double* Aref_all() const { return Aref_; }
  double* anchors() const { return anch_; }
  int64_t offset(int m) const { return off_[m]; }
  bool sharded() const { return sharded_; }
  int64_t max_dim() const {
    int64_t d = 1;
    for (int m = 0; m < N_; ++m) d = std::max(d, g_.dims[m]);
    return d;
  }

  void allreduce(double* buf, size_t count) {
    if (c_.nccl) {  // in place on the engine stream; graph-capturable
      nccl_allreduce_sum(c_.nccl, buf, count, c_.stream);
      return;
    }
    if (!c_.allreduce) return;
    double* target = buf;
    if (c_.comm_buf) {
      if (count > c_.comm_cap) throw Error(NTFG_ERR_COMM, "comm buffer too small");
      c_.d2d(c_.comm_buf, buf, count * sizeof(double));
      target = c_.comm_buf;
    }
    if (c_.allreduce(c_.allreduce_user, target, count, c_.stream) != 0)
      throw Error(NTFG_ERR_COMM, "allreduce hook failed");
    if (target != buf) c_.d2d(buf, target, count * sizeof(double));
  }

 private:
  template <typename K2, typename... P>
  void launch_dyn(K2 kern, dim3 grid, dim3 block, size_t smem, const P&... p) {
    // one attribute call per kernel (keyed by its address: many kernels share
    // a signature, so a per-signature static would miss all but the first)
    static std::mutex mu;
    static std::set<const void*> done;
    {
      std::lock_guard<std::mutex> lock(mu);
      if (done.insert(reinterpret_cast<const void*>(kern)).second)
        cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)),
                   "cudaFuncSetAttribute");
    }
    kern<<<grid, block, smem, c_.stream>>>(p...);
    NTFG_LAUNCHED(c_);
  }

  // tcgen05 reconstruction: the fastest row mode has 128 | I (a 128-row tile
  // then shares the slower coordinates), K = 128..512 in 128 steps
  bool recon_tc_ok(bool row_table = false) const {
    static const bool off = [] { const char* e = std::getenv("NTFG_DISABLE_RECON_TC"); return e && e[0] == '1'; }();
    if (off || sizeof(T) != 4 || N_ < 2 || !g_.small_rows || g_.K % kRcCols != 0 || g_.K / kRcCols > 4) return false;
    return row_table ? g_.rows % kRcRows == 0 : g_.dims[N_ - 2] % kRcRows == 0;
  }
  static bool tile_disabled() {  // perf experiments: NTFG_DISABLE_RTILE=1 keeps recon3
    static const bool v = [] { const char* e = std::getenv("NTFG_DISABLE_RTILE"); return e && e[0] == '1'; }();
    return v;
  }
  template <int RP, int BK, int NPRE>
  void launch_tile_np(const ReconParams<float>& p) {
    constexpr size_t sm = RtSmem<RP>::total;
    static int per_sm = 0;
    static std::mutex mu;
    {
      std::lock_guard<std::mutex> lock(mu);
      if (!per_sm) {
        cuda_check(cudaFuncSetAttribute(recon_tile_kernel<RP, BK, NPRE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(sm)), "cudaFuncSetAttribute");
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, recon_tile_kernel<RP, BK, NPRE>, kRtThreads,
                                                                 sm),
                   "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
        per_sm = std::max(1, std::min(per_sm, 4));
      }
    }
    const int64_t ntiles = ceil_div(g_.rows, int64_t(kRtRows));
    const int64_t per = std::max<int64_t>(1, std::min<int64_t>(ntiles, int64_t(c_.sm_count) * per_sm / p.ktiles));
    recon_grid_ = int(per * p.ktiles);
    recon_tile_kernel<RP, BK, NPRE><<<recon_grid_, kRtThreads, sm, c_.stream>>>(p);
    NTFG_LAUNCHED(c_);
  }
  template <int RP, int BK>
  void launch_tile_bk(const ReconParams<float>& p) {
    // fast H: 1..3 row modes, the fastest with 32 | I (tiles never straddle its blocks)
    const int npre = N_ - 1;
    const bool fast = npre >= 1 && npre <= 3 && g_.dims[npre - 1] % kRtRows == 0 && g_.small_rows;
    if (!fast) launch_tile_np<RP, BK, 0>(p);
    else if (npre == 1) launch_tile_np<RP, BK, 1>(p);
    else if (npre == 2) launch_tile_np<RP, BK, 2>(p);
    else launch_tile_np<RP, BK, 3>(p);
  }
  template <int RP>
  void launch_tile(const ReconParams<T>& pp) {
    if constexpr (sizeof(T) == 4) {
      const ReconParams<float>& p = pp;
      switch (bk_) {
        case kBeta1: launch_tile_bk<RP, kBeta1>(p); break;
        case kBetaHalf: launch_tile_bk<RP, kBetaHalf>(p); break;
        case kBeta3Half: launch_tile_bk<RP, kBeta3Half>(p); break;
        case kBeta0: launch_tile_bk<RP, kBeta0>(p); break;
        default: launch_tile_bk<RP, kBetaGeneric>(p); break;
      }
    }
  }
  template <int RP>
  void launch_recon(const ReconParams<T>& p) {
    constexpr int KT2 = (sizeof(T) == 4 && RP <= 32) ? 2 : 1;
    const dim3 grid(recon_grid_);
    if (recon_v3_) {
      constexpr int K3 = sizeof(T) == 4 ? (RP <= 16 ? 4 : RP <= 32 ? 2 : 1) : (RP <= 16 ? 2 : 1);
      if constexpr (sizeof(T) == 4) {
        if (planes_out_ && !p.pout && !p.xhout) {
          constexpr size_t sm = R3Smem<T, RP, K3>::total;
          switch (bk_) {
            case kBeta1: launch_dyn(recon3_kernel<T, RP, K3, kBeta1>, grid, dim3(128), sm, p); return;
            case kBetaHalf: launch_dyn(recon3_kernel<T, RP, K3, kBetaHalf>, grid, dim3(128), sm, p); return;
            case kBeta3Half: launch_dyn(recon3_kernel<T, RP, K3, kBeta3Half>, grid, dim3(128), sm, p); return;
            case kBeta0: launch_dyn(recon3_kernel<T, RP, K3, kBeta0>, grid, dim3(128), sm, p); return;
            default: launch_dyn(recon3_kernel<T, RP, K3, kBetaGeneric>, grid, dim3(128), sm, p); return;
          }
        }
      }
      launch_dyn(recon3_kernel<T, RP, K3>, grid, dim3(128), R3Smem<T, RP, K3>::total, p);
      return;
    }
    if (recon_kt() == 2) {
      if constexpr (KT2 == 2) {
        if (recon_tpb() == 256) launch_dyn(recon2_kernel<T, RP, 2, 256>, grid, dim3(256), recon2_smem<T, 2, 256>(), p);
        else launch_dyn(recon2_kernel<T, RP, 2, 128>, grid, dim3(128), recon2_smem<T, 2, 128>(), p);
        return;
      }
    }
    if (recon_tpb() == 256) launch_dyn(recon2_kernel<T, RP, 1, 256>, grid, dim3(256), recon2_smem<T, 1, 256>(), p);
    else launch_dyn(recon2_kernel<T, RP, 1, 128>, grid, dim3(128), recon2_smem<T, 1, 128>(), p);
  }

  template <int NS>
  void fill_contract(ContractParams<T, NS>& p, int n, int r0, bool caseA, int64_t units, int64_t S,
                     int64_t An, int64_t Bn, T* partA, double* partB, int ktiles, const Stream* st,
                     int ns) {
    p.g = g_;
    p.n = n;
    p.R = int(R_);
    p.RP = RP_;
    p.r0 = r0;
    for (int s = 0; s < ns; ++s) {
      p.src[s] = st[s].src;
      for (int m = 0; m < N_; ++m) p.mfac[s][m] = st[s].fac[m];
      p.lastfac[s] = st[s].fac[N_ - 1];
      p.mtab[s] = st[s].mtab;
    }
    p.caseA = caseA;
    p.units = units;
    p.S = S;
    p.An = An;
    p.Bn = Bn;
    p.fB.init(Bn);
    p.partA = partA;
    p.partB = partB;
    p.ktiles = ktiles;
  }

  template <int NS, int RC, int KT, int TPS>
  void launch_c2(const ContractParams<T, NS>& p, int grid) {
    launch_dyn(contract2_kernel<T, RC, KT, NS, TPS>, dim3(grid), dim3(NS * TPS),
               contract2_smem<T, RC, KT, NS, TPS>(), p);
  }
  template <int NS, int RC, int KT>
  void launch_c2t(const ContractParams<T, NS>& p, const Plan& pl, int grid) {
    if (pl.TPS == 256) launch_c2<NS, RC, KT, 256>(p, grid);
    else launch_c2<NS, RC, KT, 128>(p, grid);
  }

  template <int NS, int RC, int KT>
  void launch_c3(const ContractParams<T, NS>& p, int grid) {
    launch_dyn(contract3_kernel<T, RC, KT, NS>, dim3(grid), dim3(NS * 128), C3Smem<T, RC, KT, NS>::total, p);
  }

  template <int NS>
  void launch_contract(const ContractParams<T, NS>& p, const Plan& pl, int grid) {
    if (pl.v3) {
      if constexpr (sizeof(T) == 4) {
        switch (pl.RC) {
          case 8: launch_c3<NS, 8, 4>(p, grid); break;
          case 16: launch_c3<NS, 16, 4>(p, grid); break;
          case 32: launch_c3<NS, 32, 4>(p, grid); break;
          default: launch_c3<NS, 64, 1>(p, grid); break;
        }
      } else {
        switch (pl.RC) {
          case 8: launch_c3<NS, 8, 2>(p, grid); break;
          case 16: launch_c3<NS, 16, 2>(p, grid); break;
          default: launch_c3<NS, 32, 2>(p, grid); break;
        }
      }
      return;
    }
    if constexpr (sizeof(T) == 4) {
      if (pl.KT == 2) {
        switch (pl.RC) {
          case 8: launch_c2t<NS, 8, 2>(p, pl, grid); break;
          case 16: launch_c2t<NS, 16, 2>(p, pl, grid); break;
          default: launch_c2t<NS, 32, 2>(p, pl, grid); break;
        }
      } else {
        switch (pl.RC) {
          case 8: launch_c2t<NS, 8, 1>(p, pl, grid); break;
          case 16: launch_c2t<NS, 16, 1>(p, pl, grid); break;
          case 32: launch_c2t<NS, 32, 1>(p, pl, grid); break;
          default: launch_c2t<NS, 64, 1>(p, pl, grid); break;
        }
      }
    } else {
      switch (pl.RC) {
        case 8: launch_c2t<NS, 8, 1>(p, pl, grid); break;
        case 16: launch_c2t<NS, 16, 1>(p, pl, grid); break;
        default: launch_c2t<NS, 32, 1>(p, pl, grid); break;
      }
    }
  }

  Context& c_;
  int N_;
  int64_t R_;
  int RP_;
  double beta_, eps_, gamma_;
  int bk_;
  Geom g_{};
  int64_t E_, E_global_;
  bool sharded_ = false;
  std::vector<int64_t> off_;
  const T* x_ = nullptr;
  T* p_ = nullptr;
  T* q_ = nullptr;
  double *A_, *Aref_, *chi1_, *chi2_, *anch_;
  T *stage_, *stage_anchor_;
  double *colsum_, *colprod_, *objpart_, *raw_, *numden_;
  double* losses_ = nullptr;
  T* partA_ = nullptr;
  double* partB_ = nullptr;
  double* partAd_ = nullptr;
  double* n1num_ = nullptr;
  bool n1_enabled_ = true;
  bool tc_ = false;
  bool tc_allowed_ = true;
  bool planes_out_ = false;
  void* planes_[4] = {nullptr, nullptr, nullptr, nullptr};
  float* lastT_ = nullptr;
  unsigned char* btiles_ = nullptr;  // static B tiles of the tensor-core contraction (tc_contract.cuh)
  float* hstage_ = nullptr;   // fp32 copy of the fastest row mode's factor (recon_tc H producers)
  unsigned* flags_;
  int* counter_;
  int* colsum_done_;  // arrival counter of the fused colsum + colprod launch (self re-arming)
  int recon_grid_ = 0;
  bool recon_v3_ = false;
  bool obj_split_ = false;    // last recon used the split objective (needs xconst_)
  double* xconst_ = nullptr;  // [0] = x-only objective constant, [1..] partials
  static constexpr int kXconstGrid = 592;
};

}  // namespace ntfg
