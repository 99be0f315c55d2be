// Tucker entry points of the C ABI (fit drivers and step-level functions).
// Reference: include/ntf/tucker.hpp, src/tucker.cpp, src/tensor.cpp:408-560.
#include <algorithm>
#include <cmath>
#include <functional>
#include <vector>

#include "fit_loop.cuh"
#include "tucker_engine.cuh"

namespace ntfg {

namespace {

std::vector<double> nesterov_alphas_t(uint64_t K) {
  std::vector<double> a(K + 1);
  double t = 1.0;
  for (uint64_t k = 0; k <= K; ++k) {
    const double tn = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * t * t));
    a[k] = (t - 1.0) / tn;
    t = tn;
  }
  return a;
}

void check_positive(const double* f, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!(f[i] > 0.0)) throw Error(NTFG_ERR_DOMAIN, "chi1: entries must be strictly positive");
}

const uint64_t* checked_ranks(const ntfg_fit_config& cfg, uint32_t order) {
  if (cfg.n_ranks != order || !cfg.ranks)
    throw Error(NTFG_ERR_SHAPE, "TuckerModel: core order does not match factor count");
  return cfg.ranks;
}

template <typename T>
std::vector<ntfg_trace_row> tucker_fit_t(Context& c, const ntfg_fit_config& cfg, int algo, uint32_t order,
                                         const uint64_t* dims, const void* x, int dtype, int loc,
                                         const ntfg_shard* shard, double* core, double* factors) {
  const uint64_t* ranks = checked_ranks(cfg, order);
  TuckerEngine<T> e(c, order, dims, ranks, cfg.beta, cfg.eps, shard);
  const size_t B = e.model_doubles();
  if (algo == NTFG_JCOMM) {
    check_positive(core, size_t(e.core_size()));
    check_positive(factors, B - size_t(e.core_size()));
  }
  e.stream().set_x(x, dtype, loc);
  e.set_model_host(core, factors);
  e.stream().prealloc(2);
  e.stream().q_always();
  double* losses = c.buf<double>("fit.losses", cfg.max_iters + 2);
  e.stream().bind_losses(losses);
  e.stream().reset_counter();
  e.stream().reset_flags();
  const size_t bytes = B * sizeof(double);
  const int L = int(cfg.inner_steps);
  LoopHooks h;
  h.fused = !cfg.extrapolate;
  h.objective = [&]() { e.objective(); };
  if (cfg.extrapolate) {
    double* prev = c.buf<double>("tk.prev", B);
    double* alpha = c.buf<double>("tk.alpha", 3);  // [alpha | norm^2 shard | rest]
    int* iter = c.buf<int>("tk.iter", 1);
    const auto an = nesterov_alphas_t(cfg.max_iters);
    double* alpha_nes = c.buf<double>("tk.alpha_nes", an.size());
    c.h2d(alpha_nes, an.data(), an.size() * sizeof(double));
    c.d2d(prev, e.model(), bytes);
    NTFG_CUDA(cudaMemsetAsync(iter, 0, sizeof(int), c.stream));
    c.sync();
    h.body = [&e, &c, &cfg, prev, alpha, iter, alpha_nes, B, bytes, algo, L]() {
      // [core | A_0 | A_1 ...]: A_0's rows are this rank's shard when data-parallel
      const bool sh = e.stream().sharded();
      const int64_t s0 = sh ? e.core_size() : 0;
      const int64_t s1 = sh ? e.core_size() + e.factor_offset(1) : 0;
      extrap_norm_kernel<<<1, 256, 0, c.stream>>>(e.model(), prev, int64_t(B), s0, s1, alpha + 1);
      NTFG_LAUNCHED(c);
      if (sh) e.stream().allreduce(alpha + 1, 1);
      extrap_alpha_finish_kernel<<<1, 1, 0, c.stream>>>(alpha + 1, alpha_nes, iter, cfg.extrap_cap,
                                                        cfg.extrap_delta, alpha);
      NTFG_LAUNCHED(c);
      extrap_apply_kernel<<<int(ceil_div(int64_t(B), 256)), 256, 0, c.stream>>>(
          e.model(), prev, int64_t(B), alpha, cfg.eps, e.anchors());
      NTFG_LAUNCHED(c);
      c.d2d(prev, e.model(), bytes);
      if (algo == NTFG_BCOMM) {
        e.bcomm_sweep_anchored(e.anchors());
      } else {
        c.d2d(e.model(), e.anchors(), bytes);
        e.restage();
        e.jcomm_outer(L, false);
      }
      e.objective();
    };
  } else {
    double* snap = c.buf<double>("tk.snap", B);
    h.snapshot = [&e, &c, snap, bytes]() { c.d2d(snap, e.model(), bytes); };
    h.restore = [&e, &c, snap, bytes]() {
      c.d2d(e.model(), snap, bytes);
      e.restage();
    };
    h.body = [&e, algo, L]() {
      if (algo == NTFG_BCOMM) e.bcomm_sweep(true);
      else e.jcomm_outer(L, true);
    };
  }
  auto trace = run_fit_loop(c, cfg, h, losses, e.stream().flags());
  e.get_model_host(core, factors);
  c.sync();
  return trace;
}

template <typename T>
void with_tucker(Context& c, uint32_t order, const uint64_t* dims, const uint64_t* ranks, double beta,
                 double eps, const std::function<void(TuckerEngine<T>&)>& fn) {
  TuckerEngine<T> e(c, order, dims, ranks, beta, eps, nullptr);
  double* losses = c.buf<double>("step.losses", 4);
  e.stream().bind_losses(losses);
  e.stream().reset_counter();
  e.stream().reset_flags();
  fn(e);
  c.sync();
  unsigned f = 0;
  NTFG_CUDA(cudaMemcpy(&f, e.stream().flags(), sizeof(unsigned), cudaMemcpyDeviceToHost));
  raise_flags(f);
}

#define NTFG_TDISPATCH(prec, body) \
  do {                             \
    if ((prec) == NTFG_F32) {      \
      using T = float;             \
      body;                        \
    } else {                       \
      using T = double;            \
      body;                        \
    }                              \
  } while (0)

template <typename T>
void upload_t(Context& c, T* dst, const double* src, size_t n) {
  if (sizeof(T) == 8) {
    c.h2d(dst, src, n * sizeof(double));
  } else {
    std::vector<T> h(src, src + n);
    c.h2d(dst, h.data(), n * sizeof(T));
    c.sync();
  }
}

}  // namespace

void tucker_fit(Context& c, const ntfg_fit_config& cfg, int algo, uint32_t order, const uint64_t* dims,
                const void* x, int dtype, int loc, const ntfg_shard* shard, double* core,
                double* factors, ntfg_trace_row* trace, uint64_t* trace_len) {
  validate_config(cfg);
  if (algo != NTFG_BCOMM && algo != NTFG_JCOMM) throw Error(NTFG_ERR_DOMAIN, "unknown algorithm");
  c.stats = ntfg_stats{};
  std::vector<ntfg_trace_row> tr =
      cfg.precision == NTFG_F32
          ? tucker_fit_t<float>(c, cfg, algo, order, dims, x, dtype, loc, shard, core, factors)
          : tucker_fit_t<double>(c, cfg, algo, order, dims, x, dtype, loc, shard, core, factors);
  for (size_t i = 0; i < tr.size(); ++i) trace[i] = tr[i];
  *trace_len = tr.size();
}

void tucker_reconstruct(Context& c, int prec, uint32_t order, const uint64_t* dims, const uint64_t* ranks,
                        const double* core, const double* factors, double* out) {
  NTFG_TDISPATCH(prec, {
    with_tucker<T>(c, order, dims, ranks, 1.0, 1e-12, [&](TuckerEngine<T>& e) {
      e.set_model_host(core, factors);
      auto& s = e.stream();
      const int64_t E = s.entries();
      T* xh = c.buf<T>("step.xhat", size_t(E));
      s.set_x(xh, sizeof(T) == 4 ? 1 : 0, NTFG_DEVICE);
      const double* fac[kMaxOrder];
      for (uint32_t m = 0; m < order; ++m) fac[m] = e.A(int(m));
      double* Y = c.buf<double>("tk.Y1", 1);  // same buffer the engine owns
      e.ychain(e.G(), fac, Y);
      s.stage(e.A(int(order) - 1), c.buf<T>("tk.stageL", 1));
      s.recon(fac, c.buf<T>("tk.stageL", 1), nullptr, nullptr, false, xh, Y);
      std::vector<T> h(static_cast<size_t>(E));
      c.d2h(h.data(), xh, h.size() * sizeof(T));
      c.sync();
      for (size_t i = 0; i < h.size(); ++i) out[i] = double(h[i]);
    });
  });
}

// tucker_multimode_contract with optional skip (skip < 0: none)
void tucker_multimode_contract(Context& c, int prec, uint32_t order, const uint64_t* dims, const double* t,
                               const uint64_t* cols, const double* factors, int32_t skip, double* out) {
  if (skip >= int32_t(order)) throw Error(NTFG_ERR_SHAPE, "tucker_multimode_contract: skip mode out of range");
  // identity core of shape cols (only used by contract_factor's pairing);
  // the plain multimode contraction needs no core.
  std::vector<uint64_t> ranks(cols, cols + order);
  NTFG_TDISPATCH(prec, {
    with_tucker<T>(c, order, dims, ranks.data(), 1.0, 1e-12, [&](TuckerEngine<T>& e) {
      size_t F = 0;
      for (uint32_t m = 0; m < order; ++m) F += dims[m] * cols[m];
      std::vector<double> zero_core(size_t(e.core_size()), 0.0);
      e.set_model_host(zero_core.data(), factors);
      auto& s = e.stream();
      T* td = c.buf<T>("step.t", size_t(s.entries()));
      upload_t<T>(c, td, t, size_t(s.entries()));
      const double* fac[kMaxOrder];
      for (uint32_t m = 0; m < order; ++m) fac[m] = e.A(int(m));
      if (skip < 0) {
        e.contract_core(td, fac, e.num());
        c.d2h(out, e.num(), size_t(e.core_size()) * sizeof(double));
      } else {
        // keep mode `skip`: chain over every other mode on the full tensor
        // (step-level API; the solvers use the fused factor path instead)
        const int64_t E = s.entries();
        int64_t big = E;
        {
          int64_t sz = E;
          for (uint32_t m = 0; m < order; ++m)
            if (int32_t(m) != skip) { sz = sz / int64_t(dims[m]) * int64_t(cols[m]); big = std::max(big, sz); }
        }
        double* w1 = c.buf<double>("mm.w1", size_t(big));
        double* w2 = c.buf<double>("mm.w2", size_t(big));
        c.h2d(w1, t, size_t(E) * sizeof(double));
        std::vector<int64_t> shape(dims, dims + order);
        double* cur = w1;
        double* nxt = w2;
        for (uint32_t m = 0; m < order; ++m) {
          if (int32_t(m) == skip) continue;
          e.ttm(cur, shape, int(m), fac[m], int64_t(cols[m]), 1, nxt);
          std::swap(cur, nxt);
        }
        int64_t outer = 1, inner = 1;
        for (int32_t a = 0; a < skip; ++a) outer *= shape[size_t(a)];
        for (uint32_t a = uint32_t(skip) + 1; a < order; ++a) inner *= shape[a];
        const int64_t total = outer * shape[size_t(skip)] * inner;
        moveaxis_last_kernel<<<int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), 4096))), 256, 0,
                               c.stream>>>(cur, outer, shape[size_t(skip)], inner, nxt);
        NTFG_LAUNCHED(c);
        c.d2h(out, nxt, size_t(total) * sizeof(double));
      }
    });
  });
}

void tucker_factor_contract(Context& c, int prec, uint32_t order, const uint64_t* dims, const double* t,
                            const uint64_t* ranks, const double* core, const double* factors, uint32_t mode,
                            double* out) {
  if (mode >= order) throw Error(NTFG_ERR_SHAPE, "tucker_factor_contract: mode out of range");
  NTFG_TDISPATCH(prec, {
    with_tucker<T>(c, order, dims, ranks, 0.5, 1e-12, [&](TuckerEngine<T>& e) {
      e.set_model_host(core, factors);
      auto& s = e.stream();
      T* td = s.q_always();  // reuse the Q scratch as the contracted stream
      upload_t<T>(c, td, t, size_t(s.entries()));
      const double* fac[kMaxOrder];
      for (uint32_t m = 0; m < order; ++m) fac[m] = e.A(int(m));
      const int L = int(order) - 1;
      if (int(mode) < L) {
        e.contract_factor(td, e.G(), fac, int(mode), e.num());
        c.d2h(out, e.num(), size_t(dims[mode] * ranks[mode]) * sizeof(double));
      } else {
        // last mode: Num(k, j) = sum_rows T(row,k) Y(row,j) via the case-A contraction
        double* Y = c.buf<double>("tk.Y1", 1);
        e.ychain(e.G(), fac, Y);
        typename CpEngine<T>::Stream st[2];
        st[0].src = td;
        for (uint32_t m = 0; m < order; ++m) st[0].fac[m] = fac[m];
        st[0].mtab = Y;
        double* junk = c.buf<double>("step.junk", size_t(dims[mode] * ranks[mode]));
        s.prealloc(1);
        s.contract_numden(L, st, junk);
        c.d2h(out, s.numden(), size_t(dims[mode] * ranks[mode]) * sizeof(double));
      }
    });
  });
}

void tucker_objective(Context& c, int prec, double beta, uint32_t order, const uint64_t* dims, const double* x,
                      const uint64_t* ranks, const double* core, const double* factors, double* mean_out) {
  gamma_of(beta);
  NTFG_TDISPATCH(prec, {
    with_tucker<T>(c, order, dims, ranks, beta, 1e-12, [&](TuckerEngine<T>& e) {
      e.stream().set_x(x, 0, NTFG_HOST);
      e.set_model_host(core, factors);
      e.objective();
    });
    NTFG_CUDA(cudaMemcpy(mean_out, c.buf<double>("step.losses", 4), sizeof(double), cudaMemcpyDeviceToHost));
  });
}

void tucker_jcomm_reference(Context& c, int prec, double beta, double eps, uint32_t order, const uint64_t* dims,
                            const double* x, const uint64_t* ranks, const double* ref_core, const double* ref_factors,
                            double* p_out, double* q_out) {
  NTFG_TDISPATCH(prec, {
    with_tucker<T>(c, order, dims, ranks, beta, eps, [&](TuckerEngine<T>& e) {
      e.stream().set_x(x, 0, NTFG_HOST);
      e.set_model_host(ref_core, ref_factors);
      e.set_ref_host(ref_core, ref_factors);
      e.stream().prealloc(2);
      e.weights_of_ref();
      const size_t E = size_t(e.stream().entries());
      std::vector<T> h(E);
      c.d2h(h.data(), e.stream().p(), E * sizeof(T));
      c.sync();
      for (size_t i = 0; i < E; ++i) p_out[i] = double(h[i]);
      c.d2h(h.data(), e.stream().q_always(), E * sizeof(T));
      c.sync();
      for (size_t i = 0; i < E; ++i) q_out[i] = double(h[i]);
    });
  });
}

void tucker_jcomm_inner_update(Context& c, int prec, double beta, double eps, uint32_t order, const uint64_t* dims,
                               const double* p, const double* q, const uint64_t* ranks, const double* ref_core,
                               const double* ref_factors, double* core, double* factors, int32_t block) {
  if (block >= int32_t(order)) throw Error(NTFG_ERR_SHAPE, "jcomm_inner_factor_update: mode out of range");
  NTFG_TDISPATCH(prec, {
    with_tucker<T>(c, order, dims, ranks, beta, eps, [&](TuckerEngine<T>& e) {
      e.set_model_host(core, factors);
      e.set_ref_host(ref_core, ref_factors);
      e.stream().prealloc(2);
      const size_t E = size_t(e.stream().entries());
      upload_t<T>(c, e.stream().p(), p, E);
      upload_t<T>(c, e.stream().q_always(), q, E);
      e.chi_from_ref();
      if (block < 0) e.jcomm_inner_core();
      else e.jcomm_inner_factor(int(block));
      e.get_model_host(core, factors);
    });
  });
}

void tucker_step(Context& c, int prec, int kind, double beta, double eps, uint64_t inner, uint32_t order,
                 const uint64_t* dims, const double* x, const uint64_t* ranks, const double* ref_core,
                 const double* ref_factors, double* core, double* factors, uint32_t mode) {
  if ((kind == 1 || kind == 5) && mode >= order)
    throw Error(NTFG_ERR_SHAPE, "block_factor_update: mode out of range");
  if (kind == 3 && inner < 1) throw Error(NTFG_ERR_DOMAIN, "jcomm_tucker_outer_step: inner_steps must be >= 1");
  if ((kind == 4 || kind == 5) && (!ref_core || !ref_factors))
    throw Error(NTFG_ERR_SHAPE, "reference model required");
  if ((kind == 6 && !ref_core) || (kind == 7 && (!ref_factors || mode >= order)))
    throw Error(NTFG_ERR_SHAPE, "anchor required");
  NTFG_TDISPATCH(prec, {
    with_tucker<T>(c, order, dims, ranks, beta, eps, [&](TuckerEngine<T>& e) {
      e.stream().set_x(x, 0, NTFG_HOST);
      e.set_model_host(core, factors);
      e.stream().prealloc(2);
      switch (kind) {
        case 0: e.block_core(e.G(), false); break;
        case 1: e.block_factor(int(mode), e.A(int(mode))); break;
        case 2: e.bcomm_sweep(false); break;
        case 3:
          check_positive(core, size_t(e.core_size()));
          e.jcomm_outer(int(inner), false);
          break;
        case 6: {  // block_core_update_anchored: ref_core is the anchor core
          c.h2d(e.anchors(), ref_core, size_t(e.core_size()) * sizeof(double));
          e.block_core(e.anchors(), false);
          break;
        }
        case 7: {  // block_factor_update_anchored: ref_factors is the anchor block of `mode`
          double* anc = e.anchors() + e.core_size() + e.factor_offset(int(mode));
          c.h2d(anc, ref_factors, size_t(dims[mode] * ranks[mode]) * sizeof(double));
          e.block_factor(int(mode), anc);
          break;
        }
        case 4:
        case 5:
          e.set_ref_host(ref_core, ref_factors);
          e.weights_of_ref();
          e.chi_from_ref();
          if (kind == 4) e.jcomm_inner_core();
          else e.jcomm_inner_factor(int(mode));
          break;
        default: throw Error(NTFG_ERR_DOMAIN, "unknown tucker step kind");
      }
      e.get_model_host(core, factors);
    });
  });
}

}  // namespace ntfg
