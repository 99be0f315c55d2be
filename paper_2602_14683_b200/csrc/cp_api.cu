// CP entry points of the C ABI (fit drivers and step-level functions).
// Reference: include/ntf/cp.hpp, src/cp.cpp; see include/ntfg.h for the
// per-function mapping.
#include <cmath>
#include <functional>
#include <vector>

#include "cp_engine.cuh"
#include "fit_loop.cuh"

namespace ntfg {

namespace {

void check_positive_host(const double* f, size_t n, const char* what) {
  for (size_t i = 0; i < n; ++i)
    if (!(f[i] > 0.0)) throw Error(NTFG_ERR_DOMAIN, std::string(what) + ": entries must be strictly positive");
}

std::vector<double> nesterov_alphas(uint64_t K) {
  // t_0 = 1, t_{k+1} = (1 + sqrt(1 + 4 t_k^2)) / 2, alpha_k = (t_k - 1) / t_{k+1}
  // (reference cp.cpp:158-163)
  std::vector<double> a(K + 1);
  double t = 1.0;
  for (uint64_t k = 0; k <= K; ++k) {
    const double tn = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * t * t));
    a[k] = (t - 1.0) / tn;
    t = tn;
  }
  return a;
}

template <typename T>
std::vector<ntfg_trace_row> cp_fit_t(Context& c, const ntfg_fit_config& cfg, int algo,
                                     uint32_t order, const uint64_t* dims,
                                     const std::function<void(CpEngine<T>&)>& set_data,
                                     const ntfg_shard* shard, double* factors) {
  CpEngine<T> e(c, order, dims, int64_t(cfg.rank), cfg.beta, cfg.eps, shard);
  if (algo == NTFG_JCOMM) check_positive_host(factors, e.factor_doubles(), "chi1");
  set_data(e);
  e.set_factors_host(factors);
  e.prealloc(cfg.beta == 1.0 ? 1 : 2);
  double* losses = c.buf<double>("fit.losses", cfg.max_iters + 2);
  e.bind_losses(losses);
  e.reset_counter();
  e.reset_flags();

  const size_t F = e.factor_doubles();
  const size_t bytes = F * sizeof(double);
  const int L = int(cfg.inner_steps);
  LoopHooks h;
  h.fused = !cfg.extrapolate;
  h.objective = [&]() { e.objective(); };
  if (cfg.extrapolate) {
    // BMMe (reference cp.cpp:249-263 / 276-292): prev = init, t_0 = 1
    double* prev = c.buf<double>("cp.prev", F);
    double* alpha = c.buf<double>("cp.alpha", 3);  // [alpha | norm^2 shard | rest]
    int* iter = c.buf<int>("cp.iter", 1);
    const auto an = nesterov_alphas(cfg.max_iters);
    double* alpha_nes = c.buf<double>("cp.alpha_nes", an.size());
    c.h2d(alpha_nes, an.data(), an.size() * sizeof(double));
    c.d2d(prev, e.A_all(), bytes);
    NTFG_CUDA(cudaMemsetAsync(iter, 0, sizeof(int), c.stream));
    c.sync();  // alpha_nes host vector goes out of scope
    h.body = [&e, &c, &cfg, prev, alpha, iter, alpha_nes, F, bytes, algo, L]() {
      // mode-0 rows [0, I0_local * R) are this rank's shard when data-parallel
      const int64_t s1 = e.sharded() ? e.offset(1) : 0;
      extrap_norm_kernel<<<1, 256, 0, c.stream>>>(e.A_all(), prev, int64_t(F), 0, s1, alpha + 1);
      NTFG_LAUNCHED(c);
      if (e.sharded()) e.allreduce(alpha + 1, 1);
      extrap_alpha_finish_kernel<<<1, 1, 0, c.stream>>>(alpha + 1, alpha_nes, iter, cfg.extrap_cap,
                                                        cfg.extrap_delta, alpha);
      NTFG_LAUNCHED(c);
      extrap_apply_kernel<<<int(ceil_div(int64_t(F), 256)), 256, 0, c.stream>>>(
          e.A_all(), prev, int64_t(F), alpha, cfg.eps, e.anchors());
      NTFG_LAUNCHED(c);
      c.d2d(prev, e.A_all(), bytes);  // previous := snapshot of this iterate
      if (algo == NTFG_BCOMM) {
        e.bcomm_sweep_anchored(e.anchors());
      } else {
        c.d2d(e.A_all(), e.anchors(), bytes);  // reference = extrapolated point
        e.restage();
        e.jcomm_outer(L, false);
      }
      e.objective();
    };
  } else {
    double* snap = c.buf<double>("cp.snap", F);
    h.snapshot = [&e, &c, snap, bytes]() { c.d2d(snap, e.A_all(), bytes); };
    h.restore = [&e, &c, snap, bytes]() {
      c.d2d(e.A_all(), snap, bytes);
      e.restage();
    };
    h.body = [&e, algo, L]() {
      if (algo == NTFG_BCOMM) e.bcomm_sweep(true);
      else e.jcomm_outer(L, true);
    };
  }
  auto trace = run_fit_loop(c, cfg, h, losses, e.flags());
  e.get_factors_host(factors);
  c.sync();
  return trace;
}

template <typename T>
struct StepCtx {
  CpEngine<T> e;
  StepCtx(Context& c, uint32_t order, const uint64_t* dims, uint64_t rank, double beta, double eps)
      : e(c, order, dims, int64_t(rank), beta, eps, nullptr) {}
};

}  // namespace

void cp_fit(Context& c, const ntfg_fit_config& cfg, int algo, uint32_t order, const uint64_t* dims,
            const void* x, int dtype, int loc, const ntfg_shard* shard, double* factors,
            ntfg_trace_row* trace, uint64_t* trace_len) {
  validate_config(cfg);
  if (algo != NTFG_BCOMM && algo != NTFG_JCOMM) throw Error(NTFG_ERR_DOMAIN, "unknown algorithm");
  c.stats = ntfg_stats{};
  std::vector<ntfg_trace_row> tr =
      cfg.precision == NTFG_F32
          ? cp_fit_t<float>(c, cfg, algo, order, dims, [&](CpEngine<float>& e) { e.set_x(x, dtype, loc); },
                            shard, factors)
          : cp_fit_t<double>(c, cfg, algo, order, dims, [&](CpEngine<double>& e) { e.set_x(x, dtype, loc); },
                             shard, factors);
  for (size_t i = 0; i < tr.size(); ++i) trace[i] = tr[i];
  *trace_len = tr.size();
}

// sparse COO fit at beta = 1 (K7, coo_kernels.cuh): all passes in fp64
// whatever cfg.precision says (the nonzero pass is latency-bound, not
// bandwidth-bound, so fp32 storage buys nothing).
void cp_fit_coo(Context& c, const ntfg_fit_config& cfg, int algo, uint32_t order, const uint64_t* dims,
                uint64_t nnz, const int32_t* indices, const void* values, int dtype, int loc, const ntfg_shard* shard,
                double* factors, ntfg_trace_row* trace, uint64_t* trace_len) {
  validate_config(cfg);
  if (algo != NTFG_BCOMM && algo != NTFG_JCOMM) throw Error(NTFG_ERR_DOMAIN, "unknown algorithm");
  c.stats = ntfg_stats{};
  std::vector<ntfg_trace_row> tr = cp_fit_t<double>(
      c, cfg, algo, order, dims,
      [&](CpEngine<double>& e) { e.set_coo(nnz, indices, values, dtype, loc); }, shard, factors);
  for (size_t i = 0; i < tr.size(); ++i) trace[i] = tr[i];
  *trace_len = tr.size();
}

// ---- step level --------------------------------------------------------------------

template <typename T>
static void with_engine(Context& c, int prec, uint32_t order, const uint64_t* dims, uint64_t rank,
                        double beta, double eps, const std::function<void(CpEngine<T>&)>& fn) {
  CpEngine<T> e(c, order, dims, int64_t(rank), beta, eps, nullptr);
  double* losses = c.buf<double>("step.losses", 4);
  e.bind_losses(losses);
  e.reset_counter();
  e.reset_flags();
  fn(e);
  c.sync();
  unsigned f = 0;
  NTFG_CUDA(cudaMemcpy(&f, e.flags(), sizeof(unsigned), cudaMemcpyDeviceToHost));
  raise_flags(f);
}

#define NTFG_DISPATCH(prec, body)            \
  do {                                       \
    if ((prec) == NTFG_F32) {                \
      using T = float;                       \
      body;                                  \
    } else {                                 \
      using T = double;                      \
      body;                                  \
    }                                        \
  } while (0)

void cp_reconstruct(Context& c, int prec, uint32_t order, const uint64_t* dims, uint64_t rank,
                    const double* factors, double* out) {
  NTFG_DISPATCH(prec, {
    with_engine<T>(c, prec, order, dims, rank, 1.0, 1e-12, [&](CpEngine<T>& e) {
      e.set_factors_host(factors);
      T* xh = c.buf<T>("step.xhat", size_t(e.entries()));
      // x is unused without weights/objective; point it at the output
      e.set_x(xh, sizeof(T) == 4 ? 1 : 0, NTFG_DEVICE);
      const double* fac[kMaxOrder];
      for (int m = 0; m < e.order(); ++m) fac[m] = e.A(m);
      e.recon(fac, e.stage_last(), nullptr, nullptr, false, xh);
      std::vector<T> h(size_t(e.entries()));
      c.d2h(h.data(), xh, h.size() * sizeof(T));
      c.sync();
      for (size_t i = 0; i < h.size(); ++i) out[i] = double(h[i]);
    });
  });
}

void cp_contract(Context& c, int prec, uint32_t order, const uint64_t* dims, const double* t,
                 uint64_t rank, const double* factors, uint32_t mode, double* out) {
  if (mode >= order) throw Error(NTFG_ERR_SHAPE, "cp_contract: mode out of range");
  NTFG_DISPATCH(prec, {
    with_engine<T>(c, prec, order, dims, rank, 0.5, 1e-12, [&](CpEngine<T>& e) {
      e.set_factors_host(factors);
      T* td = c.buf<T>("step.t", size_t(e.entries()));
      e.upload_convert(td, t, 0, NTFG_HOST, e.entries());
      typename CpEngine<T>::Stream st[2];
      st[0].src = td;
      st[1].src = td;
      for (int m = 0; m < e.order(); ++m) st[0].fac[m] = st[1].fac[m] = e.A(m);
      // MU output goes to scratch; numden holds the raw contraction (phase 1)
      double* junk = c.buf<double>("step.junk", size_t(e.dim(mode)) * rank);
      e.contract_numden(int(mode), st, junk);
      c.d2h(out, e.numden(), size_t(e.dim(mode)) * rank * sizeof(double));
    });
  });
}

void cp_objective(Context& c, int prec, double beta, uint32_t order, const uint64_t* dims,
                  const double* x, uint64_t rank, const double* factors, double* mean_out) {
  gamma_of(beta);
  NTFG_DISPATCH(prec, {
    with_engine<T>(c, prec, order, dims, rank, beta, 1e-12, [&](CpEngine<T>& e) {
      e.set_x(x, 0, NTFG_HOST);
      e.set_factors_host(factors);
      e.objective();
      c.sync();
    });
    NTFG_CUDA(cudaMemcpy(mean_out, c.buf<double>("step.losses", 4), sizeof(double), cudaMemcpyDeviceToHost));
  });
}

void cp_block_update(Context& c, int prec, double beta, double eps, uint32_t order,
                     const uint64_t* dims, const double* x, uint64_t rank, double* factors,
                     uint32_t mode, const double* anchor) {
  if (mode >= order) throw Error(NTFG_ERR_SHAPE, "bcomm_block_update: mode out of range");
  NTFG_DISPATCH(prec, {
    with_engine<T>(c, prec, order, dims, rank, beta, eps, [&](CpEngine<T>& e) {
      e.set_x(x, 0, NTFG_HOST);
      e.set_factors_host(factors);
      const double* a = e.A(int(mode));
      if (anchor) {
        c.h2d(e.anchors() + e.offset(int(mode)), anchor, size_t(e.dim(int(mode))) * rank * sizeof(double));
        a = e.anchors() + e.offset(int(mode));
      }
      e.block_update(int(mode), a, false);
      e.get_factors_host(factors);
    });
  });
}

void cp_bcomm_sweep(Context& c, int prec, double beta, double eps, uint32_t order,
                    const uint64_t* dims, const double* x, uint64_t rank, double* factors) {
  NTFG_DISPATCH(prec, {
    with_engine<T>(c, prec, order, dims, rank, beta, eps, [&](CpEngine<T>& e) {
      e.set_x(x, 0, NTFG_HOST);
      e.set_factors_host(factors);
      e.bcomm_sweep(false);
      e.get_factors_host(factors);
    });
  });
}

void cp_jcomm_reference(Context& c, int prec, double beta, double eps, uint32_t order,
                        const uint64_t* dims, const double* x, uint64_t rank,
                        const double* factors, double* p_out, double* q_out) {
  NTFG_DISPATCH(prec, {
    with_engine<T>(c, prec, order, dims, rank, beta, eps, [&](CpEngine<T>& e) {
      e.set_x(x, 0, NTFG_HOST);
      e.set_factors_host(factors);
      e.jcomm_reference(false);
      if (e.tc()) {  // bf16 hi/lo planes: return hi + lo (the values the contraction uses)
        const int64_t E = e.entries();
        double* tmp = c.buf<double>("step.join", size_t(E));
        const int grid = int(std::min<int64_t>(ceil_div(E, 256), 4096));
        join_planes_kernel<<<grid, 256, 0, c.stream>>>(static_cast<const __nv_bfloat16*>(e.plane(0)),
                                                       static_cast<const __nv_bfloat16*>(e.plane(1)), E, tmp);
        NTFG_LAUNCHED(c);
        c.d2h(p_out, tmp, size_t(E) * sizeof(double));
        c.sync();
        if (beta == 1.0) {
          for (int64_t i = 0; i < E; ++i) q_out[i] = 1.0;
        } else {
          join_planes_kernel<<<grid, 256, 0, c.stream>>>(static_cast<const __nv_bfloat16*>(e.plane(2)),
                                                         static_cast<const __nv_bfloat16*>(e.plane(3)), E, tmp);
          NTFG_LAUNCHED(c);
          c.d2h(q_out, tmp, size_t(E) * sizeof(double));
          c.sync();
        }
        return;
      }
      std::vector<T> h(size_t(e.entries()));
      c.d2h(h.data(), e.p(), h.size() * sizeof(T));
      c.sync();
      for (size_t i = 0; i < h.size(); ++i) p_out[i] = double(h[i]);
      if (beta == 1.0) {
        for (size_t i = 0; i < h.size(); ++i) q_out[i] = 1.0;  // weights: Q == 1 (kernels.hpp:36)
      } else {
        c.d2h(h.data(), e.q(), h.size() * sizeof(T));
        c.sync();
        for (size_t i = 0; i < h.size(); ++i) q_out[i] = double(h[i]);
      }
    });
  });
}

void cp_jcomm_inner_update(Context& c, int prec, double beta, double eps, uint32_t order,
                           const uint64_t* dims, const double* p, const double* q, uint64_t rank,
                           const double* ref, double* current, uint32_t mode) {
  if (mode >= order) throw Error(NTFG_ERR_SHAPE, "jcomm_inner_update: mode out of range");
  NTFG_DISPATCH(prec, {
    with_engine<T>(c, prec, order, dims, rank, beta, eps, [&](CpEngine<T>& e) {
      e.set_factors_host(current);
      c.h2d(e.Aref_all(), ref, e.factor_doubles() * sizeof(double));
      if (e.tc()) {
        const int64_t E = e.entries();
        double* tmp = c.buf<double>("step.join", size_t(E));
        const int grid = int(std::min<int64_t>(ceil_div(E, 256), 4096));
        for (int w = 0; w < (beta != 1.0 ? 2 : 1); ++w) {
          c.h2d(tmp, w == 0 ? p : q, size_t(E) * sizeof(double));
          split_planes_kernel<<<grid, 256, 0, c.stream>>>(tmp, E, static_cast<__nv_bfloat16*>(e.plane(2 * w)),
                                                          static_cast<__nv_bfloat16*>(e.plane(2 * w + 1)));
          NTFG_LAUNCHED(c);
        }
      } else {
        e.upload_convert(e.p(), p, 0, NTFG_HOST, e.entries());
        if (beta != 1.0) e.upload_convert(e.q(), q, 0, NTFG_HOST, e.entries());
      }
      const int64_t F = int64_t(e.factor_doubles());
      chi_all_kernel<<<int(ceil_div(F, 256)), 256, 0, c.stream>>>(
          e.A_all(), e.Aref_all(), F, beta, e.chi1_all(), e.chi2_all(), e.flags());
      NTFG_LAUNCHED(c);
      e.jcomm_inner(int(mode));
      e.get_factors_host(current);
    });
  });
}

void cp_jcomm_outer_step(Context& c, int prec, double beta, double eps, uint64_t inner,
                         uint32_t order, const uint64_t* dims, const double* x, uint64_t rank,
                         double* factors) {
  if (inner < 1) throw Error(NTFG_ERR_DOMAIN, "jcomm_outer_step: inner_steps must be >= 1");
  NTFG_DISPATCH(prec, {
    with_engine<T>(c, prec, order, dims, rank, beta, eps, [&](CpEngine<T>& e) {
      check_positive_host(factors, e.factor_doubles(), "chi1");
      e.set_x(x, 0, NTFG_HOST);
      e.set_factors_host(factors);
      e.jcomm_outer(int(inner), false);
      e.get_factors_host(factors);
    });
  });
}

void D_beta(Context& c, double beta, uint64_t n, const double* x, const double* xhat, double* out) {
  gamma_of(beta);
  if (n == 0) { *out = 0.0; return; }
  double* dx = c.buf<double>("db.x", n);
  double* dy = c.buf<double>("db.y", n);
  const int grid = int(std::min<uint64_t>(ceil_div(int64_t(n), 256), 1024));
  double* part = c.buf<double>("db.part", size_t(grid));
  unsigned* flags = c.buf<unsigned>("db.flags", 1);
  double* losses = c.buf<double>("db.loss", 1);
  int* counter = c.buf<int>("db.counter", 1);
  c.h2d(dx, x, n * sizeof(double));
  c.h2d(dy, xhat, n * sizeof(double));
  NTFG_CUDA(cudaMemsetAsync(flags, 0, sizeof(unsigned), c.stream));
  NTFG_CUDA(cudaMemsetAsync(counter, 0, sizeof(int), c.stream));
  dbeta_sum_kernel<<<grid, 256, 0, c.stream>>>(dx, dy, int64_t(n), beta_kind_of(beta), beta, part, flags);
  NTFG_LAUNCHED(c);
  objective_finalize_kernel<<<1, 256, 0, c.stream>>>(part, grid, 1.0, losses, counter, nullptr);
  NTFG_LAUNCHED(c);
  c.sync();
  unsigned f = 0;
  NTFG_CUDA(cudaMemcpy(&f, flags, sizeof(unsigned), cudaMemcpyDeviceToHost));
  raise_flags(f);
  NTFG_CUDA(cudaMemcpy(out, losses, sizeof(double), cudaMemcpyDeviceToHost));
}

}  // namespace ntfg
