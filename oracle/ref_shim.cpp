// Test infrastructure only (never linked into the product).
//
// C-ABI shim over the UNMODIFIED reference library, which oracle/Makefile
// compiles straight from /root/reference/proj/src into oracle/_ref/.  The
// shim lets Python (ctypes) drive the reference's own public API
// (ntf::bcomm_fit / jcomm_fit / tucker_*_fit and the step-level functions,
// reference include/ntf/{cp,tucker,tensor,divergence,io}.hpp) on plain host
// buffers, so the parity tests and the CPU baseline can run the real thing.
//
// Layout conventions: tensors are row-major fp64 with u64 dims; CP factors
// are concatenated row-major I_n x R blocks; Tucker factors are concatenated
// row-major I_n x J_n blocks.  Every entry point returns 0 on success or a
// status code mirroring the product's ntfg_status (1 shape, 2 domain,
// 3 numerical, 4 format, 8 other) with the message in ntfref_last_error().
#include <chrono>
#include <cstdint>
#include <cstring>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "ntf/config.hpp"
#include "ntf/cp.hpp"
#include "ntf/divergence.hpp"
#include "ntf/errors.hpp"
#include "ntf/io.hpp"
#include "ntf/oracle.hpp"
#include "ntf/tensor.hpp"
#include "ntf/tucker.hpp"
#include "ntf/unfold.hpp"

#define SHIM extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ntf::ShapeError& e) {
        g_err = e.what();
        return 1;
    } catch (const ntf::DomainError& e) {
        g_err = e.what();
        return 2;
    } catch (const ntf::NumericalError& e) {
        g_err = e.what();
        return 3;
    } catch (const ntf::FormatError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 8;
    }
}

std::vector<std::size_t> to_shape(int order, const std::uint64_t* dims) {
    return std::vector<std::size_t>(dims, dims + order);
}

std::size_t prod(const std::vector<std::size_t>& s) {
    std::size_t n = 1;
    for (auto d : s) n *= d;
    return n;
}

ntf::DenseTensor tensor_in(const std::vector<std::size_t>& shape, const double* v) {
    return ntf::DenseTensor(shape, std::vector<double>(v, v + prod(shape)));
}

void tensor_out(const ntf::DenseTensor& t, double* out) {
    std::memcpy(out, t.data(), t.size() * sizeof(double));
}

ntf::CpFactors cp_in(const std::vector<std::size_t>& dims, std::size_t rank, const double* f) {
    std::vector<ntf::Matrix> ms;
    for (auto d : dims) {
        ms.emplace_back(d, rank, std::vector<double>(f, f + d * rank));
        f += d * rank;
    }
    return ntf::CpFactors(std::move(ms));
}

void cp_out(const ntf::CpFactors& c, double* f) {
    for (const auto& m : c.factors) {
        std::memcpy(f, m.values().data(), m.size() * sizeof(double));
        f += m.size();
    }
}

std::vector<ntf::Matrix> mats_in(const std::vector<std::size_t>& rows,
                                 const std::vector<std::size_t>& cols, const double* f) {
    std::vector<ntf::Matrix> ms;
    for (std::size_t n = 0; n < rows.size(); ++n) {
        ms.emplace_back(rows[n], cols[n], std::vector<double>(f, f + rows[n] * cols[n]));
        f += rows[n] * cols[n];
    }
    return ms;
}

ntf::TuckerModel tucker_in(const std::vector<std::size_t>& dims,
                           const std::vector<std::size_t>& ranks, const double* core,
                           const double* f) {
    return ntf::TuckerModel(tensor_in(ranks, core), mats_in(dims, ranks, f));
}

void tucker_out(const ntf::TuckerModel& m, double* core, double* f) {
    if (core) tensor_out(m.core, core);
    if (f) {
        for (const auto& a : m.factors) {
            std::memcpy(f, a.values().data(), a.size() * sizeof(double));
            f += a.size();
        }
    }
}

ntf::FitConfig make_cfg(double beta, double eps, int inner, int max_iters, double tol, int extrap,
                        double cap, double delta) {
    ntf::FitConfig cfg;
    cfg.beta = beta;
    cfg.eps = eps;
    cfg.inner_steps = static_cast<std::size_t>(inner);
    cfg.max_iters = static_cast<std::size_t>(max_iters);
    cfg.tol = tol;
    cfg.extrapolate = extrap != 0;
    cfg.extrap_cap = cap;
    cfg.extrap_delta = delta;
    return cfg;
}

void trace_out(const std::vector<ntf::TraceRecord>& tr, double* t, double* l, int* len) {
    for (std::size_t k = 0; k < tr.size(); ++k) {
        if (t) t[k] = tr[k].time_s;
        if (l) l[k] = tr[k].loss;
    }
    *len = static_cast<int>(tr.size());
}

}  // namespace

SHIM const char* ntfref_last_error() { return g_err.c_str(); }

// ---- fits --------------------------------------------------------------------

SHIM int ntfref_cp_fit(int algo, int order, const std::uint64_t* dims, const double* x, int rank,
                       double* factors, double beta, double eps, int inner, int max_iters,
                       double tol, int extrap, double cap, double delta, double* trace_time,
                       double* trace_loss, int* trace_len) {
    return guarded([&] {
        const auto shape = to_shape(order, dims);
        const ntf::DenseTensor xt = tensor_in(shape, x);
        ntf::CpFactors init = cp_in(shape, rank, factors);
        ntf::FitConfig cfg = make_cfg(beta, eps, inner, max_iters, tol, extrap, cap, delta);
        cfg.rank = static_cast<std::size_t>(rank);
        const ntf::CpFitResult r = algo == 0 ? ntf::bcomm_fit(xt, std::move(init), cfg)
                                             : ntf::jcomm_fit(xt, std::move(init), cfg);
        cp_out(r.model, factors);
        trace_out(r.trace, trace_time, trace_loss, trace_len);
    });
}

SHIM int ntfref_tucker_fit(int algo, int order, const std::uint64_t* dims, const double* x,
                           const std::uint64_t* ranks, double* core, double* factors, double beta,
                           double eps, int inner, int max_iters, double tol, int extrap,
                           double cap, double delta, double* trace_time, double* trace_loss,
                           int* trace_len) {
    return guarded([&] {
        const auto shape = to_shape(order, dims);
        const auto rk = to_shape(order, ranks);
        const ntf::DenseTensor xt = tensor_in(shape, x);
        ntf::TuckerModel init = tucker_in(shape, rk, core, factors);
        ntf::FitConfig cfg = make_cfg(beta, eps, inner, max_iters, tol, extrap, cap, delta);
        cfg.model = ntf::ModelKind::tucker;
        cfg.ranks = rk;
        const ntf::TuckerFitResult r = algo == 0 ? ntf::tucker_bcomm_fit(xt, std::move(init), cfg)
                                                 : ntf::tucker_jcomm_fit(xt, std::move(init), cfg);
        tucker_out(r.model, core, factors);
        trace_out(r.trace, trace_time, trace_loss, trace_len);
    });
}

// Times `steps` outer iterations of the reference solver on one problem
// (the timed region is exactly the reference's own step, as in
// fit_common.hpp:40-44); used by the CPU baseline.
SHIM int ntfref_cp_time_outer(int algo, int order, const std::uint64_t* dims, const double* x,
                              int rank, double* factors, double beta, double eps, int inner,
                              int steps, double* seconds) {
    return guarded([&] {
        const auto shape = to_shape(order, dims);
        const ntf::DenseTensor xt = tensor_in(shape, x);
        ntf::CpFactors f = cp_in(shape, rank, factors);
        const ntf::BetaParam p(beta);
        const auto t0 = std::chrono::steady_clock::now();
        for (int s = 0; s < steps; ++s)
            f = algo == 0 ? ntf::bcomm_sweep(f, xt, p, eps)
                          : ntf::jcomm_outer_step(f, xt, p, static_cast<std::size_t>(inner), eps);
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        cp_out(f, factors);
    });
}

// ---- CP step level --------------------------------------------------------------

SHIM int ntfref_cp_block_update(int order, const std::uint64_t* dims, const double* x, int rank,
                                double* factors, int mode, const double* anchor, double beta,
                                double eps) {
    return guarded([&] {
        const auto shape = to_shape(order, dims);
        const ntf::DenseTensor xt = tensor_in(shape, x);
        ntf::CpFactors f = cp_in(shape, rank, factors);
        const ntf::BetaParam p(beta);
        if (anchor) {
            const ntf::Matrix a(shape[mode], rank,
                                std::vector<double>(anchor, anchor + shape[mode] * rank));
            f = ntf::cp_block_update_anchored(f, mode, a, xt, p, eps);
        } else {
            f = ntf::bcomm_block_update(f, mode, xt, p, eps);
        }
        cp_out(f, factors);
    });
}

SHIM int ntfref_cp_bcomm_sweep(int order, const std::uint64_t* dims, const double* x, int rank,
                               double* factors, double beta, double eps) {
    return guarded([&] {
        const auto shape = to_shape(order, dims);
        ntf::CpFactors f = cp_in(shape, rank, factors);
        f = ntf::bcomm_sweep(f, tensor_in(shape, x), ntf::BetaParam(beta), eps);
        cp_out(f, factors);
    });
}

SHIM int ntfref_cp_jcomm_reference(int order, const std::uint64_t* dims, const double* x,
                                   int rank, const double* factors, double beta, double eps,
                                   double* p_out, double* q_out) {
    return guarded([&] {
        const auto shape = to_shape(order, dims);
        const auto ctx = ntf::make_jcomm_reference(cp_in(shape, rank, factors), tensor_in(shape, x),
                                                   ntf::BetaParam(beta), eps);
        tensor_out(ctx.p, p_out);
        tensor_out(ctx.q, q_out);
    });
}

SHIM int ntfref_cp_jcomm_inner_update(int order, const std::uint64_t* dims, const double* x,
                                      int rank, const double* ref, double* current, int mode,
                                      double beta, double eps) {
    return guarded([&] {
        const auto shape = to_shape(order, dims);
        const ntf::BetaParam p(beta);
        const auto ctx = ntf::make_jcomm_reference(cp_in(shape, rank, ref), tensor_in(shape, x), p, eps);
        ntf::CpFactors cur = cp_in(shape, rank, current);
        cur = ntf::jcomm_inner_update(cur, ctx, mode, p, eps);
        cp_out(cur, current);
    });
}

SHIM int ntfref_cp_jcomm_outer_step(int order, const std::uint64_t* dims, const double* x, int rank,
                                    double* factors, double beta, int inner, double eps) {
    return guarded([&] {
        const auto shape = to_shape(order, dims);
        ntf::CpFactors f = cp_in(shape, rank, factors);
        f = ntf::jcomm_outer_step(f, tensor_in(shape, x), ntf::BetaParam(beta),
                                  static_cast<std::size_t>(inner), eps);
        cp_out(f, factors);
    });
}

SHIM int ntfref_cp_reconstruct(int order, const std::uint64_t* dims, int rank,
                               const double* factors, double* out) {
    return guarded([&] { tensor_out(ntf::cp_reconstruct(cp_in(to_shape(order, dims), rank, factors)), out); });
}

SHIM int ntfref_cp_contract(int order, const std::uint64_t* dims, const double* t, int rank,
                            const double* factors, int mode, double* out) {
    return guarded([&] {
        const auto shape = to_shape(order, dims);
        const auto fs = mats_in(shape, std::vector<std::size_t>(order, rank), factors);
        const ntf::Matrix m = ntf::cp_contract(tensor_in(shape, t), fs, mode);
        std::memcpy(out, m.values().data(), m.size() * sizeof(double));
    });
}

// ---- divergence ------------------------------------------------------------------

SHIM int ntfref_D_beta(std::uint64_t n, const double* x, const double* xhat, double beta,
                       double* out) {
    return guarded([&] {
        const std::vector<std::size_t> s{static_cast<std::size_t>(n)};
        *out = ntf::D_beta(tensor_in(s, x), tensor_in(s, xhat), ntf::BetaParam(beta));
    });
}

SHIM int ntfref_d_beta(double x, double y, double beta, double* out) {
    return guarded([&] { *out = ntf::d_beta(x, y, ntf::BetaParam(beta)); });
}

SHIM int ntfref_gamma(double beta, double* out) {
    return guarded([&] { *out = ntf::BetaParam(beta).gamma(); });
}

SHIM int ntfref_weights(std::uint64_t n, const double* x, const double* xhat, double beta,
                        double eps, double* p, double* q) {
    return guarded([&] {
        const std::vector<std::size_t> s{static_cast<std::size_t>(n)};
        const auto [pt, qt] = ntf::weights(tensor_in(s, x), tensor_in(s, xhat), ntf::BetaParam(beta), eps);
        tensor_out(pt, p);
        tensor_out(qt, q);
    });
}

SHIM int ntfref_chi(int which, std::uint64_t n, const double* z, const double* zref, double beta,
                    double* out) {
    return guarded([&] {
        const std::vector<std::size_t> s{static_cast<std::size_t>(n)};
        const ntf::BetaParam p(beta);
        const auto r = which == 1 ? ntf::chi1(tensor_in(s, z), tensor_in(s, zref), p)
                                  : ntf::chi2(tensor_in(s, z), tensor_in(s, zref), p);
        tensor_out(r, out);
    });
}

SHIM int ntfref_multiplicative_update(std::uint64_t n, const double* anchor, const double* num,
                                      const double* den, double gamma, double eps, double* out) {
    return guarded([&] {
        const std::vector<std::size_t> s{static_cast<std::size_t>(n)};
        tensor_out(ntf::multiplicative_update(tensor_in(s, anchor), tensor_in(s, num),
                                              tensor_in(s, den), gamma, eps),
                   out);
    });
}

// ---- Tucker contractions and step level ------------------------------------------

SHIM int ntfref_tucker_reconstruct(int order, const std::uint64_t* dims, const std::uint64_t* ranks,
                                   const double* core, const double* factors, double* out) {
    return guarded([&] {
        const auto shape = to_shape(order, dims);
        const auto rk = to_shape(order, ranks);
        tensor_out(ntf::tucker_reconstruct(tucker_in(shape, rk, core, factors)), out);
    });
}

SHIM int ntfref_tucker_multimode_contract(int order, const std::uint64_t* dims, const double* t,
                                          const std::uint64_t* cols, const double* factors,
                                          int skip, double* out) {
    return guarded([&] {
        const auto shape = to_shape(order, dims);
        const auto fs = mats_in(shape, to_shape(order, cols), factors);
        std::optional<std::size_t> sk;
        if (skip >= 0) sk = static_cast<std::size_t>(skip);
        tensor_out(ntf::tucker_multimode_contract(tensor_in(shape, t), fs, sk), out);
    });
}

SHIM int ntfref_tucker_factor_contract(int order, const std::uint64_t* dims, const double* t,
                                       const std::uint64_t* ranks, const double* core,
                                       const double* factors, int mode, std::uint64_t budget,
                                       double* out) {
    return guarded([&] {
        const auto shape = to_shape(order, dims);
        const auto rk = to_shape(order, ranks);
        const auto fs = mats_in(shape, rk, factors);
        const ntf::Matrix m = ntf::tucker_factor_contract(tensor_in(shape, t), tensor_in(rk, core),
                                                          fs, mode, budget);
        std::memcpy(out, m.values().data(), m.size() * sizeof(double));
    });
}

// kind: 0 core block update, 1 factor block update (mode), 2 bcomm sweep,
// 3 jcomm outer step (inner), 4 jcomm inner core update from reference `ref`,
// 5 jcomm inner factor update (mode) from reference `ref`.
SHIM int ntfref_tucker_step(int kind, int order, const std::uint64_t* dims, const double* x,
                            const std::uint64_t* ranks, const double* ref_core,
                            const double* ref_factors, double* core, double* factors, int mode,
                            double beta, int inner, double eps) {
    return guarded([&] {
        const auto shape = to_shape(order, dims);
        const auto rk = to_shape(order, ranks);
        const ntf::DenseTensor xt = tensor_in(shape, x);
        const ntf::BetaParam p(beta);
        ntf::TuckerModel m = tucker_in(shape, rk, core, factors);
        switch (kind) {
            case 0: m = ntf::block_core_update(m, xt, p, eps); break;
            case 1: m = ntf::block_factor_update(m, mode, xt, p, eps); break;
            case 2: m = ntf::tucker_bcomm_sweep(m, xt, p, eps); break;
            case 3: m = ntf::jcomm_tucker_outer_step(m, xt, p, static_cast<std::size_t>(inner), eps); break;
            case 4:
            case 5: {
                const auto ctx = ntf::make_jcomm_tucker_reference(
                    tucker_in(shape, rk, ref_core, ref_factors), xt, p, eps);
                m = kind == 4 ? ntf::jcomm_inner_core_update(m, ctx, p, eps)
                              : ntf::jcomm_inner_factor_update(m, ctx, mode, p, eps);
                break;
            }
            default: throw ntf::DomainError("unknown tucker step kind");
        }
        tucker_out(m, core, factors);
    });
}

// ---- generators ---------------------------------------------------------------------

SHIM int ntfref_rng_uniform(std::uint64_t seed, std::uint64_t stream, std::uint64_t n, double* out) {
    return guarded([&] {
        ntf::Rng rng(seed, stream);
        for (std::uint64_t i = 0; i < n; ++i) out[i] = rng.uniform01();
    });
}

SHIM int ntfref_init_cp_factors(int order, const std::uint64_t* dims, int rank, std::uint64_t seed,
                                double eps, double* out) {
    return guarded([&] {
        const auto shape = to_shape(order, dims);
        cp_out(ntf::init_cp_factors(shape, rank, seed, eps), out);
    });
}

SHIM int ntfref_init_tucker_model(int order, const std::uint64_t* dims, const std::uint64_t* ranks,
                                  std::uint64_t seed, double eps, double* core, double* factors) {
    return guarded([&] {
        tucker_out(ntf::init_tucker_model(to_shape(order, dims), to_shape(order, ranks), seed, eps),
                   core, factors);
    });
}

SHIM int ntfref_synth_cp(int order, const std::uint64_t* dims, int rank, std::uint64_t seed,
                         double eps, double* x, double* truth) {
    return guarded([&] {
        const auto [xt, f] = ntf::synth_cp(to_shape(order, dims), rank, seed, eps);
        tensor_out(xt, x);
        cp_out(f, truth);
    });
}

SHIM int ntfref_synth_tucker(int order, const std::uint64_t* dims, const std::uint64_t* ranks,
                             std::uint64_t seed, double eps, double* x, double* core,
                             double* factors) {
    return guarded([&] {
        const auto [xt, m] = ntf::synth_tucker(to_shape(order, dims), to_shape(order, ranks), seed, eps);
        tensor_out(xt, x);
        tucker_out(m, core, factors);
    });
}

// MU-unfold baseline sweep (reference unfold.cpp:109-185), an independent
// equivalence oracle for the contraction path (acceptance criterion 2).
SHIM int ntfref_mu_unfold_cp_sweep(int order, const std::uint64_t* dims, const double* x, int rank,
                                   double* factors, double beta, double eps) {
    return guarded([&] {
        const auto shape = to_shape(order, dims);
        ntf::CpFactors f = cp_in(shape, rank, factors);
        f = ntf::mu_unfold_cp_sweep(f, tensor_in(shape, x), ntf::BetaParam(beta), eps);
        cp_out(f, factors);
    });
}

// I/O (reference io.cpp): CTF1 write/read, COO text densify, trace CSV --
// fixtures for the byte-exact interchange tests (tests/test_io_cpu.py).
SHIM int ntfref_write_tensor(const char* path, int order, const std::uint64_t* dims, const double* x) {
    return guarded([&] { ntf::write_tensor(path, tensor_in(to_shape(order, dims), x)); });
}

SHIM int ntfref_read_coo_dense(const char* path, int has_floor, double floor, std::uint64_t cap, double* out,
                               int* order, std::uint64_t* dims) {
    return guarded([&] {
        const ntf::DenseTensor t =
            ntf::read_coo(path, has_floor ? std::optional<double>(floor) : std::nullopt);
        *order = int(t.order());
        for (std::size_t n = 0; n < t.order(); ++n) dims[n] = t.shape()[n];
        if (t.size() > cap) throw std::runtime_error("capacity");
        for (std::size_t i = 0; i < t.size(); ++i) out[i] = t[i];
    });
}

SHIM int ntfref_write_trace(const char* path, int n, const double* times, const double* losses) {
    return guarded([&] {
        std::vector<ntf::TraceRecord> r(static_cast<std::size_t>(n));
        for (int i = 0; i < n; ++i) r[std::size_t(i)] = ntf::TraceRecord{std::size_t(i), times[i], losses[i]};
        ntf::write_trace(path, r);
    });
}

// ---- joint-surrogate oracle (reference oracle.hpp:41-80, oracle.cpp:181-281) -------

SHIM int ntfref_joint_surrogate_cp(int order, const std::uint64_t* dims, const double* x, int rank,
                                   const double* theta, const double* ref, double beta, double eps,
                                   double* out) {
    return guarded([&] {
        const auto shape = to_shape(order, dims);
        *out = ntf::oracle::eval_joint_surrogate_cp(cp_in(shape, rank, theta), cp_in(shape, rank, ref),
                                                    tensor_in(shape, x), ntf::BetaParam(beta), eps);
    });
}

SHIM int ntfref_joint_surrogate_tucker(int order, const std::uint64_t* dims, const double* x,
                                       const std::uint64_t* ranks, const double* theta_core,
                                       const double* theta, const double* ref_core, const double* ref,
                                       double beta, double eps, double* out) {
    return guarded([&] {
        const auto shape = to_shape(order, dims);
        const auto rk = to_shape(order, ranks);
        *out = ntf::oracle::eval_joint_surrogate_tucker(tucker_in(shape, rk, theta_core, theta),
                                                        tucker_in(shape, rk, ref_core, ref),
                                                        tensor_in(shape, x), ntf::BetaParam(beta), eps);
    });
}

SHIM int ntfref_scalar_minimizer(double num, double den, double beta, double floor, double* u, double* g) {
    return guarded([&] {
        const ntf::BetaParam p(beta);
        *u = ntf::oracle::scalar_minimizer(num, den, p, floor);
        *g = ntf::oracle::jmm_scalar_objective(*u, num, den, p);
    });
}
