// Drop-in C++ API (namespace ntf, include/ntf/ntf.hpp) over the C ABI of
// libntfg.so.  Value types and argument checks mirror the reference
// (/root/reference/proj/src/{tensor,cp,tucker,divergence,config}.cpp);
// every E-sized computation runs on the GPU through ntfg_*.
#include "ntf/ntf.hpp"
#include "ntf/io.hpp"
#include "ntf/unfold.hpp"

#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>

#include "ntfg.h"

namespace ntf {

namespace {

[[noreturn]] void rethrow(ntfg_status s) {
    const std::string msg = ntfg_last_error();
    switch (s) {
        case NTFG_ERR_SHAPE: throw ShapeError(msg);
        case NTFG_ERR_DOMAIN: throw DomainError(msg);
        case NTFG_ERR_NUMERICAL: throw NumericalError(msg);
        case NTFG_ERR_FORMAT: throw FormatError(msg);
        default: throw DeviceError(msg);
    }
}

void ok(ntfg_status s) {
    if (s != NTFG_OK) rethrow(s);
}

// one context per (thread, device): contexts are not shared across threads
// (reference threading contract).
struct Ctx {
    ntfg_context* h = nullptr;
    int device = -1;
    ~Ctx() {
        if (h) ntfg_context_destroy(h);
    }
};

ntfg_context* ctx(int device = 0) {
    thread_local Ctx c;
    if (!c.h || c.device != device) {
        if (c.h) ntfg_context_destroy(c.h);
        c.h = nullptr;
        ok(ntfg_context_create(device, &c.h));
        c.device = device;
    }
    return c.h;
}

std::size_t product(const std::vector<std::size_t>& s) {
    std::size_t n = 1;
    for (auto d : s) n *= d;
    return n;
}

std::vector<std::uint64_t> u64(const std::vector<std::size_t>& v) {
    return std::vector<std::uint64_t>(v.begin(), v.end());
}

std::vector<double> concat(const std::vector<Matrix>& ms) {
    std::vector<double> out;
    for (const auto& m : ms) out.insert(out.end(), m.values().begin(), m.values().end());
    return out;
}

void split_into(const std::vector<double>& flat, std::vector<Matrix>& ms) {
    std::size_t off = 0;
    for (auto& m : ms) {
        std::memcpy(m.values().data(), flat.data() + off, m.size() * sizeof(double));
        off += m.size();
    }
}

void require_dims(const std::vector<Matrix>& f, const DenseTensor& x, const char* op) {
    if (f.size() != x.order()) throw ShapeError(std::string(op) + ": order mismatch");
    for (std::size_t n = 0; n < f.size(); ++n)
        if (f[n].rows() != x.dim(n))
            throw ShapeError(std::string(op) + ": factor rows do not match data dimension");
}

ntfg_fit_config to_c(const FitConfig& cfg, std::vector<std::uint64_t>& ranks_keep) {
    ntfg_fit_config c{};
    c.beta = cfg.beta;
    c.rank = cfg.rank;
    ranks_keep = u64(cfg.ranks);
    c.ranks = ranks_keep.empty() ? nullptr : ranks_keep.data();
    c.n_ranks = std::uint32_t(ranks_keep.size());
    c.eps = cfg.eps;
    c.inner_steps = cfg.inner_steps;
    c.max_iters = cfg.max_iters;
    c.tol = cfg.tol;
    c.seed = cfg.seed;
    c.extrapolate = cfg.extrapolate;
    c.extrap_cap = cfg.extrap_cap;
    c.extrap_delta = cfg.extrap_delta;
    c.has_data_floor = cfg.data_floor.has_value();
    c.data_floor = cfg.data_floor.value_or(0.0);
    c.precision = cfg.precision == Precision::f32 ? NTFG_F32 : NTFG_F64;
    c.use_graphs = cfg.use_graphs;
    return c;
}

std::vector<TraceRecord> trace_of(const std::vector<ntfg_trace_row>& rows, std::uint64_t n) {
    std::vector<TraceRecord> out(n);
    for (std::uint64_t i = 0; i < n; ++i) out[i] = {std::size_t(rows[i].iter), rows[i].time_s, rows[i].loss};
    return out;
}

}  // namespace

// ---- value types (reference tensor.cpp:35-116) ----------------------------------------

static void validate_shape(const std::vector<std::size_t>& s) {
    if (s.empty()) throw ShapeError("tensor order must be >= 1");
    for (auto d : s)
        if (d == 0) throw ShapeError("tensor dimensions must be >= 1");
}

DenseTensor::DenseTensor(std::vector<std::size_t> shape) : shape_(std::move(shape)) {
    validate_shape(shape_);
    values_.assign(product(shape_), 0.0);
}

DenseTensor::DenseTensor(std::vector<std::size_t> shape, std::vector<double> values)
    : shape_(std::move(shape)), values_(std::move(values)) {
    validate_shape(shape_);
    if (values_.size() != product(shape_)) throw ShapeError("tensor value count does not match shape product");
}

DenseTensor DenseTensor::full(std::vector<std::size_t> shape, double value) {
    DenseTensor t(std::move(shape));
    for (auto& v : t.values_) v = value;
    return t;
}

std::size_t DenseTensor::flat_index(std::span<const std::size_t> index) const {
    if (index.size() != shape_.size()) throw ShapeError("multi-index length does not match order");
    std::size_t flat = 0;
    for (std::size_t a = 0; a < shape_.size(); ++a) {
        if (index[a] >= shape_[a]) throw ShapeError("multi-index coordinate out of range");
        flat = flat * shape_[a] + index[a];
    }
    return flat;
}

Matrix::Matrix(std::size_t rows, std::size_t cols) : rows_(rows), cols_(cols), values_(rows * cols, 0.0) {}

Matrix::Matrix(std::size_t rows, std::size_t cols, std::vector<double> values)
    : rows_(rows), cols_(cols), values_(std::move(values)) {
    if (values_.size() != rows_ * cols_) throw ShapeError("matrix value count does not match rows * cols");
}

Matrix Matrix::full(std::size_t rows, std::size_t cols, double value) {
    Matrix m(rows, cols);
    for (auto& v : m.values_) v = value;
    return m;
}

Matrix Matrix::identity(std::size_t n) {
    Matrix m(n, n);
    for (std::size_t i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
}

bool next_multi_index(MultiIndex& index, std::span<const std::size_t> shape) {
    for (std::size_t a = shape.size(); a-- > 0;) {
        if (++index[a] < shape[a]) return true;
        index[a] = 0;
    }
    return false;
}

// ---- config / divergence ------------------------------------------------------------------

void validate_fit_config(const FitConfig& cfg) {
    std::vector<std::uint64_t> keep;
    const ntfg_fit_config c = to_c(cfg, keep);
    ok(ntfg_validate_fit_config(&c));
}

BetaParam::BetaParam(double beta) : beta_(beta) {
    if (!(beta >= 0.0 && beta < 2.0)) throw DomainError("beta must lie in [0, 2)");
    gamma_ = beta < 1.0 ? 1.0 / (2.0 - beta) : 1.0;
}

double d_beta(double x, double y, const BetaParam& p) {
    double out = 0.0;
    ok(ntfg_D_beta(ctx(), p.beta(), 1, &x, &y, &out));
    return out;
}

double D_beta(const DenseTensor& x, const DenseTensor& xhat, const BetaParam& p) {
    if (x.shape() != xhat.shape()) throw ShapeError("D_beta: shape mismatch");
    double out = 0.0;
    ok(ntfg_D_beta(ctx(), p.beta(), x.size(), x.data(), xhat.data(), &out));
    return out;
}

double D_beta_mean(const DenseTensor& x, const DenseTensor& xhat, const BetaParam& p) {
    return D_beta(x, xhat, p) / double(x.size());
}

// ---- CP -------------------------------------------------------------------------------------

CpFactors::CpFactors(std::vector<Matrix> f) : factors(std::move(f)) {
    if (factors.empty()) throw ShapeError("CpFactors: at least one factor required");
    const std::size_t r = factors.front().cols();
    for (const Matrix& m : factors) {
        if (m.cols() != r) throw ShapeError("CpFactors: factors must share a column count");
        if (m.rows() == 0 || r == 0) throw ShapeError("CpFactors: empty factor");
    }
}

std::vector<std::size_t> CpFactors::dims() const {
    std::vector<std::size_t> d;
    for (const auto& m : factors) d.push_back(m.rows());
    return d;
}

DenseTensor cp_reconstruct(const CpFactors& f) {
    DenseTensor out(f.dims());
    const auto dims = u64(f.dims());
    const auto flat = concat(f.factors);
    ok(ntfg_cp_reconstruct(ctx(), NTFG_F64, std::uint32_t(dims.size()), dims.data(), f.rank(), flat.data(),
                           out.data()));
    return out;
}

Matrix cp_contract(const DenseTensor& t, std::span<const Matrix> factors, std::size_t mode) {
    if (factors.size() != t.order()) throw ShapeError("cp_contract: expected one factor per mode");
    if (mode >= t.order()) throw ShapeError("cp_contract: mode out of range");
    const std::size_t r = factors[mode].cols();
    std::vector<Matrix> fs;
    for (std::size_t m = 0; m < t.order(); ++m) {
        if (m == mode) {
            fs.push_back(Matrix::full(t.dim(m), r, 1.0));
            continue;
        }
        if (factors[m].rows() != t.dim(m)) throw ShapeError("cp_contract: factor rows do not match tensor dimension");
        if (factors[m].cols() != r) throw ShapeError("cp_contract: inconsistent column counts");
        fs.push_back(factors[m]);
    }
    Matrix out(t.dim(mode), r);
    const auto dims = u64(t.shape());
    const auto flat = concat(fs);
    ok(ntfg_cp_contract(ctx(), NTFG_F64, std::uint32_t(dims.size()), dims.data(), t.data(), r, flat.data(),
                        std::uint32_t(mode), out.values().data()));
    return out;
}

CpFactors cp_block_update_anchored(const CpFactors& f, std::size_t mode, const Matrix& anchor,
                                   const DenseTensor& x, const BetaParam& p, double eps) {
    require_dims(f.factors, x, "cp_block_update");
    if (mode >= f.order()) throw ShapeError("cp_block_update: mode out of range");
    if (anchor.rows() != x.dim(mode) || anchor.cols() != f.rank())
        throw ShapeError("cp_block_update: anchor shape mismatch");
    CpFactors g = f;
    auto flat = concat(g.factors);
    const auto dims = u64(x.shape());
    ok(ntfg_cp_block_update(ctx(), NTFG_F64, p.beta(), eps, std::uint32_t(dims.size()), dims.data(), x.data(),
                            f.rank(), flat.data(), std::uint32_t(mode), anchor.values().data()));
    split_into(flat, g.factors);
    return g;
}

CpFactors bcomm_block_update(const CpFactors& f, std::size_t mode, const DenseTensor& x, const BetaParam& p,
                             double eps) {
    if (mode >= f.order()) throw ShapeError("bcomm_block_update: mode out of range");
    return cp_block_update_anchored(f, mode, f.factors[mode], x, p, eps);
}

CpFactors bcomm_sweep(const CpFactors& f, const DenseTensor& x, const BetaParam& p, double eps) {
    require_dims(f.factors, x, "bcomm_sweep");
    CpFactors g = f;
    auto flat = concat(g.factors);
    const auto dims = u64(x.shape());
    ok(ntfg_cp_bcomm_sweep(ctx(), NTFG_F64, p.beta(), eps, std::uint32_t(dims.size()), dims.data(), x.data(),
                           f.rank(), flat.data()));
    split_into(flat, g.factors);
    return g;
}

static CpFitResult cp_fit(int algo, const DenseTensor& x, CpFactors init, const FitConfig& cfg) {
    validate_fit_config(cfg);
    require_dims(init.factors, x, algo == NTFG_BCOMM ? "bcomm_fit" : "jcomm_fit");
    std::vector<std::uint64_t> keep;
    ntfg_fit_config c = to_c(cfg, keep);
    c.rank = init.rank();
    auto flat = concat(init.factors);
    std::vector<ntfg_trace_row> rows(cfg.max_iters + 1);
    std::uint64_t n = 0;
    const auto dims = u64(x.shape());
    ok(ntfg_cp_fit(ctx(cfg.device), &c, algo, std::uint32_t(dims.size()), dims.data(), x.data(), 0, NTFG_HOST,
                   nullptr, flat.data(), rows.data(), &n));
    CpFitResult out{std::move(init), trace_of(rows, n)};
    split_into(flat, out.model.factors);
    return out;
}

CpFitResult bcomm_fit(const DenseTensor& x, CpFactors init, const FitConfig& cfg) {
    return cp_fit(NTFG_BCOMM, x, std::move(init), cfg);
}

CpFitResult jcomm_fit(const DenseTensor& x, CpFactors init, const FitConfig& cfg) {
    return cp_fit(NTFG_JCOMM, x, std::move(init), cfg);
}

JcommCpReference make_jcomm_reference(const CpFactors& ref, const DenseTensor& x, const BetaParam& p,
                                      double eps) {
    require_dims(ref.factors, x, "make_jcomm_reference");
    JcommCpReference out{ref, DenseTensor(x.shape()), DenseTensor(x.shape())};
    const auto flat = concat(ref.factors);
    const auto dims = u64(x.shape());
    ok(ntfg_cp_jcomm_reference(ctx(), NTFG_F64, p.beta(), eps, std::uint32_t(dims.size()), dims.data(), x.data(),
                               ref.rank(), flat.data(), out.p.data(), out.q.data()));
    return out;
}

CpFactors jcomm_inner_update(const CpFactors& current, const JcommCpReference& c, std::size_t mode,
                             const BetaParam& p, double eps) {
    if (mode >= current.order()) throw ShapeError("jcomm_inner_update: mode out of range");
    require_dims(current.factors, c.p, "jcomm_inner_update");
    CpFactors out = current;
    auto flat = concat(out.factors);
    const auto ref = concat(c.ref.factors);
    const auto dims = u64(c.p.shape());
    ok(ntfg_cp_jcomm_inner_update(ctx(), NTFG_F64, p.beta(), eps, std::uint32_t(dims.size()), dims.data(),
                                  c.p.data(), c.q.data(), current.rank(), ref.data(), flat.data(),
                                  std::uint32_t(mode)));
    split_into(flat, out.factors);
    return out;
}

CpFactors jcomm_outer_step(const CpFactors& f, const DenseTensor& x, const BetaParam& p, std::size_t inner_steps,
                           double eps) {
    if (inner_steps < 1) throw DomainError("jcomm_outer_step: inner_steps must be >= 1");
    require_dims(f.factors, x, "jcomm_outer_step");
    CpFactors g = f;
    auto flat = concat(g.factors);
    const auto dims = u64(x.shape());
    ok(ntfg_cp_jcomm_outer_step(ctx(), NTFG_F64, p.beta(), eps, inner_steps, std::uint32_t(dims.size()),
                                dims.data(), x.data(), f.rank(), flat.data()));
    split_into(flat, g.factors);
    return g;
}

// ---- Tucker ------------------------------------------------------------------------------------

TuckerModel::TuckerModel(DenseTensor c, std::vector<Matrix> f) : core(std::move(c)), factors(std::move(f)) {
    if (factors.empty()) throw ShapeError("TuckerModel: at least one factor required");
    if (core.order() != factors.size()) throw ShapeError("TuckerModel: core order does not match factor count");
    for (std::size_t n = 0; n < factors.size(); ++n)
        if (factors[n].cols() != core.dim(n))
            throw ShapeError("TuckerModel: factor columns do not match core dimension");
}

std::vector<std::size_t> TuckerModel::dims() const {
    std::vector<std::size_t> d;
    for (const auto& m : factors) d.push_back(m.rows());
    return d;
}

DenseTensor tucker_reconstruct(const DenseTensor& core, std::span<const Matrix> factors) {
    if (factors.size() != core.order()) throw ShapeError("tucker_reconstruct: expected one factor per mode");
    std::vector<std::size_t> shape;
    for (std::size_t n = 0; n < core.order(); ++n) {
        if (factors[n].cols() != core.dim(n))
            throw ShapeError("tucker_reconstruct: factor columns do not match core dimension");
        shape.push_back(factors[n].rows());
    }
    DenseTensor out(shape);
    const auto dims = u64(shape);
    const auto ranks = u64(core.shape());
    const auto flat = concat(std::vector<Matrix>(factors.begin(), factors.end()));
    ok(ntfg_tucker_reconstruct(ctx(), NTFG_F64, std::uint32_t(dims.size()), dims.data(), ranks.data(), core.data(),
                               flat.data(), out.data()));
    return out;
}

DenseTensor tucker_reconstruct(const TuckerModel& m) { return tucker_reconstruct(m.core, m.factors); }

DenseTensor tucker_multimode_contract(const DenseTensor& t, std::span<const Matrix> factors,
                                      std::optional<std::size_t> skip) {
    if (factors.size() != t.order()) throw ShapeError("tucker_multimode_contract: expected one factor per mode");
    if (skip && *skip >= t.order()) throw ShapeError("tucker_multimode_contract: skip mode out of range");
    std::vector<std::size_t> shape, cols;
    std::vector<Matrix> fs;
    for (std::size_t m = 0; m < t.order(); ++m) {
        cols.push_back(factors[m].cols());
        if (skip && *skip == m) {
            fs.push_back(Matrix(t.dim(m), factors[m].cols()));
            continue;
        }
        if (factors[m].rows() != t.dim(m))
            throw ShapeError("tucker_multimode_contract: factor rows do not match dimension");
        shape.push_back(factors[m].cols());
        fs.push_back(factors[m]);
    }
    if (skip) shape.push_back(t.dim(*skip));
    DenseTensor out(shape);
    const auto dims = u64(t.shape());
    const auto c = u64(cols);
    const auto flat = concat(fs);
    ok(ntfg_tucker_multimode_contract(ctx(), NTFG_F64, std::uint32_t(dims.size()), dims.data(), t.data(), c.data(),
                                      flat.data(), skip ? std::int32_t(*skip) : -1, out.data()));
    return out;
}

Matrix tucker_factor_contract(const DenseTensor& t, const DenseTensor& core, std::span<const Matrix> factors,
                              std::size_t mode) {
    if (factors.size() != t.order()) throw ShapeError("tucker_factor_contract: expected one factor per mode");
    if (core.order() != t.order()) throw ShapeError("tucker_factor_contract: core order does not match tensor order");
    if (mode >= t.order()) throw ShapeError("tucker_factor_contract: mode out of range");
    std::vector<Matrix> fs;
    for (std::size_t m = 0; m < t.order(); ++m) {
        if (m == mode) {
            fs.push_back(Matrix(t.dim(m), core.dim(m)));
            continue;
        }
        if (factors[m].rows() != t.dim(m) || factors[m].cols() != core.dim(m))
            throw ShapeError("tucker_factor_contract: factor shape mismatch");
        fs.push_back(factors[m]);
    }
    Matrix out(t.dim(mode), core.dim(mode));
    const auto dims = u64(t.shape());
    const auto ranks = u64(core.shape());
    const auto flat = concat(fs);
    ok(ntfg_tucker_factor_contract(ctx(), NTFG_F64, std::uint32_t(dims.size()), dims.data(), t.data(),
                                   ranks.data(), core.data(), flat.data(), std::uint32_t(mode),
                                   out.values().data()));
    return out;
}

static TuckerModel tucker_step(int kind, const TuckerModel& m, const DenseTensor& x, const BetaParam& p, double eps,
                               std::size_t mode, std::size_t inner, const double* ref_core,
                               const double* ref_factors) {
    require_dims(m.factors, x, "tucker_step");
    TuckerModel g = m;
    auto flat = concat(g.factors);
    const auto dims = u64(x.shape());
    const auto ranks = u64(m.core.shape());
    ok(ntfg_tucker_step(ctx(), NTFG_F64, kind, p.beta(), eps, inner, std::uint32_t(dims.size()), dims.data(),
                        x.data(), ranks.data(), ref_core, ref_factors, g.core.data(), flat.data(),
                        std::uint32_t(mode)));
    split_into(flat, g.factors);
    return g;
}

TuckerModel block_core_update(const TuckerModel& m, const DenseTensor& x, const BetaParam& p, double eps) {
    return tucker_step(0, m, x, p, eps, 0, 1, nullptr, nullptr);
}

TuckerModel block_core_update_anchored(const TuckerModel& m, const DenseTensor& anchor_core, const DenseTensor& x,
                                       const BetaParam& p, double eps) {
    if (anchor_core.shape() != m.core.shape()) throw ShapeError("block_core_update: anchor shape mismatch");
    return tucker_step(6, m, x, p, eps, 0, 1, anchor_core.data(), nullptr);
}

TuckerModel block_factor_update(const TuckerModel& m, std::size_t mode, const DenseTensor& x, const BetaParam& p,
                                double eps) {
    if (mode >= m.order()) throw ShapeError("block_factor_update: mode out of range");
    return tucker_step(1, m, x, p, eps, mode, 1, nullptr, nullptr);
}

TuckerModel block_factor_update_anchored(const TuckerModel& m, std::size_t mode, const Matrix& anchor,
                                         const DenseTensor& x, const BetaParam& p, double eps) {
    if (mode >= m.order()) throw ShapeError("block_factor_update: mode out of range");
    if (anchor.rows() != m.factors[mode].rows() || anchor.cols() != m.factors[mode].cols())
        throw ShapeError("block_factor_update: anchor shape mismatch");
    return tucker_step(7, m, x, p, eps, mode, 1, nullptr, anchor.values().data());
}

TuckerModel tucker_bcomm_sweep(const TuckerModel& m, const DenseTensor& x, const BetaParam& p, double eps) {
    return tucker_step(2, m, x, p, eps, 0, 1, nullptr, nullptr);
}

JcommTuckerReference make_jcomm_tucker_reference(const TuckerModel& ref, const DenseTensor& x, const BetaParam& p,
                                                 double eps) {
    require_dims(ref.factors, x, "make_jcomm_tucker_reference");
    JcommTuckerReference out{ref, DenseTensor(x.shape()), DenseTensor(x.shape())};
    const auto flat = concat(ref.factors);
    const auto dims = u64(x.shape());
    const auto ranks = u64(ref.core.shape());
    ok(ntfg_tucker_jcomm_reference(ctx(), NTFG_F64, p.beta(), eps, std::uint32_t(dims.size()), dims.data(), x.data(),
                                   ranks.data(), ref.core.data(), flat.data(), out.p.data(), out.q.data()));
    return out;
}

static TuckerModel tucker_inner(const TuckerModel& current, const JcommTuckerReference& c, int block,
                                const BetaParam& p, double eps) {
    require_dims(current.factors, c.p, "jcomm_inner_update");
    if (c.q.shape() != c.p.shape()) throw ShapeError("jcomm_inner_update: P/Q shape mismatch");
    TuckerModel g = current;
    auto flat = concat(g.factors);
    const auto rf = concat(c.ref.factors);
    const auto dims = u64(c.p.shape());
    const auto ranks = u64(current.core.shape());
    ok(ntfg_tucker_jcomm_inner_update(ctx(), NTFG_F64, p.beta(), eps, std::uint32_t(dims.size()), dims.data(),
                                      c.p.data(), c.q.data(), ranks.data(), c.ref.core.data(), rf.data(),
                                      g.core.data(), flat.data(), block));
    split_into(flat, g.factors);
    return g;
}

TuckerModel jcomm_inner_core_update(const TuckerModel& current, const JcommTuckerReference& c, const BetaParam& p,
                                    double eps) {
    return tucker_inner(current, c, -1, p, eps);
}

TuckerModel jcomm_inner_factor_update(const TuckerModel& current, const JcommTuckerReference& c, std::size_t mode,
                                      const BetaParam& p, double eps) {
    if (mode >= current.order()) throw ShapeError("jcomm_inner_factor_update: mode out of range");
    return tucker_inner(current, c, int(mode), p, eps);
}

TuckerModel jcomm_tucker_outer_step(const TuckerModel& m, const DenseTensor& x, const BetaParam& p,
                                    std::size_t inner_steps, double eps) {
    if (inner_steps < 1) throw DomainError("jcomm_tucker_outer_step: inner_steps must be >= 1");
    return tucker_step(3, m, x, p, eps, 0, inner_steps, nullptr, nullptr);
}

static TuckerFitResult tucker_fit(int algo, const DenseTensor& x, TuckerModel init, const FitConfig& cfg) {
    validate_fit_config(cfg);
    require_dims(init.factors, x, algo == NTFG_BCOMM ? "tucker_bcomm_fit" : "tucker_jcomm_fit");
    FitConfig c2 = cfg;
    c2.ranks = init.core.shape();
    std::vector<std::uint64_t> keep;
    ntfg_fit_config c = to_c(c2, keep);
    auto flat = concat(init.factors);
    std::vector<ntfg_trace_row> rows(cfg.max_iters + 1);
    std::uint64_t n = 0;
    const auto dims = u64(x.shape());
    ok(ntfg_tucker_fit(ctx(cfg.device), &c, algo, std::uint32_t(dims.size()), dims.data(), x.data(), 0, NTFG_HOST,
                       nullptr, init.core.data(), flat.data(), rows.data(), &n));
    TuckerFitResult out{std::move(init), trace_of(rows, n)};
    split_into(flat, out.model.factors);
    return out;
}

TuckerFitResult tucker_bcomm_fit(const DenseTensor& x, TuckerModel init, const FitConfig& cfg) {
    return tucker_fit(NTFG_BCOMM, x, std::move(init), cfg);
}

TuckerFitResult tucker_jcomm_fit(const DenseTensor& x, TuckerModel init, const FitConfig& cfg) {
    return tucker_fit(NTFG_JCOMM, x, std::move(init), cfg);
}

// ---- io.hpp (reference io.cpp): CTF1 / COO / trace through the C ABI ----------------

void write_tensor(const std::string& path, const DenseTensor& t) {
    const auto dims = u64(t.shape());
    ok(ntfg_ctf1_write(nullptr, path.c_str(), std::uint32_t(dims.size()), dims.data(), t.data(), 0, NTFG_HOST));
}

DenseTensor read_tensor(const std::string& path, std::size_t max_entries) {
    std::uint32_t order = 0;
    std::uint64_t dims[256];
    ok(ntfg_ctf1_header(path.c_str(), &order, dims, 256, max_entries));
    DenseTensor t(std::vector<std::size_t>(dims, dims + order));
    ok(ntfg_ctf1_read(nullptr, path.c_str(), t.data(), 0, NTFG_HOST, max_entries));
    return t;
}

DenseTensor cwise_max(const DenseTensor& a, double s) {
    DenseTensor out = a;
    for (double& v : out.values()) v = std::max(v, s);
    return out;
}

DenseTensor read_coo(const std::string& path, std::optional<double> floor, std::size_t max_entries) {
    std::uint32_t order = 0;
    std::uint64_t dims[256];
    std::uint64_t nnz = 0;
    ok(ntfg_coo_text_read(path.c_str(), &order, dims, 256, &nnz, nullptr, nullptr, 0, max_entries));
    std::vector<std::int32_t> idx(std::max<std::uint64_t>(nnz, 1) * order);
    std::vector<double> vals(std::max<std::uint64_t>(nnz, 1));
    ok(ntfg_coo_text_read(path.c_str(), &order, dims, 256, &nnz, idx.data(), vals.data(), nnz, max_entries));
    DenseTensor t(std::vector<std::size_t>(dims, dims + order));
    for (std::uint64_t e = 0; e < nnz; ++e) {  // duplicates accumulate in input order (io.cpp:138)
        std::size_t flat = 0;
        for (std::uint32_t m = 0; m < order; ++m) flat = flat * dims[m] + std::size_t(idx[e * order + m]);
        t[flat] += vals[e];
    }
    if (floor) return cwise_max(t, *floor);
    return t;
}

DenseTensor read_tensor_auto(const std::string& path, std::size_t max_entries) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw FormatError("cannot open: " + path);
    char head[4] = {};
    const std::size_t got = std::fread(head, 1, 4, f);
    std::fclose(f);
    if (got == 4 && std::memcmp(head, "CTF1", 4) == 0) return read_tensor(path, max_entries);
    return read_coo(path, std::nullopt, max_entries);
}

void write_trace(const std::string& path, std::span<const TraceRecord> records) {
    std::vector<ntfg_trace_row> rows(records.size());
    for (std::size_t i = 0; i < records.size(); ++i) rows[i] = {records[i].iter, records[i].time_s, records[i].loss};
    ok(ntfg_trace_write(path.c_str(), rows.data(), rows.size()));
}

std::vector<TraceRecord> read_trace(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "r");
    if (!f) throw FormatError("cannot open: " + path);
    std::vector<TraceRecord> out;
    char line[512];
    std::size_t lineno = 0;
    while (std::fgets(line, sizeof line, f)) {
        ++lineno;
        if (lineno == 1) {
            if (std::strncmp(line, "iter,time_s,loss", 16) != 0) {
                std::fclose(f);
                throw ParseError("trace header must be iter,time_s,loss", lineno);
            }
            continue;
        }
        unsigned long long it = 0;
        double t = 0.0, l = 0.0;
        if (std::sscanf(line, "%llu,%lf,%lf", &it, &t, &l) != 3) {
            std::fclose(f);
            throw ParseError("malformed trace row", lineno);
        }
        out.push_back({std::size_t(it), t, l});
    }
    std::fclose(f);
    return out;
}

// the reference generator: std::mt19937_64 seeded with seed_seq{seed lo, seed hi,
// stream lo, stream hi}; uniform01 keeps the top 53 bits (io.cpp:190-200)
Rng::Rng(std::uint64_t seed, std::uint64_t stream) {
    std::seed_seq seq{std::uint32_t(seed & 0xffffffffu), std::uint32_t(seed >> 32), std::uint32_t(stream & 0xffffffffu),
                      std::uint32_t(stream >> 32)};
    engine_.seed(seq);
}

double Rng::uniform01() { return double(engine_() >> 11) * 0x1.0p-53; }

static Matrix random_matrix(std::size_t rows, std::size_t cols, Rng& rng, double eps) {
    Matrix m(rows, cols);
    for (double& v : m.values()) v = std::max(rng.uniform01(), eps);
    return m;
}

CpFactors random_cp_factors(std::span<const std::size_t> dims, std::size_t rank, Rng& rng, double eps) {
    std::vector<Matrix> f;
    for (std::size_t d : dims) f.push_back(random_matrix(d, rank, rng, eps));
    return CpFactors(std::move(f));
}

TuckerModel random_tucker_model(std::span<const std::size_t> dims, std::span<const std::size_t> ranks, Rng& rng,
                                double eps) {
    if (dims.size() != ranks.size()) throw ShapeError("random_tucker_model: dims and ranks length mismatch");
    DenseTensor core(std::vector<std::size_t>(ranks.begin(), ranks.end()));
    for (double& v : core.values()) v = std::max(rng.uniform01(), eps);
    std::vector<Matrix> f;
    for (std::size_t n = 0; n < dims.size(); ++n) f.push_back(random_matrix(dims[n], ranks[n], rng, eps));
    return TuckerModel(std::move(core), std::move(f));
}

CpFactors init_cp_factors(std::span<const std::size_t> dims, std::size_t rank, std::uint64_t seed, double eps) {
    Rng rng(seed, Rng::kInitStream);
    return random_cp_factors(dims, rank, rng, eps);
}

TuckerModel init_tucker_model(std::span<const std::size_t> dims, std::span<const std::size_t> ranks,
                              std::uint64_t seed, double eps) {
    Rng rng(seed, Rng::kInitStream);
    return random_tucker_model(dims, ranks, rng, eps);
}

std::pair<DenseTensor, CpFactors> synth_cp(std::span<const std::size_t> dims, std::size_t rank, std::uint64_t seed,
                                           double eps) {
    Rng rng(seed, Rng::kSynthStream);
    CpFactors truth = random_cp_factors(dims, rank, rng, eps);
    DenseTensor x = cp_reconstruct(truth);
    return {std::move(x), std::move(truth)};
}

std::pair<DenseTensor, TuckerModel> synth_tucker(std::span<const std::size_t> dims,
                                                 std::span<const std::size_t> ranks, std::uint64_t seed,
                                                 double eps) {
    Rng rng(seed, Rng::kSynthStream);
    TuckerModel truth = random_tucker_model(dims, ranks, rng, eps);
    DenseTensor x = tucker_reconstruct(truth);
    return {std::move(x), std::move(truth)};
}

// ---- unfold.hpp (reference unfold.cpp) ---------------------------------------------

static std::vector<std::size_t> unfold_strides(const std::vector<std::size_t>& shape, std::size_t mode) {
    std::vector<std::size_t> st(shape.size(), 0);
    std::size_t stride = 1;
    for (std::size_t a = shape.size(); a-- > 0;) {  // remaining modes ascending, last fastest
        if (a == mode) continue;
        st[a] = stride;
        stride *= shape[a];
    }
    return st;
}

UnfoldedView unfold(const DenseTensor& t, std::size_t mode) {
    if (mode >= t.order()) throw ShapeError("unfold: mode out of range");
    const std::size_t rows = t.shape()[mode];
    const auto st = unfold_strides(t.shape(), mode);
    Matrix m(rows, t.size() / rows);
    MultiIndex idx(t.order(), 0);
    std::size_t flat = 0;
    do {
        std::size_t c = 0;
        for (std::size_t a = 0; a < t.order(); ++a)
            if (a != mode) c += idx[a] * st[a];
        m(idx[mode], c) = t[flat++];
    } while (next_multi_index(idx, t.shape()));
    return {std::move(m), mode};
}

DenseTensor refold(const UnfoldedView& u, std::span<const std::size_t> shape) {
    if (u.mode >= shape.size()) throw ShapeError("refold: mode out of range");
    DenseTensor t(std::vector<std::size_t>(shape.begin(), shape.end()));
    if (u.matrix.rows() != t.shape()[u.mode] || u.matrix.size() != t.size())
        throw ShapeError("refold: matrix does not match target shape");
    const auto st = unfold_strides(t.shape(), u.mode);
    MultiIndex idx(t.order(), 0);
    std::size_t flat = 0;
    do {
        std::size_t c = 0;
        for (std::size_t a = 0; a < t.order(); ++a)
            if (a != u.mode) c += idx[a] * st[a];
        t[flat++] = u.matrix(idx[u.mode], c);
    } while (next_multi_index(idx, t.shape()));
    return t;
}

Matrix khatri_rao(std::span<const Matrix> mats) {
    if (mats.empty()) throw ShapeError("khatri_rao: at least one matrix required");
    const std::size_t r = mats.front().cols();
    for (const Matrix& m : mats)
        if (m.cols() != r) throw ShapeError("khatri_rao: inconsistent column counts");
    Matrix out = mats.front();
    for (std::size_t k = 1; k < mats.size(); ++k) {
        const Matrix& b = mats[k];
        Matrix next(out.rows() * b.rows(), r);
        for (std::size_t ia = 0; ia < out.rows(); ++ia)
            for (std::size_t ib = 0; ib < b.rows(); ++ib)
                for (std::size_t c = 0; c < r; ++c) next(ia * b.rows() + ib, c) = out(ia, c) * b(ib, c);
        out = std::move(next);
    }
    return out;
}

CpFactors mu_unfold_cp_sweep(const CpFactors& f, const DenseTensor& x, const BetaParam& p, double eps) {
    require_dims(f.factors, x, "mu_unfold_cp_sweep");
    auto flat = concat(f.factors);
    const auto dims = u64(x.shape());
    ok(ntfg_cp_mu_unfold_sweep(ctx(), NTFG_F64, p.beta(), eps, std::uint32_t(dims.size()), dims.data(), x.data(),
                               f.rank(), flat.data()));
    CpFactors out = f;
    split_into(flat, out.factors);
    return out;
}

CpFitResult mu_unfold_cp_fit(const DenseTensor& x, CpFactors init, const FitConfig& cfg) {
    validate_fit_config(cfg);
    require_dims(init.factors, x, "mu_unfold_cp_fit");
    std::vector<std::uint64_t> keep;
    ntfg_fit_config c = to_c(cfg, keep);
    c.rank = init.rank();
    auto flat = concat(init.factors);
    std::vector<ntfg_trace_row> rows(cfg.max_iters + 1);
    std::uint64_t n = 0;
    const auto dims = u64(x.shape());
    ok(ntfg_cp_mu_unfold_fit(ctx(cfg.device), &c, std::uint32_t(dims.size()), dims.data(), x.data(), 0, NTFG_HOST,
                             flat.data(), rows.data(), &n));
    CpFitResult out{std::move(init), trace_of(rows, n)};
    split_into(flat, out.model.factors);
    return out;
}

TuckerModel mu_unfold_tucker_sweep(const TuckerModel& m, const DenseTensor& x, const BetaParam& p, double eps) {
    require_dims(m.factors, x, "mu_unfold_tucker_sweep");
    TuckerModel out = m;
    auto flat = concat(out.factors);
    const auto dims = u64(x.shape());
    const auto ranks = u64(m.core.shape());
    if (ranks.size() != dims.size()) throw ShapeError("TuckerModel: core order does not match factor count");
    ok(ntfg_tucker_mu_unfold_sweep(ctx(), NTFG_F64, p.beta(), eps, std::uint32_t(dims.size()), dims.data(),
                                   ranks.data(), x.data(), out.core.data(), flat.data()));
    split_into(flat, out.factors);
    return out;
}

TuckerFitResult mu_unfold_tucker_fit(const DenseTensor& x, TuckerModel init, const FitConfig& cfg) {
    validate_fit_config(cfg);
    require_dims(init.factors, x, "mu_unfold_tucker_fit");
    FitConfig c2 = cfg;
    c2.ranks = init.core.shape();
    std::vector<std::uint64_t> keep;
    ntfg_fit_config c = to_c(c2, keep);
    auto flat = concat(init.factors);
    std::vector<ntfg_trace_row> rows(cfg.max_iters + 1);
    std::uint64_t n = 0;
    const auto dims = u64(x.shape());
    ok(ntfg_tucker_mu_unfold_fit(ctx(cfg.device), &c, std::uint32_t(dims.size()), dims.data(), x.data(), 0,
                                 NTFG_HOST, init.core.data(), flat.data(), rows.data(), &n));
    TuckerFitResult out{std::move(init), trace_of(rows, n)};
    split_into(flat, out.model.factors);
    return out;
}

}  // namespace ntf

// ---- BMMe step-level API (reference cp.hpp:80-110, tucker.hpp:88-106) -----------------
namespace ntf {
namespace {
// sum over i of ([cur_i - prev_i]_+)^2
double pos_sq(const std::vector<double>& cur, const std::vector<double>& prev) {
    if (cur.size() != prev.size()) throw ShapeError("extrapolation: shape mismatch with recorded iterate");
    double s = 0.0;
    for (std::size_t i = 0; i < cur.size(); ++i) {
        const double d = cur[i] - prev[i];
        if (d > 0.0) s += d * d;
    }
    return s;
}
// max(cur + alpha [cur - prev]_+, eps)
void inertial(const std::vector<double>& cur, const std::vector<double>& prev, double alpha, double eps,
              std::vector<double>& out) {
    out.resize(cur.size());
    for (std::size_t i = 0; i < cur.size(); ++i) {
        const double d = cur[i] - prev[i];
        const double v = cur[i] + alpha * (d > 0.0 ? d : 0.0);
        out[i] = v < eps ? eps : v;
    }
}
// Nesterov: alpha_k = (t_k - 1) / t_{k+1}, t_{k+1} = (1 + sqrt(1 + 4 t_k^2)) / 2
double nesterov_step(double& t) {
    const double tn = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * t * t));
    const double a = (t - 1.0) / tn;
    t = tn;
    return a;
}
}  // namespace

ExtrapolationState make_extrapolation_state(const CpFactors& initial, bool enabled, double cap, double delta,
                                            double eps) {
    ExtrapolationState st;
    st.previous = initial;
    st.enabled = enabled;
    st.cap = cap;
    st.delta = delta;
    st.eps = eps;
    return st;
}

void extrapolation_begin_iteration(ExtrapolationState& st, const CpFactors& current) {
    if (current.order() != st.previous.order()) throw ShapeError("extrapolation: order mismatch");
    const double an = nesterov_step(st.t);
    double sq = 0.0;
    for (std::size_t n = 0; n < current.order(); ++n)
        sq += pos_sq(current.factors[n].values(), st.previous.factors[n].values());
    st.alpha = std::min(an, st.cap / (std::sqrt(sq) + st.delta));
}

Matrix extrapolate_block(const Matrix& current, const ExtrapolationState& st, std::size_t block) {
    if (block >= st.previous.order()) throw ShapeError("extrapolate_block: block out of range");
    const Matrix& prev = st.previous.factors[block];
    if (prev.rows() != current.rows() || prev.cols() != current.cols())
        throw ShapeError("extrapolate_block: shape mismatch with recorded iterate");
    Matrix out(current.rows(), current.cols());
    inertial(current.values(), prev.values(), st.alpha, st.eps, out.values());
    return out;
}

void extrapolation_end_iteration(ExtrapolationState& st, const CpFactors& iterate) { st.previous = iterate; }

TuckerExtrapolationState make_tucker_extrapolation_state(const TuckerModel& initial, bool enabled, double cap,
                                                         double delta, double eps) {
    TuckerExtrapolationState st;
    st.previous = initial;
    st.enabled = enabled;
    st.cap = cap;
    st.delta = delta;
    st.eps = eps;
    return st;
}

void extrapolation_begin_iteration(TuckerExtrapolationState& st, const TuckerModel& current) {
    if (current.order() != st.previous.order()) throw ShapeError("extrapolation: order mismatch");
    const double an = nesterov_step(st.t);
    double sq = pos_sq(current.core.values(), st.previous.core.values());
    for (std::size_t n = 0; n < current.order(); ++n)
        sq += pos_sq(current.factors[n].values(), st.previous.factors[n].values());
    st.alpha = std::min(an, st.cap / (std::sqrt(sq) + st.delta));
}

DenseTensor extrapolate_core(const DenseTensor& current, const TuckerExtrapolationState& st) {
    if (current.shape() != st.previous.core.shape())
        throw ShapeError("extrapolate_core: shape mismatch with recorded iterate");
    DenseTensor out(current.shape());
    inertial(current.values(), st.previous.core.values(), st.alpha, st.eps, out.values());
    return out;
}

Matrix extrapolate_block(const Matrix& current, const TuckerExtrapolationState& st, std::size_t mode) {
    if (mode >= st.previous.order()) throw ShapeError("extrapolate_block: mode out of range");
    const Matrix& prev = st.previous.factors[mode];
    if (prev.rows() != current.rows() || prev.cols() != current.cols())
        throw ShapeError("extrapolate_block: shape mismatch with recorded iterate");
    Matrix out(current.rows(), current.cols());
    inertial(current.values(), prev.values(), st.alpha, st.eps, out.values());
    return out;
}

void extrapolation_end_iteration(TuckerExtrapolationState& st, const TuckerModel& iterate) { st.previous = iterate; }

}  // namespace ntf
