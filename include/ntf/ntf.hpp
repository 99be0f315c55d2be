// ntf -- drop-in C++ solver API of the B200 engine (libntf_b200.so).
//
// Same namespace, type names, signatures and exception behaviour as the
// reference library (/root/reference/proj/include/ntf/*.hpp); every compute
// entry point forwards through the C ABI of libntfg.so (include/ntfg.h) to
// the sm_100a kernels.  Source-compatible for the reference's callers: the
// per-module headers (ntf/cp.hpp, ntf/tucker.hpp, ...) all include this file.
//
// Additions (north star: new options as NEW fields): FitConfig::precision
// (fp64 validation build by default, fp32 streaming) and FitConfig::use_graphs.
#pragma once

#include <cstddef>
#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace ntf {

// ---- errors (reference errors.hpp) -------------------------------------------
class ShapeError : public std::invalid_argument {
public:
    using std::invalid_argument::invalid_argument;
};
class DomainError : public std::domain_error {
public:
    using std::domain_error::domain_error;
};
class FormatError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class ParseError : public FormatError {
public:
    ParseError(const std::string& message, std::size_t line)
        : FormatError("line " + std::to_string(line) + ": " + message), line_(line) {}
    std::size_t line() const { return line_; }

private:
    std::size_t line_;
};
class NumericalError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
/// CUDA / collective failures of the device engine (no reference analogue).
class DeviceError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

// ---- value types (reference tensor.hpp) ------------------------------------------
using MultiIndex = std::vector<std::size_t>;

class DenseTensor {
public:
    DenseTensor() = default;
    explicit DenseTensor(std::vector<std::size_t> shape);
    DenseTensor(std::vector<std::size_t> shape, std::vector<double> values);
    static DenseTensor full(std::vector<std::size_t> shape, double value);

    std::size_t order() const { return shape_.size(); }
    const std::vector<std::size_t>& shape() const { return shape_; }
    std::size_t dim(std::size_t axis) const { return shape_[axis]; }
    std::size_t size() const { return values_.size(); }
    double* data() { return values_.data(); }
    const double* data() const { return values_.data(); }
    std::vector<double>& values() { return values_; }
    const std::vector<double>& values() const { return values_; }
    double operator[](std::size_t i) const { return values_[i]; }
    double& operator[](std::size_t i) { return values_[i]; }
    std::size_t flat_index(std::span<const std::size_t> index) const;
    double at(std::span<const std::size_t> index) const { return values_[flat_index(index)]; }
    double& at(std::span<const std::size_t> index) { return values_[flat_index(index)]; }

private:
    std::vector<std::size_t> shape_;
    std::vector<double> values_;
};

class Matrix {
public:
    Matrix() = default;
    Matrix(std::size_t rows, std::size_t cols);
    Matrix(std::size_t rows, std::size_t cols, std::vector<double> values);
    static Matrix full(std::size_t rows, std::size_t cols, double value);
    static Matrix identity(std::size_t n);

    std::size_t rows() const { return rows_; }
    std::size_t cols() const { return cols_; }
    std::size_t size() const { return values_.size(); }
    double operator()(std::size_t i, std::size_t j) const { return values_[i * cols_ + j]; }
    double& operator()(std::size_t i, std::size_t j) { return values_[i * cols_ + j]; }
    const double* row(std::size_t i) const { return values_.data() + i * cols_; }
    double* row(std::size_t i) { return values_.data() + i * cols_; }
    std::vector<double>& values() { return values_; }
    const std::vector<double>& values() const { return values_; }

private:
    std::size_t rows_ = 0, cols_ = 0;
    std::vector<double> values_;
};

bool next_multi_index(MultiIndex& index, std::span<const std::size_t> shape);

// ---- config (reference config.hpp) -------------------------------------------------
enum class ModelKind { cp, tucker };
enum class Algo { bcomm, jcomm, mu_unfold };
enum class Precision { f64, f32 };

struct TraceRecord {
    std::size_t iter = 0;
    double time_s = 0.0;
    double loss = 0.0;
};

struct FitConfig {
    ModelKind model = ModelKind::cp;
    Algo algo = Algo::bcomm;
    double beta = 1.0;
    std::size_t rank = 1;
    std::vector<std::size_t> ranks;
    double eps = 1e-12;
    std::size_t inner_steps = 3;
    std::size_t max_iters = 500;
    double tol = 0.0;
    std::uint64_t seed = 0;
    bool extrapolate = false;
    double extrap_cap = 1.0;
    double extrap_delta = 1e-6;
    std::optional<double> data_floor;
    // additions
    Precision precision = Precision::f64;
    bool use_graphs = true;
    int device = 0;
};

void validate_fit_config(const FitConfig& cfg);

// ---- divergence (reference divergence.hpp) -------------------------------------------
class BetaParam {
public:
    explicit BetaParam(double beta);
    double beta() const { return beta_; }
    double gamma() const { return gamma_; }

private:
    double beta_, gamma_;
};

double d_beta(double x, double y, const BetaParam& p);
double D_beta(const DenseTensor& x, const DenseTensor& xhat, const BetaParam& p);
double D_beta_mean(const DenseTensor& x, const DenseTensor& xhat, const BetaParam& p);

// ---- CP (reference cp.hpp) ------------------------------------------------------------
struct CpFactors {
    std::vector<Matrix> factors;
    CpFactors() = default;
    explicit CpFactors(std::vector<Matrix> f);
    std::size_t order() const { return factors.size(); }
    std::size_t rank() const { return factors.empty() ? 0 : factors.front().cols(); }
    std::vector<std::size_t> dims() const;
};

struct CpFitResult {
    CpFactors model;
    std::vector<TraceRecord> trace;
};

DenseTensor cp_reconstruct(const CpFactors& f);
Matrix cp_contract(const DenseTensor& t, std::span<const Matrix> factors, std::size_t mode);

CpFactors bcomm_block_update(const CpFactors& f, std::size_t mode, const DenseTensor& x,
                             const BetaParam& p, double eps);
CpFactors cp_block_update_anchored(const CpFactors& f, std::size_t mode, const Matrix& anchor,
                                   const DenseTensor& x, const BetaParam& p, double eps);
CpFactors bcomm_sweep(const CpFactors& f, const DenseTensor& x, const BetaParam& p, double eps);
CpFitResult bcomm_fit(const DenseTensor& x, CpFactors init, const FitConfig& cfg);

struct JcommCpReference {
    CpFactors ref;
    DenseTensor p;
    DenseTensor q;
};
JcommCpReference make_jcomm_reference(const CpFactors& ref, const DenseTensor& x, const BetaParam& p,
                                      double eps);
CpFactors jcomm_inner_update(const CpFactors& current, const JcommCpReference& ctx, std::size_t mode,
                             const BetaParam& p, double eps);
CpFactors jcomm_outer_step(const CpFactors& f, const DenseTensor& x, const BetaParam& p,
                           std::size_t inner_steps, double eps);
CpFitResult jcomm_fit(const DenseTensor& x, CpFactors init, const FitConfig& cfg);

/// BMMe step-level API (reference cp.hpp:80-110).  Factor-sized host
/// arithmetic, as in the reference; the fit drivers run the same scheme on
/// the device (extrap_norm / extrap_apply kernels).
struct ExtrapolationState {
    CpFactors previous;
    double t = 1.0;
    double alpha = 0.0;
    double cap = 1.0;
    double delta = 1e-6;
    double eps = 1e-12;
    bool enabled = false;
};
ExtrapolationState make_extrapolation_state(const CpFactors& initial, bool enabled, double cap, double delta,
                                            double eps);
void extrapolation_begin_iteration(ExtrapolationState& st, const CpFactors& current);
Matrix extrapolate_block(const Matrix& current, const ExtrapolationState& st, std::size_t block);
void extrapolation_end_iteration(ExtrapolationState& st, const CpFactors& iterate);

// ---- Tucker (reference tucker.hpp, tensor.hpp contractions) -------------------------------
struct TuckerModel {
    DenseTensor core;
    std::vector<Matrix> factors;
    TuckerModel() = default;
    TuckerModel(DenseTensor core, std::vector<Matrix> factors);
    std::size_t order() const { return factors.size(); }
    std::vector<std::size_t> dims() const;
    const std::vector<std::size_t>& ranks() const { return core.shape(); }
};

struct TuckerFitResult {
    TuckerModel model;
    std::vector<TraceRecord> trace;
};

DenseTensor tucker_reconstruct(const DenseTensor& core, std::span<const Matrix> factors);
DenseTensor tucker_reconstruct(const TuckerModel& m);
DenseTensor tucker_multimode_contract(const DenseTensor& t, std::span<const Matrix> factors,
                                      std::optional<std::size_t> skip = std::nullopt);
Matrix tucker_factor_contract(const DenseTensor& t, const DenseTensor& core,
                              std::span<const Matrix> factors, std::size_t mode);

TuckerModel block_core_update(const TuckerModel& m, const DenseTensor& x, const BetaParam& p, double eps);
TuckerModel block_core_update_anchored(const TuckerModel& m, const DenseTensor& anchor_core,
                                       const DenseTensor& x, const BetaParam& p, double eps);
TuckerModel block_factor_update(const TuckerModel& m, std::size_t mode, const DenseTensor& x,
                                const BetaParam& p, double eps);
TuckerModel block_factor_update_anchored(const TuckerModel& m, std::size_t mode, const Matrix& anchor,
                                         const DenseTensor& x, const BetaParam& p, double eps);
TuckerModel tucker_bcomm_sweep(const TuckerModel& m, const DenseTensor& x, const BetaParam& p, double eps);
TuckerFitResult tucker_bcomm_fit(const DenseTensor& x, TuckerModel init, const FitConfig& cfg);

/// Reference tucker.hpp:59-63: the reference model plus host copies of its
/// P~/Q~ (computed on the device by make_jcomm_tucker_reference and uploaded
/// again by the inner updates, like the CP JcommCpReference).
struct JcommTuckerReference {
    TuckerModel ref;
    DenseTensor p;
    DenseTensor q;
};
JcommTuckerReference make_jcomm_tucker_reference(const TuckerModel& ref, const DenseTensor& x,
                                                 const BetaParam& p, double eps);
TuckerModel jcomm_inner_core_update(const TuckerModel& current, const JcommTuckerReference& ctx,
                                    const BetaParam& p, double eps);
TuckerModel jcomm_inner_factor_update(const TuckerModel& current, const JcommTuckerReference& ctx,
                                      std::size_t mode, const BetaParam& p, double eps);
TuckerModel jcomm_tucker_outer_step(const TuckerModel& m, const DenseTensor& x, const BetaParam& p,
                                    std::size_t inner_steps, double eps);
TuckerFitResult tucker_jcomm_fit(const DenseTensor& x, TuckerModel init, const FitConfig& cfg);

/// reference tucker.hpp:88-106: block 0 is the core, block n+1 is factor n.
struct TuckerExtrapolationState {
    TuckerModel previous;
    double t = 1.0;
    double alpha = 0.0;
    double cap = 1.0;
    double delta = 1e-6;
    double eps = 1e-12;
    bool enabled = false;
};
TuckerExtrapolationState make_tucker_extrapolation_state(const TuckerModel& initial, bool enabled, double cap,
                                                         double delta, double eps);
void extrapolation_begin_iteration(TuckerExtrapolationState& st, const TuckerModel& current);
DenseTensor extrapolate_core(const DenseTensor& current, const TuckerExtrapolationState& st);
Matrix extrapolate_block(const Matrix& current, const TuckerExtrapolationState& st, std::size_t mode);
void extrapolation_end_iteration(TuckerExtrapolationState& st, const TuckerModel& iterate);

}  // namespace ntf
