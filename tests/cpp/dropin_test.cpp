// Drop-in check of the C++ API (include/ntf/ntf.hpp -> libntf_b200.so ->
// libntfg.so): a reference-style caller, written against the reference's
// public names and semantics (reference tests/test_cp.cpp, test_tucker.cpp,
// test_divergence.cpp), compiled unchanged against our headers.
// Exit code 0 and "ALL PASS" on success.
#include <cmath>
#include <cstdio>
#include <limits>
#include <string>

#include "ntf/cp.hpp"
#include "ntf/divergence.hpp"
#include "ntf/tucker.hpp"

using namespace ntf;

static int failures = 0;
#define CHECK(cond)                                                    \
    do {                                                               \
        if (!(cond)) {                                                 \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                \
        }                                                              \
    } while (0)

template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static DenseTensor data(std::vector<std::size_t> dims, unsigned seed) {
    DenseTensor t(dims);
    unsigned s = seed * 2654435761u + 1;
    for (double& v : t.values()) {
        s = s * 1664525u + 1013904223u;
        v = 0.1 + double(s >> 8) / double(1u << 24);
    }
    return t;
}

static CpFactors init(const std::vector<std::size_t>& dims, std::size_t r, unsigned seed) {
    std::vector<Matrix> f;
    unsigned s = seed * 97 + 13;
    for (auto d : dims) {
        Matrix m(d, r);
        for (double& v : m.values()) {
            s = s * 1664525u + 1013904223u;
            v = 0.1 + double(s >> 8) / double(1u << 24);
        }
        f.push_back(m);
    }
    return CpFactors(f);
}

static int run();
static const char* only = nullptr;  // debugging: run one stage (argv[1])
static bool want(const char* name) { return !only || std::string(only) == name; }
static const char* stage = "start";
int main(int argc, char** argv) {
    if (argc > 1) only = argv[1];
    std::setvbuf(stdout, nullptr, _IONBF, 0);
    try {
        return run();
    } catch (const std::exception& e) {
        std::printf("EXCEPTION in stage '%s': %s\n", stage, e.what());
        return 2;
    }
}

static int run() {
    stage = "kat";
    std::printf("stage %s\n", stage);
    // reconstruct KAT (test_cp.cpp:22-33)
    CpFactors rank1({Matrix(2, 1, {1.0, 2.0}), Matrix(2, 1, {3.0, 4.0})});
    CHECK(cp_reconstruct(rank1).values() == std::vector<double>({3.0, 4.0, 6.0, 8.0}));

    // scalar problem solved in one step (test_cp.cpp:35-42)
    const DenseTensor x1({1, 1}, {2.0});
    const BetaParam kl(1.0);
    CpFactors g = bcomm_block_update(CpFactors({Matrix::full(1, 1, 1.0), Matrix::full(1, 1, 1.0)}), 0, x1, kl, 1e-12);
    CHECK(g.factors[0](0, 0) == 2.0);
    CHECK(D_beta(x1, cp_reconstruct(g), kl) == 0.0);

    stage = "first-inner";
    std::printf("stage %s\n", stage);
    // first joint inner update == block update, bitwise (test_cp.cpp:116-128)
    if (want("first-inner"))
    for (double b : {0.0, 0.5, 1.0, 1.5}) {
        const DenseTensor x = data({6, 5, 4}, 3);
        const CpFactors f = init(x.shape(), 2, 3);
        const BetaParam p(b);
        const JcommCpReference ctx = make_jcomm_reference(f, x, p, 1e-12);
        CHECK(jcomm_inner_update(f, ctx, 0, p, 1e-12).factors[0].values() ==
              bcomm_block_update(f, 0, x, p, 1e-12).factors[0].values());
    }

    stage = "fit-drivers";
    std::printf("stage %s\n", stage);
    // fit drivers: stopping rules, monotone traces (test_cp.cpp:88-114)
    if (want("fit-drivers"))
    {
        const DenseTensor x = data({8, 7, 6}, 5);
        FitConfig cfg;
        cfg.rank = 3;
        cfg.max_iters = 0;
        const CpFactors f = init(x.shape(), 3, 5);
        const CpFitResult r0 = bcomm_fit(x, f, cfg);
        CHECK(r0.trace.size() == 1 && r0.model.factors[0].values() == f.factors[0].values());
        cfg.max_iters = 50;
        cfg.tol = std::numeric_limits<double>::infinity();
        CHECK(bcomm_fit(x, f, cfg).trace.size() == 2);
        cfg.tol = 0.0;
        for (double b : {0.0, 0.5, 1.0, 1.5}) {
            cfg.beta = b;
            for (auto* fit : {&bcomm_fit, &jcomm_fit}) {
                const CpFitResult r = (*fit)(x, f, cfg);
                CHECK(r.trace.size() == 51);
                for (std::size_t k = 1; k < r.trace.size(); ++k)
                    CHECK(r.trace[k].loss <= r.trace[k - 1].loss + 1e-12 * (1.0 + r.trace[k - 1].loss));
            }
        }
    }

    stage = "errors";
    std::printf("stage %s\n", stage);
    // error behaviour (config.cpp:7-18, fit_common.hpp:14-23)
    if (want("errors"))
    {
        FitConfig bad;
        bad.beta = 2.0;
        CHECK(throws<DomainError>([&] { validate_fit_config(bad); }));
        const DenseTensor x = data({4, 3, 2}, 1);
        FitConfig cfg;
        CHECK(throws<ShapeError>([&] { bcomm_fit(x, init({4, 3}, 1, 1), cfg); }));
        DenseTensor z = x;
        z[0] = 0.0;
        cfg.beta = 0.0;
        cfg.max_iters = 2;
        bool named = false;
        try {
            bcomm_fit(z, init(z.shape(), 1, 1), cfg);
        } catch (const NumericalError& e) {
            named = std::string(e.what()).find("data-floor") != std::string::npos;
        }
        CHECK(named);
    }

    stage = "tucker";
    std::printf("stage %s\n", stage);
    // Tucker: core KAT and joint descent (test_tucker.cpp:21-29, 96-115)
    if (want("tucker"))
    {
        const DenseTensor x = DenseTensor::full({2, 2}, 1.0);
        TuckerModel m(DenseTensor({1, 1}, {2.0}), {Matrix::full(2, 1, 1.0), Matrix::full(2, 1, 1.0)});
        const TuckerModel gm = block_core_update(m, x, kl, 1e-12);
        CHECK(gm.core[0] == 1.0);
        CHECK(D_beta(x, tucker_reconstruct(gm), kl) == 0.0);

        const DenseTensor y = data({5, 4, 3}, 23);
        const CpFactors f = init(y.shape(), 2, 23);
        TuckerModel t(DenseTensor::full({2, 2, 2}, 0.7), f.factors);
        for (double b : {0.0, 0.5, 1.0, 1.5}) {
            const BetaParam p(b);
            TuckerModel cur = t;
            for (int it = 0; it < 5; ++it) {
                const double before = D_beta(y, tucker_reconstruct(cur), p);
                cur = jcomm_tucker_outer_step(cur, y, p, 3, 1e-12);
                const double after = D_beta(y, tucker_reconstruct(cur), p);
                CHECK(after <= before + 1e-12 * (1.0 + before));
            }
        }
        FitConfig cfg;
        cfg.max_iters = 30;
        const TuckerFitResult r = tucker_jcomm_fit(y, t, cfg);
        CHECK(r.trace.size() == 31);
    }

    stage = "bmme";
    std::printf("stage %s\n", stage);
    // BMMe step-level API (cp.hpp:80-110): a hand-written extrapolated B-CoMM
    // loop equals bcomm_fit(extrapolate) (reference test_cp.cpp:169-216 style);
    // cap = 0 pins alpha to 0 (test_cp.cpp:218-234)
    if (want("bmme"))
    {
        const DenseTensor x = data({6, 5, 4}, 31);
        const BetaParam p(0.5);
        FitConfig cfg;
        cfg.beta = 0.5;
        cfg.max_iters = 4;
        cfg.extrapolate = true;
        cfg.extrap_cap = 5.0;
        const CpFactors f0 = init(x.shape(), 3, 31);
        const CpFitResult r = bcomm_fit(x, f0, cfg);
        CpFactors f = f0;
        ExtrapolationState st = make_extrapolation_state(f, true, cfg.extrap_cap, cfg.extrap_delta, cfg.eps);
        for (int it = 0; it < 4; ++it) {
            const CpFactors snap = f;
            extrapolation_begin_iteration(st, f);
            for (std::size_t n = 0; n < f.order(); ++n)
                f = cp_block_update_anchored(f, n, extrapolate_block(f.factors[n], st, n), x, p, cfg.eps);
            extrapolation_end_iteration(st, snap);
        }
        double err = 0.0;
        for (std::size_t n = 0; n < f.order(); ++n)
            for (std::size_t i = 0; i < f.factors[n].size(); ++i)
                err = std::max(err, std::abs(f.factors[n].values()[i] - r.model.factors[n].values()[i]) /
                                        std::max(1.0, std::abs(r.model.factors[n].values()[i])));
        CHECK(err < 1e-10);
        ExtrapolationState z = make_extrapolation_state(f0, true, 0.0, 1e-6, 1e-12);
        extrapolation_begin_iteration(z, f);
        CHECK(z.alpha == 0.0);
        CHECK(extrapolate_block(f.factors[0], z, 0).values() == f.factors[0].values());
        TuckerModel tm(DenseTensor::full({3, 3, 3}, 0.7), f.factors);
        TuckerExtrapolationState ts = make_tucker_extrapolation_state(tm, true, 1.0, 1e-6, 1e-12);
        extrapolation_begin_iteration(ts, tm);
        CHECK(extrapolate_core(tm.core, ts).values() == tm.core.values());
    }

    stage = "tucker-cache";
    std::printf("stage %s\n", stage);
    // Tucker joint-MM cache holds host P~/Q~ (tucker.hpp:59-63); first inner
    // core update == block core update (test_tucker.cpp:83-94)
    if (want("tucker-cache"))
    {
        const DenseTensor y = data({5, 4, 3}, 41);
        const CpFactors f = init(y.shape(), 2, 41);
        const TuckerModel t(DenseTensor::full({2, 2, 2}, 0.6), f.factors);
        for (double b : {0.0, 0.5, 1.0, 1.5}) {
            const BetaParam p(b);
            const JcommTuckerReference c = make_jcomm_tucker_reference(t, y, p, 1e-12);
            CHECK(c.p.shape() == y.shape() && c.q.shape() == y.shape());
            const TuckerModel j = jcomm_inner_core_update(t, c, p, 1e-12);
            const TuckerModel k = block_core_update(t, y, p, 1e-12);
            CHECK(j.core.values() == k.core.values());
            const TuckerModel j1 = jcomm_inner_factor_update(t, c, 1, p, 1e-12);
            const TuckerModel k1 = block_factor_update(t, 1, y, p, 1e-12);
            CHECK(j1.factors[1].values() == k1.factors[1].values());
        }
    }

    if (failures == 0) std::printf("ALL PASS\n");
    return failures == 0 ? 0 : 1;
}
