// ntf-cli: the reference command-line front end (tools/ntf_main.cpp:1-360)
// over the B200 drop-in library -- same subcommands (synth-cp, synth-tucker,
// fit, bench), options, outputs (CTF1 models, trace CSV, long-format bench
// CSV) and exit codes (0 ok, 1 usage/domain, 2 numerical failure, 3 format).
// Fits run on the GPU (libntf_b200 -> libntfg).  Extra option (new):
// --precision f64|f32 selects the streaming type (default f64, the
// reference's arithmetic).  The reference's CLI11 is not used: the grammar
// here is `--name value` / `--name=value`, lists comma separated.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "ntf/io.hpp"
#include "ntf/ntf.hpp"
#include "ntf/unfold.hpp"

namespace {

struct Usage : std::runtime_error {
    using std::runtime_error::runtime_error;
};

double default_eps() {  // NTF_EPS overrides (ntf_main.cpp:24-31)
    if (const char* env = std::getenv("NTF_EPS")) {
        char* end = nullptr;
        const double v = std::strtod(env, &end);
        if (end != env && v > 0.0) return v;
    }
    return 1e-12;
}

// --name value | --name=value | flags; every option must be known to the subcommand
struct Args {
    std::map<std::string, std::string> kv;
    std::map<std::string, bool> flags;

    Args(int argc, char** argv, int first, const std::vector<std::string>& options,
         const std::vector<std::string>& flag_names) {
        for (int i = first; i < argc; ++i) {
            std::string a = argv[i];
            if (a.rfind("--", 0) != 0) throw Usage("unexpected argument: " + a);
            std::string name = a.substr(2), val;
            const auto eq = name.find('=');
            bool has_val = false;
            if (eq != std::string::npos) {
                val = name.substr(eq + 1);
                name = name.substr(0, eq);
                has_val = true;
            }
            if (std::find(flag_names.begin(), flag_names.end(), name) != flag_names.end()) {
                if (has_val) throw Usage("--" + name + " takes no value");
                flags[name] = true;
                continue;
            }
            if (std::find(options.begin(), options.end(), name) == options.end())
                throw Usage("unknown option: --" + name);
            if (!has_val) {
                if (i + 1 >= argc) throw Usage("--" + name + " requires a value");
                val = argv[++i];
            }
            kv[name] = val;
        }
    }
    bool has(const std::string& n) const { return kv.count(n) != 0; }
    std::string str(const std::string& n, const std::string& def = "") const {
        auto it = kv.find(n);
        return it == kv.end() ? def : it->second;
    }
    std::string req(const std::string& n) const {
        if (!has(n)) throw Usage("--" + n + " is required");
        return kv.at(n);
    }
    double num(const std::string& n, double def) const {
        if (!has(n)) return def;
        char* end = nullptr;
        const std::string& s = kv.at(n);
        const double v = std::strtod(s.c_str(), &end);
        if (end == s.c_str() || *end) throw Usage("--" + n + ": not a number: " + s);
        return v;
    }
    std::uint64_t u64(const std::string& n, std::uint64_t def) const {
        if (!has(n)) return def;
        return parse_u64(n, kv.at(n));
    }
    static std::uint64_t parse_u64(const std::string& n, const std::string& s) {
        char* end = nullptr;
        if (s.empty() || s[0] == '-') throw Usage("--" + n + ": not a nonnegative integer: " + s);
        const unsigned long long v = std::strtoull(s.c_str(), &end, 10);
        if (*end) throw Usage("--" + n + ": not a nonnegative integer: " + s);
        return v;
    }
    std::vector<std::uint64_t> list(const std::string& n) const {
        std::vector<std::uint64_t> out;
        if (!has(n)) return out;
        std::string s = kv.at(n);
        std::size_t p = 0;
        while (p <= s.size()) {
            const auto q = s.find(',', p);
            out.push_back(parse_u64(n, s.substr(p, q == std::string::npos ? std::string::npos : q - p)));
            if (q == std::string::npos) break;
            p = q + 1;
        }
        return out;
    }
    std::vector<std::string> strs(const std::string& n) const {
        std::vector<std::string> out;
        if (!has(n)) return out;
        std::string s = kv.at(n);
        std::size_t p = 0;
        while (true) {
            const auto q = s.find(',', p);
            out.push_back(s.substr(p, q == std::string::npos ? std::string::npos : q - p));
            if (q == std::string::npos) break;
            p = q + 1;
        }
        return out;
    }
};

std::vector<std::size_t> sizes(const std::vector<std::uint64_t>& v) { return {v.begin(), v.end()}; }

std::string dims_to_string(const std::vector<std::size_t>& dims) {
    std::string out;
    for (std::size_t i = 0; i < dims.size(); ++i) out += (i ? "," : "") + std::to_string(dims[i]);
    return out;
}

ntf::Algo parse_algo(const std::string& s) {
    if (s == "bcomm") return ntf::Algo::bcomm;
    if (s == "jcomm") return ntf::Algo::jcomm;
    if (s == "mu-unfold") return ntf::Algo::mu_unfold;
    throw ntf::DomainError("unknown algorithm: " + s);
}

void write_cp_model(const std::string& prefix, const ntf::CpFactors& f) {
    for (std::size_t n = 0; n < f.factors.size(); ++n) {
        const ntf::Matrix& m = f.factors[n];
        ntf::write_tensor(prefix + ".factor" + std::to_string(n) + ".ctf", ntf::DenseTensor({m.rows(), m.cols()}, m.values()));
    }
}

void write_tucker_model(const std::string& prefix, const ntf::TuckerModel& m) {
    ntf::write_tensor(prefix + ".core.ctf", m.core);
    for (std::size_t n = 0; n < m.factors.size(); ++n) {
        const ntf::Matrix& a = m.factors[n];
        ntf::write_tensor(prefix + ".factor" + std::to_string(n) + ".ctf", ntf::DenseTensor({a.rows(), a.cols()}, a.values()));
    }
}

int run_synth(const Args& a, bool tucker) {
    const auto dims = sizes(a.list("dims"));
    if (!a.has("dims") || dims.empty()) throw Usage("--dims is required and must be nonempty");
    for (std::size_t d : dims)
        if (d == 0) throw Usage("--dims entries must be positive");
    const std::uint64_t seed = a.u64("seed", 0);
    const double eps = a.num("eps", default_eps());
    const std::string out = a.req("out");
    const std::string truth_prefix = a.str("truth");
    ntf::DenseTensor x;
    double loss = 0.0;
    const ntf::BetaParam p(1.0);
    if (!tucker) {
        const std::size_t rank = a.u64("rank", 0);
        if (!a.has("rank")) throw Usage("--rank is required");
        if (rank < 1) throw Usage("--rank must be >= 1");
        auto [xx, truth] = ntf::synth_cp(dims, rank, seed, eps);
        x = std::move(xx);
        if (!truth_prefix.empty()) write_cp_model(truth_prefix, truth);
        loss = ntf::D_beta_mean(x, ntf::cp_reconstruct(truth), p);
    } else {
        const auto ranks = sizes(a.list("ranks"));
        if (!a.has("ranks")) throw Usage("--ranks is required");
        if (ranks.size() != dims.size()) throw Usage("--ranks must match --dims in length");
        for (std::size_t j : ranks)
            if (j == 0) throw Usage("--ranks entries must be positive");
        auto [xx, truth] = ntf::synth_tucker(dims, ranks, seed, eps);
        x = std::move(xx);
        if (!truth_prefix.empty()) write_tucker_model(truth_prefix, truth);
        loss = ntf::D_beta_mean(x, ntf::tucker_reconstruct(truth), p);
    }
    ntf::write_tensor(out, x);
    std::printf("dims %s seed %llu loss %.17g\n", dims_to_string(dims).c_str(), (unsigned long long)seed, loss);
    return 0;
}

struct FitOpts {
    std::string model = "cp", algo = "bcomm";
    double beta = 1.0;
    std::size_t rank = 1, inner = 3, max_iters = 500;
    std::vector<std::size_t> ranks;
    double tol = 0.0, eps = default_eps(), extrap_cap = 1.0;
    std::uint64_t seed = 0;
    bool extrapolate = false;
    std::optional<double> data_floor;
    ntf::Precision precision = ntf::Precision::f64;
};

FitOpts common_opts(const Args& a, std::size_t default_iters) {
    FitOpts o;
    o.model = a.str("model", "cp");
    if (o.model != "cp" && o.model != "tucker") throw Usage("--model: must be cp or tucker");
    o.beta = a.num("beta", 1.0);
    o.rank = a.u64("rank", 1);
    o.ranks = sizes(a.list("ranks"));
    o.inner = a.u64("inner", 3);
    o.max_iters = a.u64("max-iters", default_iters);
    o.eps = a.num("eps", default_eps());
    const std::string prec = a.str("precision", "f64");
    if (prec != "f64" && prec != "f32") throw Usage("--precision: must be f64 or f32");
    o.precision = prec == "f32" ? ntf::Precision::f32 : ntf::Precision::f64;
    return o;
}

ntf::FitConfig to_config(const FitOpts& o) {
    ntf::FitConfig cfg;
    cfg.model = o.model == "cp" ? ntf::ModelKind::cp : ntf::ModelKind::tucker;
    cfg.algo = parse_algo(o.algo);
    cfg.beta = o.beta;
    cfg.rank = o.rank;
    cfg.ranks = o.ranks;
    cfg.eps = o.eps;
    cfg.inner_steps = o.inner;
    cfg.max_iters = o.max_iters;
    cfg.tol = o.tol;
    cfg.seed = o.seed;
    cfg.extrapolate = o.extrapolate;
    cfg.extrap_cap = o.extrap_cap;
    cfg.data_floor = o.data_floor;
    cfg.precision = o.precision;
    ntf::validate_fit_config(cfg);
    return cfg;
}

// one fit from the seeded init (init stream), as run_fit / run_bench do
std::vector<ntf::TraceRecord> fit_once(const ntf::DenseTensor& x, const ntf::FitConfig& cfg, const std::string& out_prefix) {
    if (cfg.model == ntf::ModelKind::cp) {
        ntf::CpFactors init = ntf::init_cp_factors(x.shape(), cfg.rank, cfg.seed, cfg.eps);
        ntf::CpFitResult res;
        switch (cfg.algo) {
            case ntf::Algo::bcomm: res = ntf::bcomm_fit(x, std::move(init), cfg); break;
            case ntf::Algo::jcomm: res = ntf::jcomm_fit(x, std::move(init), cfg); break;
            case ntf::Algo::mu_unfold: res = ntf::mu_unfold_cp_fit(x, std::move(init), cfg); break;
        }
        if (!out_prefix.empty()) write_cp_model(out_prefix, res.model);
        return res.trace;
    }
    if (cfg.ranks.size() != x.order()) throw Usage("--ranks must provide one core rank per tensor mode");
    ntf::TuckerModel init = ntf::init_tucker_model(x.shape(), cfg.ranks, cfg.seed, cfg.eps);
    ntf::TuckerFitResult res;
    switch (cfg.algo) {
        case ntf::Algo::bcomm: res = ntf::tucker_bcomm_fit(x, std::move(init), cfg); break;
        case ntf::Algo::jcomm: res = ntf::tucker_jcomm_fit(x, std::move(init), cfg); break;
        case ntf::Algo::mu_unfold: res = ntf::mu_unfold_tucker_fit(x, std::move(init), cfg); break;
    }
    if (!out_prefix.empty()) write_tucker_model(out_prefix, res.model);
    return res.trace;
}

int run_fit(const Args& a) {
    FitOpts o = common_opts(a, 500);
    o.algo = a.str("algo", "bcomm");
    if (o.algo != "bcomm" && o.algo != "jcomm" && o.algo != "mu-unfold")
        throw Usage("--algo: must be bcomm, jcomm or mu-unfold");
    o.tol = a.num("tol", 0.0);
    o.seed = a.u64("seed", 0);
    o.extrapolate = a.flags.count("extrapolate") != 0;
    o.extrap_cap = a.num("extrap-cap", 1.0);
    if (a.has("data-floor")) o.data_floor = a.num("data-floor", 0.0);
    const ntf::FitConfig cfg = to_config(o);
    ntf::DenseTensor x = ntf::read_tensor_auto(a.req("input"));
    if (cfg.data_floor) x = ntf::cwise_max(x, *cfg.data_floor);
    const auto trace = fit_once(x, cfg, a.str("out"));
    if (a.has("trace")) ntf::write_trace(a.str("trace"), trace);
    std::printf("iters %zu final_loss %.17g\n", trace.back().iter, trace.back().loss);
    return 0;
}

int run_bench(const Args& a) {
    const auto algos = a.strs("algos");
    const auto seeds = a.list("seeds");
    if (!a.has("algos") || algos.empty()) throw Usage("--algos must name at least one algorithm");
    if (!a.has("seeds") || seeds.empty()) throw Usage("--seeds must list at least one seed");
    FitOpts base = common_opts(a, 100);
    for (const std::string& s : algos) parse_algo(s);  // validate up front
    const std::string out = a.req("out");
    const ntf::DenseTensor x = ntf::read_tensor_auto(a.req("input"));
    std::FILE* os = std::fopen(out.c_str(), "w");
    if (!os) throw ntf::FormatError("cannot open for writing: " + out);
    std::fputs("algo,seed,iter,time_s,loss\n", os);
    for (const std::string& algo : algos) {
        for (std::uint64_t seed : seeds) {
            FitOpts o = base;
            o.algo = algo;
            o.seed = seed;
            for (const ntf::TraceRecord& r : fit_once(x, to_config(o), "")) {
                if (r.iter == 0) continue;  // data rows start at the first iteration
                std::fprintf(os, "%s,%llu,%zu,%.17g,%.17g\n", algo.c_str(), (unsigned long long)seed, r.iter, r.time_s,
                             r.loss);
            }
        }
    }
    std::fclose(os);
    return 0;
}

const char* kUsage =
    "usage: ntf-cli <synth-cp|synth-tucker|fit|bench> [options]\n"
    "  synth-cp     --dims I1,I2,.. --rank R --out X.ctf [--seed S] [--eps E] [--truth PREFIX]\n"
    "  synth-tucker --dims I1,.. --ranks J1,.. --out X.ctf [--seed S] [--eps E] [--truth PREFIX]\n"
    "  fit          --input X [--model cp|tucker] [--algo bcomm|jcomm|mu-unfold] [--beta B] [--rank R]\n"
    "               [--ranks J1,..] [--inner L] [--max-iters K] [--tol T] [--seed S] [--eps E]\n"
    "               [--extrapolate] [--extrap-cap C] [--data-floor F] [--trace CSV] [--out PREFIX]\n"
    "               [--precision f64|f32]\n"
    "  bench        --input X --algos a,b --seeds s1,s2 --out CSV [--model ..] [--beta ..] [--rank ..]\n"
    "               [--ranks ..] [--inner ..] [--max-iters ..] [--eps ..] [--precision ..]\n";

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fputs(kUsage, stderr);
        return 1;
    }
    const std::string cmd = argv[1];
    if (cmd == "--help" || cmd == "-h") {
        std::fputs(kUsage, stdout);
        return 0;
    }
    try {
        if (cmd == "synth-cp")
            return run_synth(Args(argc, argv, 2, {"dims", "rank", "seed", "eps", "out", "truth"}, {}), false);
        if (cmd == "synth-tucker")
            return run_synth(Args(argc, argv, 2, {"dims", "ranks", "seed", "eps", "out", "truth"}, {}), true);
        if (cmd == "fit")
            return run_fit(Args(argc, argv, 2,
                                {"input", "model", "algo", "beta", "rank", "ranks", "inner", "max-iters", "tol", "seed",
                                 "eps", "extrap-cap", "data-floor", "trace", "out", "precision"},
                                {"extrapolate"}));
        if (cmd == "bench")
            return run_bench(Args(argc, argv, 2,
                                  {"input", "model", "algos", "seeds", "beta", "rank", "ranks", "inner", "max-iters",
                                   "eps", "out", "precision"},
                                  {}));
        std::cerr << "error: unknown subcommand: " << cmd << "\n" << kUsage;
        return 1;
    } catch (const Usage& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    } catch (const ntf::NumericalError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    } catch (const ntf::FormatError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 3;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
