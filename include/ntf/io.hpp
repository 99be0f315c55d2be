// Drop-in for reference include/ntf/io.hpp (io.cpp): CTF1 / coordinate-text
// ingestion, trace CSV, and the seeded generators.  The CTF1, COO and trace
// paths go through the C ABI (ntfg_ctf1_*, ntfg_coo_text_read,
// ntfg_trace_write; byte-exact with the reference's files); Rng is the same
// standard-specified engine (std::mt19937_64 seeded through std::seed_seq),
// so init_cp_factors / synth_cp draw exactly the reference's values.
#pragma once

#include <cstdint>
#include <optional>
#include <random>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "ntf/ntf.hpp"

namespace ntf {

inline constexpr std::size_t kDefaultEntryBudget = std::size_t{1} << 27;  // io.hpp:19

void write_tensor(const std::string& path, const DenseTensor& t);                    // io.cpp:30-44
DenseTensor read_tensor(const std::string& path, std::size_t max_entries = kDefaultEntryBudget);  // io.cpp:46-77
DenseTensor read_coo(const std::string& path, std::optional<double> floor = std::nullopt,
                     std::size_t max_entries = kDefaultEntryBudget);                  // io.cpp:87-142
DenseTensor read_tensor_auto(const std::string& path, std::size_t max_entries = kDefaultEntryBudget);  // io.cpp:144-152
void write_trace(const std::string& path, std::span<const TraceRecord> records);    // io.cpp:154-164
std::vector<TraceRecord> read_trace(const std::string& path);

// X <- max(X, s) entrywise (reference tensor.hpp:105)
DenseTensor cwise_max(const DenseTensor& a, double s);

class Rng {  // io.hpp:45-62, io.cpp:190-200
public:
    static constexpr std::uint64_t kSynthStream = 1;
    static constexpr std::uint64_t kInitStream = 2;
    static constexpr std::uint64_t kDataStream = 3;
    Rng(std::uint64_t seed, std::uint64_t stream);
    double uniform01();

private:
    std::mt19937_64 engine_;
};

CpFactors random_cp_factors(std::span<const std::size_t> dims, std::size_t rank, Rng& rng, double eps);
TuckerModel random_tucker_model(std::span<const std::size_t> dims, std::span<const std::size_t> ranks, Rng& rng,
                                double eps);
CpFactors init_cp_factors(std::span<const std::size_t> dims, std::size_t rank, std::uint64_t seed, double eps);
TuckerModel init_tucker_model(std::span<const std::size_t> dims, std::span<const std::size_t> ranks,
                              std::uint64_t seed, double eps);
std::pair<DenseTensor, CpFactors> synth_cp(std::span<const std::size_t> dims, std::size_t rank, std::uint64_t seed,
                                           double eps = 1e-12);
std::pair<DenseTensor, TuckerModel> synth_tucker(std::span<const std::size_t> dims,
                                                 std::span<const std::size_t> ranks, std::uint64_t seed,
                                                 double eps = 1e-12);

}  // namespace ntf
