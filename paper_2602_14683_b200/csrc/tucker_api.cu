// Tucker entry points (placeholder until the Tucker engine lands).
#include "engine.cuh"

namespace ntfg {
[[noreturn]] static void todo() { throw Error(NTFG_ERR_INTERNAL, "Tucker engine not built yet"); }
void tucker_fit(Context&, const ntfg_fit_config&, int, uint32_t, const uint64_t*, const void*, int,
                int, const ntfg_shard*, double*, double*, ntfg_trace_row*, uint64_t*) { todo(); }
void tucker_reconstruct(Context&, int, uint32_t, const uint64_t*, const uint64_t*, const double*,
                        const double*, double*) { todo(); }
void tucker_multimode_contract(Context&, int, uint32_t, const uint64_t*, const double*,
                               const uint64_t*, const double*, int32_t, double*) { todo(); }
void tucker_factor_contract(Context&, int, uint32_t, const uint64_t*, const double*,
                            const uint64_t*, const double*, const double*, uint32_t, double*) { todo(); }
void tucker_objective(Context&, int, double, uint32_t, const uint64_t*, const double*,
                      const uint64_t*, const double*, const double*, double*) { todo(); }
void tucker_step(Context&, int, int, double, double, uint64_t, uint32_t, const uint64_t*,
                 const double*, const uint64_t*, const double*, const double*, double*, double*,
                 uint32_t) { todo(); }
}  // namespace ntfg
