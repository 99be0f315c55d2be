// extern "C" boundary of libntfg.so (declared in include/ntfg.h).  Converts
// internal exceptions into status codes + a thread-local message; no C++
// exception crosses this boundary.
#include <cstdio>
#include <cstring>
#include <string>

#include "engine.cuh"
#include "nccl_comm.cuh"

namespace ntfg {
// cp_api.cu
void cp_fit(Context&, const ntfg_fit_config&, int, uint32_t, const uint64_t*, const void*, int, int,
            const ntfg_shard*, double*, ntfg_trace_row*, uint64_t*);
void cp_fit_coo(Context&, const ntfg_fit_config&, int, uint32_t, const uint64_t*, uint64_t, const int32_t*,
                const void*, int, int, const ntfg_shard*, double*, ntfg_trace_row*, uint64_t*);
void cp_reconstruct(Context&, int, uint32_t, const uint64_t*, uint64_t, const double*, double*);
// unfold_api.cu
void cp_mu_unfold_fit(Context&, const ntfg_fit_config&, uint32_t, const uint64_t*, const void*, int, int, double*,
                      ntfg_trace_row*, uint64_t*);
void cp_mu_unfold_sweep(Context&, int, double, double, uint32_t, const uint64_t*, const double*, uint64_t, double*);
void tucker_mu_unfold_fit(Context&, const ntfg_fit_config&, uint32_t, const uint64_t*, const void*, int, int, double*,
                          double*, ntfg_trace_row*, uint64_t*);
void tucker_mu_unfold_sweep(Context&, int, double, double, uint32_t, const uint64_t*, const uint64_t*, const double*,
                            double*, double*);
// io_api.cu
void ctf1_header_api(const char*, uint32_t*, uint64_t*, uint32_t, uint64_t);
void ctf1_read(Context*, const char*, void*, int, int, uint64_t);
void ctf1_write(Context*, const char*, uint32_t, const uint64_t*, const void*, int, int);
void coo_text_read(const char*, uint32_t*, uint64_t*, uint32_t, uint64_t*, int32_t*, double*, uint64_t, uint64_t);
void trace_write(const char*, const ntfg_trace_row*, uint64_t);
void philox_uniforms(uint64_t, uint64_t, uint64_t, uint64_t, double*);
void cp_factors_philox(uint32_t, const uint64_t*, uint64_t, uint64_t, int, double, double*);
void generate_cp_gamma(Context&, uint32_t, const uint64_t*, uint64_t, uint64_t, uint32_t, double, uint64_t,
                       uint64_t, void*, int);
void cp_contract(Context&, int, uint32_t, const uint64_t*, const double*, uint64_t, const double*,
                 uint32_t, double*);
void cp_objective(Context&, int, double, uint32_t, const uint64_t*, const double*, uint64_t,
                  const double*, double*);
void cp_block_update(Context&, int, double, double, uint32_t, const uint64_t*, const double*,
                     uint64_t, double*, uint32_t, const double*);
void cp_bcomm_sweep(Context&, int, double, double, uint32_t, const uint64_t*, const double*,
                    uint64_t, double*);
void cp_jcomm_reference(Context&, int, double, double, uint32_t, const uint64_t*, const double*,
                        uint64_t, const double*, double*, double*);
void cp_jcomm_inner_update(Context&, int, double, double, uint32_t, const uint64_t*, const double*,
                           const double*, uint64_t, const double*, double*, uint32_t);
void cp_jcomm_outer_step(Context&, int, double, double, uint64_t, uint32_t, const uint64_t*,
                         const double*, uint64_t, double*);
void D_beta(Context&, double, uint64_t, const double*, const double*, double*);
// tucker_api.cu
void tucker_fit(Context&, const ntfg_fit_config&, int, uint32_t, const uint64_t*, const void*, int,
                int, const ntfg_shard*, double*, double*, ntfg_trace_row*, uint64_t*);
void tucker_reconstruct(Context&, int, uint32_t, const uint64_t*, const uint64_t*, const double*,
                        const double*, double*);
void tucker_multimode_contract(Context&, int, uint32_t, const uint64_t*, const double*,
                               const uint64_t*, const double*, int32_t, double*);
void tucker_factor_contract(Context&, int, uint32_t, const uint64_t*, const double*,
                            const uint64_t*, const double*, const double*, uint32_t, double*);
void tucker_objective(Context&, int, double, uint32_t, const uint64_t*, const double*,
                      const uint64_t*, const double*, const double*, double*);
void tucker_jcomm_reference(Context&, int, double, double, uint32_t, const uint64_t*, const double*,
                            const uint64_t*, const double*, const double*, double*, double*);
void tucker_jcomm_inner_update(Context&, int, double, double, uint32_t, const uint64_t*, const double*,
                               const double*, const uint64_t*, const double*, const double*, double*, double*,
                               int32_t);
void tucker_step(Context&, int, int, double, double, uint64_t, uint32_t, const uint64_t*,
                 const double*, const uint64_t*, const double*, const double*, double*, double*,
                 uint32_t);
}  // namespace ntfg

struct ntfg_context : ntfg::Context {};

namespace {
// Thread-local last-error text in a trivially destructible buffer: callers may
// reach the C ABI from their own thread_local destructors at thread exit (the
// drop-in's per-thread context does), after a std::string here would already
// have been destroyed.
struct LastError {
  char text[512];
  void clear() { text[0] = '\0'; }
  LastError& operator=(const char* s) {
    std::strncpy(text, s ? s : "", sizeof(text) - 1);
    text[sizeof(text) - 1] = '\0';
    return *this;
  }
  const char* c_str() const { return text; }
};
thread_local LastError g_last_error = {{0}};

template <class F>
ntfg_status guard(F&& f) {
  try {
    f();
    g_last_error.clear();
    return NTFG_OK;
  } catch (const ntfg::Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return NTFG_ERR_OOM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return NTFG_ERR_INTERNAL;
  }
}

template <class F>
ntfg_status with_ctx(ntfg_context* ctx, F&& f) {
  if (!ctx) {
    g_last_error = "null context";
    return NTFG_ERR_INTERNAL;
  }
  return guard([&] {
    ctx->activate();
    f(*ctx);
  });
}

void need(const void* p, const char* what) {
  if (!p) throw ntfg::Error(NTFG_ERR_SHAPE, std::string(what) + " must not be NULL");
}
}  // namespace

#define NTFG_API extern "C" __attribute__((visibility("default")))

NTFG_API int ntfg_abi_version(void) { return NTFG_ABI_VERSION; }
NTFG_API const char* ntfg_last_error(void) { return g_last_error.c_str(); }

NTFG_API ntfg_status ntfg_context_create(int device, ntfg_context** out) {
  return guard([&] {
    need(out, "out");
    int n = 0;
    ntfg::cuda_check(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
    if (device < 0 || device >= n) throw ntfg::Error(NTFG_ERR_CUDA, "no such CUDA device");
    auto* c = new ntfg_context();
    c->device = device;
    try {
      c->activate();
      ntfg::cuda_check(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
      c->own_stream = true;
      cudaDeviceProp prop;
      ntfg::cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
      c->sm_count = prop.multiProcessorCount;
      if (prop.major < 10)
        throw ntfg::Error(NTFG_ERR_CUDA, "libntfg is built for sm_100a (B200); device is sm_" +
                                             std::to_string(prop.major) + std::to_string(prop.minor));
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

NTFG_API ntfg_status ntfg_context_destroy(ntfg_context* ctx) {
  if (!ctx) return NTFG_OK;
  return guard([&] {
    ctx->activate();
    cudaStreamSynchronize(ctx->stream);
    ctx->bufs.release();
    if (ctx->nccl) ntfg::nccl_comm_destroy(ctx->nccl);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

NTFG_API ntfg_status ntfg_context_set_stream(ntfg_context* ctx, void* stream) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    if (c.own_stream) cudaStreamDestroy(c.stream);
    c.stream = static_cast<cudaStream_t>(stream);
    c.own_stream = false;
  });
}

NTFG_API ntfg_status ntfg_context_set_allreduce(ntfg_context* ctx, ntfg_allreduce_fn fn, void* user) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    c.allreduce = fn;
    c.allreduce_user = user;
  });
}

NTFG_API ntfg_status ntfg_context_stats(const ntfg_context* ctx, ntfg_stats* out) {
  if (!ctx || !out) return NTFG_ERR_INTERNAL;
  *out = ctx->stats;
  return NTFG_OK;
}

NTFG_API ntfg_status ntfg_context_set_profiling(ntfg_context* ctx, int enabled) {
  return with_ctx(ctx, [&](ntfg::Context& c) { c.profile = enabled != 0; });
}

NTFG_API ntfg_status ntfg_context_set_comm_buffer(ntfg_context* ctx, double* buf, size_t cap) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    c.comm_buf = buf;
    c.comm_cap = buf ? cap : 0;
  });
}

NTFG_API ntfg_status ntfg_nccl_unique_id(void* id_out) {
  return guard([&] {
    need(id_out, "id_out");
    ntfg::nccl_unique_id(id_out);
  });
}

NTFG_API ntfg_status ntfg_context_init_nccl(ntfg_context* ctx, const void* id, int32_t nranks, int32_t rank) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(id, "id");
    if (nranks < 1 || rank < 0 || rank >= nranks) throw ntfg::Error(NTFG_ERR_DOMAIN, "invalid nranks/rank");
    if (c.nccl) {
      ntfg::nccl_comm_destroy(c.nccl);
      c.nccl = nullptr;
    }
    c.nccl = ntfg::nccl_comm_init(id, nranks, rank);
    c.nccl_ranks = nranks;
  });
}

NTFG_API ntfg_status ntfg_context_trim(ntfg_context* ctx) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    c.sync();
    c.bufs.release();
  });
}

NTFG_API ntfg_status ntfg_validate_fit_config(const ntfg_fit_config* cfg) {
  return guard([&] {
    need(cfg, "cfg");
    ntfg::validate_config(*cfg);
  });
}

NTFG_API ntfg_status ntfg_cp_fit(ntfg_context* ctx, const ntfg_fit_config* cfg, int32_t algo,
                                 uint32_t order, const uint64_t* dims, const void* x,
                                 int32_t x_dtype, int32_t x_location, const ntfg_shard* shard,
                                 double* factors, ntfg_trace_row* trace, uint64_t* trace_len) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(cfg, "cfg"); need(dims, "dims"); need(x, "x"); need(factors, "factors");
    need(trace, "trace"); need(trace_len, "trace_len");
    ntfg::cp_fit(c, *cfg, algo, order, dims, x, x_dtype, x_location, shard, factors, trace, trace_len);
  });
}

NTFG_API ntfg_status ntfg_cp_fit_coo(ntfg_context* ctx, const ntfg_fit_config* cfg, int32_t algo,
                                     uint32_t order, const uint64_t* dims, uint64_t nnz,
                                     const int32_t* indices, const void* values, int32_t values_dtype,
                                     int32_t location, const ntfg_shard* shard, double* factors,
                                     ntfg_trace_row* trace, uint64_t* trace_len) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(cfg, "cfg"); need(dims, "dims"); need(factors, "factors");
    need(trace, "trace"); need(trace_len, "trace_len");
    if (nnz > 0) { need(indices, "indices"); need(values, "values"); }
    ntfg::cp_fit_coo(c, *cfg, algo, order, dims, nnz, indices, values, values_dtype, location, shard, factors,
                     trace, trace_len);
  });
}

NTFG_API ntfg_status ntfg_cp_mu_unfold_fit(ntfg_context* ctx, const ntfg_fit_config* cfg, uint32_t order,
                                           const uint64_t* dims, const void* x, int32_t x_dtype, int32_t x_location,
                                           double* factors, ntfg_trace_row* trace, uint64_t* trace_len) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(cfg, "cfg"); need(dims, "dims"); need(x, "x"); need(factors, "factors");
    need(trace, "trace"); need(trace_len, "trace_len");
    ntfg::cp_mu_unfold_fit(c, *cfg, order, dims, x, x_dtype, x_location, factors, trace, trace_len);
  });
}

NTFG_API ntfg_status ntfg_cp_mu_unfold_sweep(ntfg_context* ctx, int32_t precision, double beta, double eps,
                                             uint32_t order, const uint64_t* dims, const double* x, uint64_t rank,
                                             double* factors) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(dims, "dims"); need(x, "x"); need(factors, "factors");
    ntfg::cp_mu_unfold_sweep(c, precision, beta, eps, order, dims, x, rank, factors);
  });
}

NTFG_API ntfg_status ntfg_tucker_mu_unfold_fit(ntfg_context* ctx, const ntfg_fit_config* cfg, uint32_t order,
                                               const uint64_t* dims, const void* x, int32_t x_dtype,
                                               int32_t x_location, double* core, double* factors,
                                               ntfg_trace_row* trace, uint64_t* trace_len) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(cfg, "cfg"); need(dims, "dims"); need(x, "x"); need(core, "core"); need(factors, "factors");
    need(trace, "trace"); need(trace_len, "trace_len");
    ntfg::tucker_mu_unfold_fit(c, *cfg, order, dims, x, x_dtype, x_location, core, factors, trace, trace_len);
  });
}

NTFG_API ntfg_status ntfg_tucker_mu_unfold_sweep(ntfg_context* ctx, int32_t precision, double beta, double eps,
                                                 uint32_t order, const uint64_t* dims, const uint64_t* ranks,
                                                 const double* x, double* core, double* factors) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(dims, "dims"); need(ranks, "ranks"); need(x, "x"); need(core, "core"); need(factors, "factors");
    ntfg::tucker_mu_unfold_sweep(c, precision, beta, eps, order, dims, ranks, x, core, factors);
  });
}

// ---- io / generators ----------------------------------------------------------------
NTFG_API ntfg_status ntfg_ctf1_header(const char* path, uint32_t* order, uint64_t* dims, uint32_t cap,
                                      uint64_t max_entries) {
  return guard([&] {
    need(path, "path"); need(order, "order");
    ntfg::ctf1_header_api(path, order, dims, cap, max_entries);
  });
}

NTFG_API ntfg_status ntfg_ctf1_read(ntfg_context* ctx, const char* path, void* dst, int32_t dtype,
                                    int32_t location, uint64_t max_entries) {
  return guard([&] {
    need(path, "path"); need(dst, "dst");
    if (ctx) ctx->activate();
    ntfg::ctf1_read(ctx, path, dst, dtype, location, max_entries);
  });
}

NTFG_API ntfg_status ntfg_ctf1_write(ntfg_context* ctx, const char* path, uint32_t order, const uint64_t* dims,
                                     const void* src, int32_t dtype, int32_t location) {
  return guard([&] {
    need(path, "path"); need(dims, "dims"); need(src, "src");
    if (ctx) ctx->activate();
    ntfg::ctf1_write(ctx, path, order, dims, src, dtype, location);
  });
}

NTFG_API ntfg_status ntfg_coo_text_read(const char* path, uint32_t* order, uint64_t* dims, uint32_t cap,
                                        uint64_t* nnz, int32_t* indices, double* values, uint64_t capacity,
                                        uint64_t max_entries) {
  return guard([&] {
    need(path, "path"); need(order, "order"); need(dims, "dims"); need(nnz, "nnz");
    if (indices) need(values, "values");
    ntfg::coo_text_read(path, order, dims, cap, nnz, indices, values, capacity, max_entries);
  });
}

NTFG_API ntfg_status ntfg_trace_write(const char* path, const ntfg_trace_row* rows, uint64_t n) {
  return guard([&] {
    need(path, "path");
    if (n) need(rows, "rows");
    ntfg::trace_write(path, rows, n);
  });
}

NTFG_API ntfg_status ntfg_philox_uniforms(uint64_t seed, uint64_t stream, uint64_t offset, uint64_t n,
                                          double* out) {
  return guard([&] {
    if (n) need(out, "out");
    ntfg::philox_uniforms(seed, stream, offset, n, out);
  });
}

NTFG_API ntfg_status ntfg_cp_factors_generate(uint32_t order, const uint64_t* dims, uint64_t rank, uint64_t seed,
                                              int32_t which, double eps, double* out) {
  return guard([&] {
    need(dims, "dims"); need(out, "out");
    ntfg::cp_factors_philox(order, dims, rank, seed, which, eps, out);
  });
}

NTFG_API ntfg_status ntfg_generate_cp_gamma(ntfg_context* ctx, uint32_t order, const uint64_t* dims,
                                            uint64_t rank, uint64_t seed, uint32_t gamma_k, double gamma_theta,
                                            uint64_t row0, uint64_t row1, void* x, int32_t dtype) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(dims, "dims"); need(x, "x");
    ntfg::generate_cp_gamma(c, order, dims, rank, seed, gamma_k, gamma_theta, row0, row1, x, dtype);
  });
}

NTFG_API ntfg_status ntfg_tucker_fit(ntfg_context* ctx, const ntfg_fit_config* cfg, int32_t algo,
                                     uint32_t order, const uint64_t* dims, const void* x,
                                     int32_t x_dtype, int32_t x_location, const ntfg_shard* shard,
                                     double* core, double* factors, ntfg_trace_row* trace,
                                     uint64_t* trace_len) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(cfg, "cfg"); need(dims, "dims"); need(x, "x"); need(core, "core");
    need(factors, "factors"); need(trace, "trace"); need(trace_len, "trace_len");
    ntfg::tucker_fit(c, *cfg, algo, order, dims, x, x_dtype, x_location, shard, core, factors,
                     trace, trace_len);
  });
}

NTFG_API ntfg_status ntfg_cp_reconstruct(ntfg_context* ctx, int32_t precision, uint32_t order,
                                         const uint64_t* dims, uint64_t rank,
                                         const double* factors, double* out) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(dims, "dims"); need(factors, "factors"); need(out, "out");
    ntfg::cp_reconstruct(c, precision, order, dims, rank, factors, out);
  });
}

NTFG_API ntfg_status ntfg_cp_contract(ntfg_context* ctx, int32_t precision, uint32_t order,
                                      const uint64_t* dims, const double* t, uint64_t rank,
                                      const double* factors, uint32_t mode, double* out) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(dims, "dims"); need(t, "t"); need(factors, "factors"); need(out, "out");
    ntfg::cp_contract(c, precision, order, dims, t, rank, factors, mode, out);
  });
}

NTFG_API ntfg_status ntfg_cp_objective(ntfg_context* ctx, int32_t precision, double beta,
                                       uint32_t order, const uint64_t* dims, const double* x,
                                       uint64_t rank, const double* factors, double* mean_out) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(dims, "dims"); need(x, "x"); need(factors, "factors"); need(mean_out, "mean_out");
    ntfg::cp_objective(c, precision, beta, order, dims, x, rank, factors, mean_out);
  });
}

NTFG_API ntfg_status ntfg_cp_block_update(ntfg_context* ctx, int32_t precision, double beta,
                                          double eps, uint32_t order, const uint64_t* dims,
                                          const double* x, uint64_t rank, double* factors,
                                          uint32_t mode, const double* anchor) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(dims, "dims"); need(x, "x"); need(factors, "factors");
    ntfg::cp_block_update(c, precision, beta, eps, order, dims, x, rank, factors, mode, anchor);
  });
}

NTFG_API ntfg_status ntfg_cp_bcomm_sweep(ntfg_context* ctx, int32_t precision, double beta,
                                         double eps, uint32_t order, const uint64_t* dims,
                                         const double* x, uint64_t rank, double* factors) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(dims, "dims"); need(x, "x"); need(factors, "factors");
    ntfg::cp_bcomm_sweep(c, precision, beta, eps, order, dims, x, rank, factors);
  });
}

NTFG_API ntfg_status ntfg_cp_jcomm_reference(ntfg_context* ctx, int32_t precision, double beta,
                                             double eps, uint32_t order, const uint64_t* dims,
                                             const double* x, uint64_t rank, const double* factors,
                                             double* p_out, double* q_out) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(dims, "dims"); need(x, "x"); need(factors, "factors"); need(p_out, "p_out"); need(q_out, "q_out");
    ntfg::cp_jcomm_reference(c, precision, beta, eps, order, dims, x, rank, factors, p_out, q_out);
  });
}

NTFG_API ntfg_status ntfg_cp_jcomm_inner_update(ntfg_context* ctx, int32_t precision, double beta,
                                                double eps, uint32_t order, const uint64_t* dims,
                                                const double* p, const double* q, uint64_t rank,
                                                const double* ref, double* current, uint32_t mode) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(dims, "dims"); need(p, "p"); need(q, "q"); need(ref, "ref"); need(current, "current");
    ntfg::cp_jcomm_inner_update(c, precision, beta, eps, order, dims, p, q, rank, ref, current, mode);
  });
}

NTFG_API ntfg_status ntfg_cp_jcomm_outer_step(ntfg_context* ctx, int32_t precision, double beta,
                                              double eps, uint64_t inner_steps, uint32_t order,
                                              const uint64_t* dims, const double* x, uint64_t rank,
                                              double* factors) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(dims, "dims"); need(x, "x"); need(factors, "factors");
    ntfg::cp_jcomm_outer_step(c, precision, beta, eps, inner_steps, order, dims, x, rank, factors);
  });
}

NTFG_API ntfg_status ntfg_D_beta(ntfg_context* ctx, double beta, uint64_t n, const double* x,
                                 const double* xhat, double* out) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(out, "out");
    ntfg::D_beta(c, beta, n, x, xhat, out);
  });
}

NTFG_API ntfg_status ntfg_tucker_reconstruct(ntfg_context* ctx, int32_t precision, uint32_t order,
                                             const uint64_t* dims, const uint64_t* ranks,
                                             const double* core, const double* factors,
                                             double* out) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(dims, "dims"); need(ranks, "ranks"); need(core, "core"); need(factors, "factors"); need(out, "out");
    ntfg::tucker_reconstruct(c, precision, order, dims, ranks, core, factors, out);
  });
}

NTFG_API ntfg_status ntfg_tucker_multimode_contract(ntfg_context* ctx, int32_t precision,
                                                    uint32_t order, const uint64_t* dims,
                                                    const double* t, const uint64_t* cols,
                                                    const double* factors, int32_t skip,
                                                    double* out) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(dims, "dims"); need(t, "t"); need(cols, "cols"); need(factors, "factors"); need(out, "out");
    ntfg::tucker_multimode_contract(c, precision, order, dims, t, cols, factors, skip, out);
  });
}

NTFG_API ntfg_status ntfg_tucker_factor_contract(ntfg_context* ctx, int32_t precision,
                                                 uint32_t order, const uint64_t* dims,
                                                 const double* t, const uint64_t* ranks,
                                                 const double* core, const double* factors,
                                                 uint32_t mode, double* out) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(dims, "dims"); need(t, "t"); need(ranks, "ranks"); need(core, "core");
    need(factors, "factors"); need(out, "out");
    ntfg::tucker_factor_contract(c, precision, order, dims, t, ranks, core, factors, mode, out);
  });
}

NTFG_API ntfg_status ntfg_tucker_objective(ntfg_context* ctx, int32_t precision, double beta,
                                           uint32_t order, const uint64_t* dims, const double* x,
                                           const uint64_t* ranks, const double* core,
                                           const double* factors, double* mean_out) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(dims, "dims"); need(x, "x"); need(ranks, "ranks"); need(core, "core");
    need(factors, "factors"); need(mean_out, "mean_out");
    ntfg::tucker_objective(c, precision, beta, order, dims, x, ranks, core, factors, mean_out);
  });
}

NTFG_API ntfg_status ntfg_tucker_step(ntfg_context* ctx, int32_t precision, int32_t kind,
                                      double beta, double eps, uint64_t inner_steps,
                                      uint32_t order, const uint64_t* dims, const double* x,
                                      const uint64_t* ranks, const double* ref_core,
                                      const double* ref_factors, double* core, double* factors,
                                      uint32_t mode) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(dims, "dims"); need(x, "x"); need(ranks, "ranks"); need(core, "core"); need(factors, "factors");
    ntfg::tucker_step(c, precision, kind, beta, eps, inner_steps, order, dims, x, ranks, ref_core,
                      ref_factors, core, factors, mode);
  });
}

NTFG_API ntfg_status ntfg_tucker_jcomm_reference(ntfg_context* ctx, int32_t precision, double beta, double eps,
                                                 uint32_t order, const uint64_t* dims, const double* x,
                                                 const uint64_t* ranks, const double* ref_core,
                                                 const double* ref_factors, double* p_out, double* q_out) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(dims, "dims"); need(x, "x"); need(ranks, "ranks"); need(ref_core, "ref_core");
    need(ref_factors, "ref_factors"); need(p_out, "p_out"); need(q_out, "q_out");
    ntfg::tucker_jcomm_reference(c, precision, beta, eps, order, dims, x, ranks, ref_core, ref_factors, p_out, q_out);
  });
}

NTFG_API ntfg_status ntfg_tucker_jcomm_inner_update(ntfg_context* ctx, int32_t precision, double beta, double eps,
                                                    uint32_t order, const uint64_t* dims, const double* p,
                                                    const double* q, const uint64_t* ranks, const double* ref_core,
                                                    const double* ref_factors, double* core, double* factors,
                                                    int32_t block) {
  return with_ctx(ctx, [&](ntfg::Context& c) {
    need(dims, "dims"); need(p, "p"); need(q, "q"); need(ranks, "ranks"); need(ref_core, "ref_core");
    need(ref_factors, "ref_factors"); need(core, "core"); need(factors, "factors");
    ntfg::tucker_jcomm_inner_update(c, precision, beta, eps, order, dims, p, q, ranks, ref_core, ref_factors, core,
                                    factors, block);
  });
}
