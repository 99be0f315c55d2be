/*
 * ntfg.h -- C ABI of the B200 beta-divergence MU engine (libntfg.so).
 *
 * This is the drop-in boundary: plain pointers, sizes and status codes, no
 * C++ or torch types.  Each entry point replaces one reference interface of
 * /root/reference/proj (cited per function).  The C++ drop-in API
 * (include/ntf/ntf.hpp, namespace ntf) is a thin layer over these calls; the
 * Python package binds them with ctypes.
 *
 * Conventions
 *  - Tensors are row-major (last index fastest) with uint64 dims, as the
 *    reference DenseTensor (include/ntf/tensor.hpp:20-53).
 *  - CP factors are passed as ONE host fp64 buffer: the row-major I_n x R
 *    blocks concatenated in mode order (reference CpFactors, cp.hpp:13-22).
 *  - Tucker: core row-major (J_0..J_{N-1}) plus concatenated I_n x J_n
 *    factor blocks (reference TuckerModel, tucker.hpp:14-24).
 *  - No exception crosses this boundary; failures return a status and
 *    ntfg_last_error() holds the message (thread-local).
 */
#ifndef NTFG_H_
#define NTFG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NTFG_ABI_VERSION 1

/* Status codes; the C++ layer maps them onto the reference exception
 * hierarchy (include/ntf/errors.hpp:10-43). */
typedef enum ntfg_status {
  NTFG_OK = 0,
  NTFG_ERR_SHAPE = 1,     /* ntf::ShapeError     */
  NTFG_ERR_DOMAIN = 2,    /* ntf::DomainError    */
  NTFG_ERR_NUMERICAL = 3, /* ntf::NumericalError */
  NTFG_ERR_FORMAT = 4,    /* ntf::FormatError    */
  NTFG_ERR_CUDA = 5,
  NTFG_ERR_COMM = 6,
  NTFG_ERR_OOM = 7,
  NTFG_ERR_INTERNAL = 8
} ntfg_status;

typedef enum ntfg_precision { NTFG_F64 = 0, NTFG_F32 = 1 } ntfg_precision;
typedef enum ntfg_algo { NTFG_BCOMM = 0, NTFG_JCOMM = 1 } ntfg_algo;
typedef enum ntfg_location { NTFG_HOST = 0, NTFG_DEVICE = 1 } ntfg_location;

typedef struct ntfg_context ntfg_context;

/* Optional collective hook for data-parallel (mode-0 slab) fits: sums
 * `count` doubles at `device_buf` across ranks, in place, ordered on
 * `cuda_stream`.  Return 0 on success. */
typedef int (*ntfg_allreduce_fn)(void* user, double* device_buf, size_t count, void* cuda_stream);

/* Mirrors ntf::FitConfig (reference include/ntf/config.hpp:24-39) plus the
 * device options the north star adds as NEW fields (precision, graphs). */
typedef struct ntfg_fit_config {
  double beta;
  uint64_t rank;          /* CP rank */
  const uint64_t* ranks;  /* Tucker core shape (n_ranks entries) */
  uint32_t n_ranks;
  double eps;
  uint64_t inner_steps;
  uint64_t max_iters;
  double tol;
  uint64_t seed;
  int32_t extrapolate;
  double extrap_cap;
  double extrap_delta;
  int32_t has_data_floor;
  double data_floor;
  int32_t precision;      /* ntfg_precision: streaming type (fp64 validation / fp32) */
  int32_t use_graphs;     /* capture the outer iteration in a CUDA graph */
} ntfg_fit_config;

/* reference TraceRecord (config.hpp:18-22) */
typedef struct ntfg_trace_row {
  uint64_t iter;
  double time_s;
  double loss;
} ntfg_trace_row;

/* Data-parallel slab placement of this rank's X: rows [slab_begin,
 * slab_begin + dims[0]) of a tensor whose mode-0 extent is global_dim0. */
typedef struct ntfg_shard {
  uint64_t global_dim0;
  uint64_t slab_begin;
} ntfg_shard;

typedef struct ntfg_stats {
  uint64_t kernel_launches;   /* kernels enqueued by the last call (graph nodes counted per replay) */
  uint64_t graph_launches;
  double device_ms;           /* device time of the last fit's timed steps (CUDA events) */
  /* per-kernel-class device time, filled only when profiling is enabled
   * (eager launches bracketed by CUDA events on the context stream) */
  double recon_ms;            /* K2/K5 reconstruction + weights (+objective) passes */
  uint64_t recon_launches;
  double contract_ms;         /* K3 contraction passes */
  uint64_t contract_launches;
  double other_ms;            /* finalize / small kernels */
  uint64_t other_launches;
} ntfg_stats;

/* ---- context ------------------------------------------------------------- */
int ntfg_abi_version(void);
const char* ntfg_last_error(void);
ntfg_status ntfg_context_create(int device, ntfg_context** out);
ntfg_status ntfg_context_destroy(ntfg_context* ctx);
ntfg_status ntfg_context_set_stream(ntfg_context* ctx, void* cuda_stream);
ntfg_status ntfg_context_set_allreduce(ntfg_context* ctx, ntfg_allreduce_fn fn, void* user);
ntfg_status ntfg_context_stats(const ntfg_context* ctx, ntfg_stats* out);
/* Per-kernel-class event timing for subsequent calls (disables graphs). */
ntfg_status ntfg_context_set_profiling(ntfg_context* ctx, int enabled);
/* Device buffer (>= capacity doubles) that allreduce payloads are staged
 * through, so the hook always sees the same caller-owned buffer. */
ntfg_status ntfg_context_set_comm_buffer(ntfg_context* ctx, double* device_buf, size_t capacity);
/* Release cached device buffers. */
ntfg_status ntfg_context_trim(ntfg_context* ctx);
/* Native data-parallel communicator (new; SURVEY.md 8(e) -- the reference is
 * single-process, so there is no reference interface to replace).  Rank 0
 * creates a 128-byte id (ncclGetUniqueId), the caller broadcasts it, then
 * every rank attaches it to its context (ncclCommInitRank on ctx's device).
 * Sharded fits then allreduce their packed fp64 partials with ncclAllReduce on
 * the context stream, inside the captured outer-iteration CUDA graph, and the
 * allreduce hook is not used.  libnccl.so.2 is resolved at run time. */
ntfg_status ntfg_nccl_unique_id(void* id_out);
ntfg_status ntfg_context_init_nccl(ntfg_context* ctx, const void* id, int32_t nranks, int32_t rank);

/* validate_fit_config (reference config.hpp:43, config.cpp:7-18) */
ntfg_status ntfg_validate_fit_config(const ntfg_fit_config* cfg);

/* ---- fit drivers ------------------------------------------------------------
 * x: `order` dims, dtype 0 = fp64, 1 = fp32, on host or device (location).
 * trace: capacity max_iters + 1 rows; *trace_len receives the row count.
 * shard: NULL for a single-device fit. */

/* bcomm_fit / jcomm_fit (reference cp.hpp:48,76; cp.cpp:244-298) */
ntfg_status ntfg_cp_fit(ntfg_context* ctx, const ntfg_fit_config* cfg, int32_t algo,
                        uint32_t order, const uint64_t* dims, const void* x, int32_t x_dtype,
                        int32_t x_location, const ntfg_shard* shard, double* factors_inout,
                        ntfg_trace_row* trace, uint64_t* trace_len);

/* Sparse COO CP fit at beta = 1 (new; the reference densifies COO input in
 * read_coo, io.cpp:87-142, and runs bcomm_fit / jcomm_fit, cp.hpp:48,76).
 * indices: [nnz][order] int32 row-major, 0-based; values: nnz fp32/fp64;
 * duplicates accumulate in input order (io.cpp:138).  Same results as the
 * dense fit of the densified tensor up to summation order. */
ntfg_status ntfg_cp_fit_coo(ntfg_context* ctx, const ntfg_fit_config* cfg, int32_t algo,
                            uint32_t order, const uint64_t* dims, uint64_t nnz,
                            const int32_t* indices, const void* values, int32_t values_dtype,
                            int32_t location, const ntfg_shard* shard, double* factors_inout,
                            ntfg_trace_row* trace, uint64_t* trace_len);
/* Data-parallel sparse fits (shard != NULL): the nonzeros are
 * partitioned by mode-0 index ranges; each rank passes the nonzeros of its
 * slab with i_0 rebased to the slab (dims[0] = slab rows) and its A_0 rows,
 * exactly like a dense slab.  Mode-0 numerators stay local; modes >= 1, the
 * mode-0 column sums and the objective's nonzero part are allreduced. */

/* MU-unfold baseline (reference unfold.hpp:35-37, unfold.cpp:109-135,187-197):
 * explicit Khatri-Rao + unfolding + cuBLAS GEMMs; the comparison path for the
 * contraction engine (acceptance criterion 2 pins sweep == bcomm_sweep). */
ntfg_status ntfg_cp_mu_unfold_fit(ntfg_context* ctx, const ntfg_fit_config* cfg, uint32_t order,
                                  const uint64_t* dims, const void* x, int32_t x_dtype, int32_t x_location,
                                  double* factors_inout, ntfg_trace_row* trace, uint64_t* trace_len);
ntfg_status ntfg_cp_mu_unfold_sweep(ntfg_context* ctx, int32_t precision, double beta, double eps,
                                    uint32_t order, const uint64_t* dims, const double* x, uint64_t rank,
                                    double* factors_inout);
/* mu_unfold_tucker_fit / mu_unfold_tucker_sweep (reference unfold.hpp:39-42,
 * unfold.cpp:137-185,199-209): core then factors ascending, every mode product
 * through an explicit unfolding + cuBLAS GEMM + refold. Core ranks from
 * cfg->ranks (fit) / ranks (sweep). */
ntfg_status ntfg_tucker_mu_unfold_fit(ntfg_context* ctx, const ntfg_fit_config* cfg, uint32_t order,
                                      const uint64_t* dims, const void* x, int32_t x_dtype, int32_t x_location,
                                      double* core_inout, double* factors_inout, ntfg_trace_row* trace,
                                      uint64_t* trace_len);
ntfg_status ntfg_tucker_mu_unfold_sweep(ntfg_context* ctx, int32_t precision, double beta, double eps,
                                        uint32_t order, const uint64_t* dims, const uint64_t* ranks,
                                        const double* x, double* core_inout, double* factors_inout);

/* ---- data ingestion and generation (reference io.hpp / io.cpp) ---------------
 * ctx may be NULL for host-only calls (location NTFG_HOST). */

/* CTF1 header (read_tensor io.cpp:46-77 checks): order and dims (capacity
 * dims_capacity); max_entries = 0 disables the entry budget (kDefaultEntryBudget
 * io.hpp:19 is 2^27). */
ntfg_status ntfg_ctf1_header(const char* path, uint32_t* order, uint64_t* dims, uint32_t dims_capacity,
                             uint64_t max_entries);
/* CTF1 payload into dst (fp64 -> x_dtype), host or device; device reads stream
 * through pinned staging without a full host copy. */
ntfg_status ntfg_ctf1_read(ntfg_context* ctx, const char* path, void* dst, int32_t dtype, int32_t location,
                           uint64_t max_entries);
/* write_tensor (io.cpp:30-44): byte-exact CTF1 from a host or device tensor. */
ntfg_status ntfg_ctf1_write(ntfg_context* ctx, const char* path, uint32_t order, const uint64_t* dims,
                            const void* src, int32_t dtype, int32_t location);
/* read_coo grammar (io.cpp:87-142) as nonzeros: indices == NULL counts only
 * (nnz out); otherwise fills [nnz][order] int32 indices and fp64 values. */
ntfg_status ntfg_coo_text_read(const char* path, uint32_t* order, uint64_t* dims, uint32_t dims_capacity,
                               uint64_t* nnz, int32_t* indices, double* values, uint64_t capacity,
                               uint64_t max_entries);
/* write_trace (io.cpp:154-164): "iter,time_s,loss", %.17g. */
ntfg_status ntfg_trace_write(const char* path, const ntfg_trace_row* rows, uint64_t n);
/* Counter-based generator (new): Philox4x32-10 keyed by (seed, stream),
 * uniform #j = (word >> 11) * 2^-53.  Streams: 1 truth factors, 2 init, 3 noise. */
ntfg_status ntfg_philox_uniforms(uint64_t seed, uint64_t stream, uint64_t offset, uint64_t n, double* out);
/* CP factors from the generator: which = 0 truth (U clamped to eps), 1 init (0.1 + U). */
ntfg_status ntfg_cp_factors_generate(uint32_t order, const uint64_t* dims, uint64_t rank, uint64_t seed,
                                     int32_t which, double eps, double* out);
/* X = [[truth]] * Gamma(gamma_k, gamma_theta) for mode-0 rows [row0, row1),
 * generated in place on the device (BASELINE C2/C5 data). */
ntfg_status ntfg_generate_cp_gamma(ntfg_context* ctx, uint32_t order, const uint64_t* dims, uint64_t rank,
                                   uint64_t seed, uint32_t gamma_k, double gamma_theta, uint64_t row0,
                                   uint64_t row1, void* x_device, int32_t dtype);

/* tucker_bcomm_fit / tucker_jcomm_fit (reference tucker.hpp:55,84; tucker.cpp:221-275) */
ntfg_status ntfg_tucker_fit(ntfg_context* ctx, const ntfg_fit_config* cfg, int32_t algo,
                            uint32_t order, const uint64_t* dims, const void* x, int32_t x_dtype,
                            int32_t x_location, const ntfg_shard* shard, double* core_inout,
                            double* factors_inout, ntfg_trace_row* trace, uint64_t* trace_len);

/* ---- CP step level (host fp64 buffers; device round trip per call) ------------ */

/* cp_reconstruct (reference cp.hpp:30, cp.cpp:26-76) */
ntfg_status ntfg_cp_reconstruct(ntfg_context* ctx, int32_t precision, uint32_t order,
                                const uint64_t* dims, uint64_t rank, const double* factors,
                                double* out);
/* cp_contract (reference tensor.hpp:105, tensor.cpp:372-406) */
ntfg_status ntfg_cp_contract(ntfg_context* ctx, int32_t precision, uint32_t order,
                             const uint64_t* dims, const double* t, uint64_t rank,
                             const double* factors, uint32_t mode, double* out);
/* D_beta_mean(x, cp_reconstruct(f)) fused (reference cp.cpp:264,293) */
ntfg_status ntfg_cp_objective(ntfg_context* ctx, int32_t precision, double beta, uint32_t order,
                              const uint64_t* dims, const double* x, uint64_t rank,
                              const double* factors, double* mean_out);
/* cp_block_update_anchored / bcomm_block_update (reference cp.hpp:37-45, cp.cpp:109-129);
 * anchor NULL => bcomm_block_update.  Updates block `mode` of factors_inout. */
ntfg_status ntfg_cp_block_update(ntfg_context* ctx, int32_t precision, double beta, double eps,
                                 uint32_t order, const uint64_t* dims, const double* x,
                                 uint64_t rank, double* factors_inout, uint32_t mode,
                                 const double* anchor);
/* bcomm_sweep (reference cp.hpp:47, cp.cpp:131-135) */
ntfg_status ntfg_cp_bcomm_sweep(ntfg_context* ctx, int32_t precision, double beta, double eps,
                                uint32_t order, const uint64_t* dims, const double* x,
                                uint64_t rank, double* factors_inout);
/* make_jcomm_reference (reference cp.hpp:61, cp.cpp:202-208): host P~, Q~ out */
ntfg_status ntfg_cp_jcomm_reference(ntfg_context* ctx, int32_t precision, double beta,
                                    double eps, uint32_t order, const uint64_t* dims,
                                    const double* x, uint64_t rank, const double* factors,
                                    double* p_out, double* q_out);
/* jcomm_inner_update (reference cp.hpp:68, cp.cpp:210-229) from cached host P~, Q~ */
ntfg_status ntfg_cp_jcomm_inner_update(ntfg_context* ctx, int32_t precision, double beta,
                                       double eps, uint32_t order, const uint64_t* dims,
                                       const double* p, const double* q, uint64_t rank,
                                       const double* ref_factors, double* current_inout,
                                       uint32_t mode);
/* jcomm_outer_step (reference cp.hpp:73, cp.cpp:231-240) */
ntfg_status ntfg_cp_jcomm_outer_step(ntfg_context* ctx, int32_t precision, double beta,
                                     double eps, uint64_t inner_steps, uint32_t order,
                                     const uint64_t* dims, const double* x, uint64_t rank,
                                     double* factors_inout);

/* ---- divergence on explicit arrays ---------------------------------------------- */
/* D_beta (reference divergence.hpp:30, divergence.cpp:35-40) */
ntfg_status ntfg_D_beta(ntfg_context* ctx, double beta, uint64_t n, const double* x,
                        const double* xhat, double* out);

/* ---- Tucker step level -------------------------------------------------------------- */
/* tucker_reconstruct (reference tensor.hpp:109, tensor.cpp:408-419) */
ntfg_status ntfg_tucker_reconstruct(ntfg_context* ctx, int32_t precision, uint32_t order,
                                    const uint64_t* dims, const uint64_t* ranks,
                                    const double* core, const double* factors, double* out);
/* tucker_multimode_contract (reference tensor.hpp:116, tensor.cpp:421-456);
 * cols[n] = factor n column count; skip < 0 => none */
ntfg_status ntfg_tucker_multimode_contract(ntfg_context* ctx, int32_t precision, uint32_t order,
                                           const uint64_t* dims, const double* t,
                                           const uint64_t* cols, const double* factors,
                                           int32_t skip, double* out);
/* tucker_factor_contract (reference tensor.hpp:128, tensor.cpp:514-560) */
ntfg_status ntfg_tucker_factor_contract(ntfg_context* ctx, int32_t precision, uint32_t order,
                                        const uint64_t* dims, const double* t,
                                        const uint64_t* ranks, const double* core,
                                        const double* factors, uint32_t mode, double* out);
/* D_beta_mean(x, tucker_reconstruct(m)) (reference tucker.cpp:242,270) */
ntfg_status ntfg_tucker_objective(ntfg_context* ctx, int32_t precision, double beta,
                                  uint32_t order, const uint64_t* dims, const double* x,
                                  const uint64_t* ranks, const double* core,
                                  const double* factors, double* mean_out);
/* Tucker step kinds (reference tucker.hpp:38-82):
 *  0 block_core_update, 1 block_factor_update(mode), 2 tucker_bcomm_sweep,
 *  3 jcomm_tucker_outer_step(inner_steps),
 *  4 jcomm_inner_core_update and 5 jcomm_inner_factor_update(mode) against the
 *    reference model (ref_core, ref_factors) whose P~/Q~ are built from x,
 *  6 block_core_update_anchored (anchor core in ref_core),
 *  7 block_factor_update_anchored(mode) (anchor I_mode x J_mode block in ref_factors). */
ntfg_status ntfg_tucker_step(ntfg_context* ctx, int32_t precision, int32_t kind, double beta,
                             double eps, uint64_t inner_steps, uint32_t order,
                             const uint64_t* dims, const double* x, const uint64_t* ranks,
                             const double* ref_core, const double* ref_factors,
                             double* core_inout, double* factors_inout, uint32_t mode);

/* make_jcomm_tucker_reference (reference tucker.hpp:59-67, tucker.cpp:92-98):
 * P~ and Q~ (E fp64 each, host) of the reference model (ref_core, ref_factors). */
ntfg_status ntfg_tucker_jcomm_reference(ntfg_context* ctx, int32_t precision, double beta, double eps,
                                        uint32_t order, const uint64_t* dims, const double* x,
                                        const uint64_t* ranks, const double* ref_core,
                                        const double* ref_factors, double* p_out, double* q_out);
/* jcomm_inner_core_update (block = -1) / jcomm_inner_factor_update (block =
 * mode) from the cached host P~/Q~ (reference tucker.hpp:69-78,
 * tucker.cpp:100-149): current model in/out, anchored at the reference. */
ntfg_status ntfg_tucker_jcomm_inner_update(ntfg_context* ctx, int32_t precision, double beta, double eps,
                                           uint32_t order, const uint64_t* dims, const double* p,
                                           const double* q, const uint64_t* ranks, const double* ref_core,
                                           const double* ref_factors, double* core_inout,
                                           double* factors_inout, int32_t block);

#ifdef __cplusplus
}
#endif
#endif /* NTFG_H_ */
