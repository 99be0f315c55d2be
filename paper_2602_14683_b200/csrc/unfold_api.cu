// MU-unfold baseline on the GPU: the classical
// matricized multiplicative update of reference unfold.cpp:109-135 --
// explicit Khatri-Rao product, explicit mode-n unfolding, and plain library
// GEMMs (cuBLAS) for Xhat_(n) = A_n KR^T, Num = P_(n) KR, Den = Q_(n) KR.
// It exists to reproduce the paper's contraction-vs-unfolding comparison on
// B200 (the contraction engine never materializes KR or X_(n)), and
// acceptance criterion 2 (acceptance.cpp:104-132) pins it to bcomm_sweep.
//
// Master factors stay fp64 (MU step in fp64 as everywhere else); the GEMMs
// run in T (fp64 DGEMM or fp32 SGEMM without TF32).
#include <cublas_v2.h>

#include <functional>
#include <vector>

#include "cp_engine.cuh"
#include "fit_loop.cuh"
#include "tucker_engine.cuh"

namespace ntfg {

namespace {

void cublas_check(cublasStatus_t s, const char* what) {
  if (s != CUBLAS_STATUS_SUCCESS) throw Error(NTFG_ERR_CUDA, std::string("cuBLAS failure in ") + what);
}

struct Cublas {
  cublasHandle_t h = nullptr;
  explicit Cublas(cudaStream_t s) {
    cublas_check(cublasCreate(&h), "cublasCreate");
    cublas_check(cublasSetStream(h, s), "cublasSetStream");
    cublas_check(cublasSetMathMode(h, CUBLAS_DEFAULT_MATH), "cublasSetMathMode");  // no TF32
  }
  ~Cublas() { if (h) cublasDestroy(h); }
};

// row-major C[M][N] = A[M][K] * B^T where B is row-major [N][K]   (transB)
// row-major C[M][N] = A[M][K] * B     where B is row-major [K][N] (plain)
template <typename T>
void gemm_rm(cublasHandle_t h, bool transB, int64_t M, int64_t N, int64_t K, const T* A, const T* B, T* C) {
  const T one = T(1), zero = T(0);
  // column-major view: C^T (N x M) = op(B)^T-ish * A^T
  const cublasOperation_t opB = transB ? CUBLAS_OP_T : CUBLAS_OP_N;
  const int ldb = int(transB ? K : N);
  if constexpr (sizeof(T) == 8)
    cublas_check(cublasDgemm(h, opB, CUBLAS_OP_N, int(N), int(M), int(K), &one, B, ldb, A, int(K), &zero, C, int(N)),
                 "cublasDgemm");
  else
    cublas_check(cublasSgemm(h, opB, CUBLAS_OP_N, int(N), int(M), int(K), &one, B, ldb, A, int(K), &zero, C, int(N)),
                 "cublasSgemm");
}

}  // namespace

// khatri_rao (unfold.cpp:66-88): rows ordered first matrix slowest, product
// accumulated left to right (bitwise the reference's in fp64)
template <typename T>
static __global__ void khatri_rao_kernel(int nmat, int64_t J, int R,
                                         const int64_t* rows, const double* m0, const double* m1, const double* m2,
                                         const double* m3, const double* m4, const double* m5, const double* m6,
                                         T* out) {
  const double* mats[kMaxOrder - 1] = {m0, m1, m2, m3, m4, m5, m6};
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < J * R;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = idx / R;
    const int r = int(idx % R);
    int64_t sub[kMaxOrder - 1];
    int64_t rem = j;
    for (int k = nmat - 1; k >= 0; --k) {
      sub[k] = rem % rows[k];
      rem /= rows[k];
    }
    double v = mats[0][sub[0] * R + r];
    for (int k = 1; k < nmat; ++k) v = v * mats[k][sub[k] * R + r];
    out[idx] = T(v);
  }
}

// unfold (unfold.cpp:11-36): X = [A][I][B] row-major -> X_(n)[i][a*B + b]
template <typename T>
static __global__ void unfold_kernel(const T* x, int64_t A, int64_t I, int64_t B, T* out) {
  const int64_t E = A * I * B;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < E; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = e % B;
    const int64_t t = e / B;
    const int64_t i = t % I;
    const int64_t a = t / I;
    out[i * (A * B) + a * B + b] = x[e];
  }
}

template <typename T>
static __global__ void unfolded_weights_kernel(const T* xn, T* xh_to_p, T* q, int64_t n, int bk, double beta,
                                               double eps) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    T pw, qw;
    weights_entry(xn[i], xh_to_p[i], bk, beta, eps, pw, qw);
    xh_to_p[i] = pw;
    q[i] = qw;
  }
}

// multiplicative_update (divergence.cpp:116-135) of one factor; refreshes its T copy
template <typename T>
static __global__ void unfold_mu_kernel(double* a, const T* num, const T* den, int64_t n, double gamma, double eps,
                                        T* a_t) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double v = mu_step(a[i], double(num[i]), double(den[i]), gamma, eps);
    a[i] = v;
    a_t[i] = T(v);
  }
}

template <typename T>
static __global__ void to_t_kernel(const double* src, int64_t n, T* dst) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = T(src[i]);
}

// mu_unfold_cp_sweep (unfold.cpp:109-135) over the engine's fp64 factors
template <typename T>
class UnfoldCp {
 public:
  UnfoldCp(Context& c, CpEngine<T>& e, double beta, double eps)
      : c_(c), e_(e), blas_(c.stream), beta_(beta), eps_(eps), gamma_(gamma_of(beta)), bk_(beta_kind_of(beta)) {
    N_ = e.order();
    E_ = e.entries();
    R_ = int64_t(e.factor_doubles() / size_t(total_rows()));
    int64_t maxJ = 0, maxI = 0;
    for (int n = 0; n < N_; ++n) {
      maxJ = std::max(maxJ, E_ / e.dim(n));
      maxI = std::max(maxI, e.dim(n));
    }
    xn_ = c.buf<T>("uf.xn", size_t(E_));
    xh_ = c.buf<T>("uf.xh", size_t(E_));
    q_ = c.buf<T>("uf.q", size_t(E_));
    kr_ = c.buf<T>("uf.kr", size_t(maxJ * R_));
    num_ = c.buf<T>("uf.num", size_t(maxI * R_));
    den_ = c.buf<T>("uf.den", size_t(maxI * R_));
    at_ = c.buf<T>("uf.at", e.factor_doubles());
    rows_ = c.buf<int64_t>("uf.rows", kMaxOrder);
  }

  void sweep() {
    const int64_t F = int64_t(e_.factor_doubles());
    to_t_kernel<T><<<grid(F), 256, 0, c_.stream>>>(e_.A_all(), F, at_);
    NTFG_LAUNCHED(c_);
    if (N_ == 1) throw Error(NTFG_ERR_SHAPE, "mu_unfold_cp_sweep: order-1 tensors are not supported on the GPU");
    for (int n = 0; n < N_; ++n) {
      const int64_t I = e_.dim(n), J = E_ / I;
      // KR of the off-mode factors, ascending modes
      const double* m[kMaxOrder - 1] = {};
      int64_t hr[kMaxOrder] = {};
      int k = 0;
      for (int mm = 0; mm < N_; ++mm)
        if (mm != n) {
          m[k] = e_.A(mm);
          hr[k] = e_.dim(mm);
          ++k;
        }
      c_.h2d(rows_, hr, sizeof(hr));
      khatri_rao_kernel<T><<<grid(J * R_), 256, 0, c_.stream>>>(k, J, int(R_), rows_, m[0], m[1], m[2], m[3],
                                                                 m[4], m[5], m[6], kr_);
      NTFG_LAUNCHED(c_);
      // X_(n)
      int64_t A = 1, B = 1;
      for (int mm = 0; mm < n; ++mm) A *= e_.dim(mm);
      for (int mm = n + 1; mm < N_; ++mm) B *= e_.dim(mm);
      unfold_kernel<T><<<grid(E_), 256, 0, c_.stream>>>(e_.x(), A, I, B, xn_);
      NTFG_LAUNCHED(c_);
      // Xhat_(n) = A_n KR^T, then P (in place) and Q
      gemm_rm<T>(blas_.h, true, I, J, R_, at_ + e_.offset(n), kr_, xh_);
      unfolded_weights_kernel<T><<<grid(E_), 256, 0, c_.stream>>>(xn_, xh_, q_, E_, bk_, beta_, eps_);
      NTFG_LAUNCHED(c_);
      gemm_rm<T>(blas_.h, false, I, R_, J, xh_, kr_, num_);
      gemm_rm<T>(blas_.h, false, I, R_, J, q_, kr_, den_);
      unfold_mu_kernel<T><<<grid(I * R_), 256, 0, c_.stream>>>(e_.A(n), num_, den_, I * R_, gamma_, eps_,
                                                               at_ + e_.offset(n));
      NTFG_LAUNCHED(c_);
    }
    e_.restage();
  }

 private:
  int64_t total_rows() const {
    int64_t s = 0;
    for (int n = 0; n < N_; ++n) s += e_.dim(n);
    return s;
  }
  int grid(int64_t n) const { return int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 148 * 32))); }

  Context& c_;
  CpEngine<T>& e_;
  Cublas blas_;
  double beta_, eps_, gamma_;
  int bk_;
  int N_ = 0;
  int64_t E_ = 0, R_ = 0;
  T *xn_, *xh_, *q_, *kr_, *num_, *den_, *at_;
  int64_t* rows_;
};

// mu_unfold_cp_fit (unfold.cpp:187-197): run_outer_loop with the sweep as the
// step and D_beta_mean of the reconstruction as the loss (eager: no graphs).
void cp_mu_unfold_fit(Context& c, const ntfg_fit_config& cfg0, uint32_t order, const uint64_t* dims, const void* x,
                      int dtype, int loc, double* factors, ntfg_trace_row* trace, uint64_t* trace_len) {
  validate_config(cfg0);
  ntfg_fit_config cfg = cfg0;
  cfg.use_graphs = 0;
  c.stats = ntfg_stats{};
  auto run = [&](auto tag) {
    using T = decltype(tag);
    CpEngine<T> e(c, order, dims, int64_t(cfg.rank), cfg.beta, cfg.eps, nullptr);
    e.disable_tc();
    e.set_x(x, dtype, loc);
    e.set_factors_host(factors);
    double* losses = c.buf<double>("fit.losses", cfg.max_iters + 2);
    e.bind_losses(losses);
    e.reset_counter();
    e.reset_flags();
    UnfoldCp<T> u(c, e, cfg.beta, cfg.eps);
    const size_t bytes = e.factor_doubles() * sizeof(double);
    double* snap = c.buf<double>("cp.snap", e.factor_doubles());
    LoopHooks h;
    h.fused = false;
    h.objective = [&]() { e.objective(); };
    h.snapshot = [&]() { c.d2d(snap, e.A_all(), bytes); };
    h.restore = [&]() {
      c.d2d(e.A_all(), snap, bytes);
      e.restage();
    };
    h.body = [&]() {
      u.sweep();
      e.objective();
    };
    auto tr = run_fit_loop(c, cfg, h, losses, e.flags());
    e.get_factors_host(factors);
    c.sync();
    return tr;
  };
  std::vector<ntfg_trace_row> tr = cfg.precision == NTFG_F32 ? run(float{}) : run(double{});
  for (size_t i = 0; i < tr.size(); ++i) trace[i] = tr[i];
  *trace_len = tr.size();
}

void cp_mu_unfold_sweep(Context& c, int prec, double beta, double eps, uint32_t order, const uint64_t* dims,
                        const double* x, uint64_t rank, double* factors) {
  auto run = [&](auto tag) {
    using T = decltype(tag);
    CpEngine<T> e(c, order, dims, int64_t(rank), beta, eps, nullptr);
    e.disable_tc();
    e.set_x(x, 0, NTFG_HOST);
    e.set_factors_host(factors);
    e.reset_flags();
    UnfoldCp<T> u(c, e, beta, eps);
    u.sweep();
    e.get_factors_host(factors);
    c.sync();
  };
  if (prec == NTFG_F32) run(float{});
  else run(double{});
}

// ---- Tucker MU-unfold (unfold.cpp:137-185): every mode product through an
// explicit matricisation (unfold -> cuBLAS GEMM -> refold), the partial
// reconstruction of the factor updates materialised in full ---------------------

// refold (unfold.cpp:38-62) of Y_(n) = [I][A*B] into [A][I][B]
template <typename T>
static __global__ void refold_kernel(const T* y, int64_t A, int64_t I, int64_t B, T* out) {
  const int64_t E = A * I * B;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < E; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = e % B;
    const int64_t t = e / B;
    const int64_t i = t % I;
    const int64_t a = t / I;
    out[e] = y[i * (A * B) + a * B + b];
  }
}

// [rows][cols] fp64 -> [cols][rows] T
template <typename T>
static __global__ void transpose_t_kernel(const double* src, int64_t rows, int64_t cols, T* dst) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < rows * cols;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c = e / rows, r = e % rows;
    dst[e] = T(src[r * cols + c]);
  }
}

template <typename T>
class UnfoldTucker {
 public:
  UnfoldTucker(Context& c, TuckerEngine<T>& e, uint32_t order, const uint64_t* dims, const uint64_t* ranks,
               double beta, double eps)
      : c_(c), e_(e), blas_(c.stream), beta_(beta), eps_(eps), gamma_(gamma_of(beta)), bk_(beta_kind_of(beta)) {
    N_ = int(order);
    E_ = 1;
    int64_t J = 1, maxIJ = 1;
    for (int m = 0; m < N_; ++m) {
      I_[m] = int64_t(dims[m]);
      J_[m] = int64_t(ranks[m]);
      E_ *= I_[m];
      J *= J_[m];
      maxIJ = std::max(maxIJ, I_[m] * J_[m]);
    }
    // largest intermediate of any chain: every mixed shape of I's and J's
    int64_t big = std::max(E_, J);
    for (int mask = 0; mask < (1 << N_); ++mask) {
      int64_t sz = 1;
      for (int m = 0; m < N_; ++m) sz *= (mask >> m & 1) ? I_[m] : J_[m];
      big = std::max(big, sz);
    }
    big_ = big;
    for (int i = 0; i < 5; ++i) w_[i] = c.buf<T>("ut.w" + std::to_string(i), size_t(big));
    mt_ = c.buf<T>("ut.mt", size_t(maxIJ));
    num_ = c.buf<T>("ut.num", size_t(std::max(maxIJ, J)));
    den_ = c.buf<T>("ut.den", size_t(std::max(maxIJ, J)));
    model_t_ = c.buf<T>("ut.model", e.model_doubles());
  }

  void sweep() {
    const int64_t Jc = e_.core_size();
    to_t_kernel<T><<<grid(int64_t(e_.model_doubles())), 256, 0, c_.stream>>>(e_.model(), int64_t(e_.model_doubles()),
                                                                             model_t_);
    NTFG_LAUNCHED(c_);
    // core update: Xhat = G x_0 A_0 ... x_{N-1} A_{N-1}; P, Q; contract back with A_k^T
    {
      T* xh = reconstruct(-1);  // into w_[0] or w_[1]
      T* p = xh;
      T* q = w_[2];
      weights(p, q);
      int64_t sh[kMaxOrder];
      for (int m = 0; m < N_; ++m) sh[m] = I_[m];
      T* pc = shrink_all(p, sh, w_[3], w_[4]);  // result in w_[3] or w_[4]
      for (int m = 0; m < N_; ++m) sh[m] = I_[m];
      // park P_core (q's chain reuses the ping-pong buffers)
      NTFG_CUDA(cudaMemcpyAsync(num_, pc, size_t(Jc) * sizeof(T), cudaMemcpyDeviceToDevice, c_.stream));
      T* qc = shrink_all(q, sh, w_[3], w_[4]);
      NTFG_CUDA(cudaMemcpyAsync(den_, qc, size_t(Jc) * sizeof(T), cudaMemcpyDeviceToDevice, c_.stream));
      unfold_mu_kernel<T><<<grid(Jc), 256, 0, c_.stream>>>(e_.G(), num_, den_, Jc, gamma_, eps_, model_t_);
      NTFG_LAUNCHED(c_);
    }
    // factor updates, ascending modes, each from the current model
    for (int n = 0; n < N_; ++n) {
      T* xh = reconstruct(-1);
      T* p = xh;
      T* q = w_[2];
      weights(p, q);
      // P_(n), Q_(n)
      int64_t A = 1, B = 1;
      for (int m = 0; m < n; ++m) A *= I_[m];
      for (int m = n + 1; m < N_; ++m) B *= I_[m];
      T* pn = w_[3];
      T* qn = w_[4];
      unfold_kernel<T><<<grid(E_), 256, 0, c_.stream>>>(p, A, I_[n], B, pn);
      NTFG_LAUNCHED(c_);
      unfold_kernel<T><<<grid(E_), 256, 0, c_.stream>>>(q, A, I_[n], B, qn);
      NTFG_LAUNCHED(c_);
      // partial = G x_{k != n} A_k, unfolded along n: [J_n][E / I_n]
      T* part = reconstruct(n);  // w_[0] or w_[1]
      T* up = part == w_[0] ? w_[1] : w_[0];
      int64_t Ap = 1, Bp = 1;
      for (int m = 0; m < n; ++m) Ap *= I_[m];
      for (int m = n + 1; m < N_; ++m) Bp *= I_[m];
      unfold_kernel<T><<<grid(Ap * J_[n] * Bp), 256, 0, c_.stream>>>(part, Ap, J_[n], Bp, up);
      NTFG_LAUNCHED(c_);
      // num = P_(n) * U^T, den = Q_(n) * U^T  ([I_n][J_n])
      gemm_rm<T>(blas_.h, true, I_[n], J_[n], E_ / I_[n], pn, up, num_);
      gemm_rm<T>(blas_.h, true, I_[n], J_[n], E_ / I_[n], qn, up, den_);
      unfold_mu_kernel<T><<<grid(I_[n] * J_[n]), 256, 0, c_.stream>>>(
          e_.A(n), num_, den_, I_[n] * J_[n], gamma_, eps_, model_t_ + Jc + e_.factor_offset(n));
      NTFG_LAUNCHED(c_);
    }
    e_.restage();
  }

 private:
  int grid(int64_t n) const { return int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 148 * 32))); }

  // t (shape sh) x_mode M, M = [rows][sh[mode]] row-major T; unfold -> GEMM -> refold
  void mode_product(const T* t, int64_t* sh, const T* M, int64_t rows, int mode, T* scratch, T* out) {
    int64_t A = 1, B = 1;
    for (int m = 0; m < mode; ++m) A *= sh[m];
    for (int m = mode + 1; m < N_; ++m) B *= sh[m];
    const int64_t I = sh[mode];
    unfold_kernel<T><<<grid(A * I * B), 256, 0, c_.stream>>>(t, A, I, B, scratch);
    NTFG_LAUNCHED(c_);
    gemm_rm<T>(blas_.h, false, rows, A * B, I, M, scratch, out);  // [rows][A*B]
    // out holds Y_(mode); refold into scratch then swap roles via copy-free pointer return
    refold_kernel<T><<<grid(A * rows * B), 256, 0, c_.stream>>>(out, A, rows, B, scratch);
    NTFG_LAUNCHED(c_);
    sh[mode] = rows;
  }

  // G x_{k != skip} A_k (skip = -1: full reconstruction); result in w_[0] or w_[1]
  T* reconstruct(int skip) {
    int64_t sh[kMaxOrder];
    for (int m = 0; m < N_; ++m) sh[m] = J_[m];
    const T* cur = model_t_;  // core first in the model layout
    T* bufs[2] = {w_[0], w_[1]};
    int which = 0;
    for (int k = 0; k < N_; ++k) {
      if (k == skip) continue;
      const T* Ak = model_t_ + e_.core_size() + e_.factor_offset(k);  // [I_k][J_k]
      // mode_product leaves the refolded result in its scratch argument
      T* scratch = bufs[which];
      mode_product(cur, sh, Ak, I_[k], k, scratch, w_[2]);
      cur = scratch;
      which ^= 1;
    }
    if (cur == model_t_) {  // nothing multiplied (order 1 with skip): copy the core
      NTFG_CUDA(cudaMemcpyAsync(w_[0], model_t_, size_t(e_.core_size()) * sizeof(T), cudaMemcpyDeviceToDevice,
                                c_.stream));
      return w_[0];
    }
    return const_cast<T*>(cur);
  }

  // t (shape I) x_k A_k^T for every k: [I...] -> [J...]; ping-pong between b0 and b1
  T* shrink_all(T* t, int64_t* sh, T* b0, T* b1) {
    const T* cur = t;
    T* bufs[2] = {b0, b1};
    int which = 0;
    for (int k = 0; k < N_; ++k) {
      transpose_t_kernel<T><<<grid(I_[k] * J_[k]), 256, 0, c_.stream>>>(e_.A(k), I_[k], J_[k], mt_);
      NTFG_LAUNCHED(c_);
      T* scratch = bufs[which];
      T* gout = (cur == w_[0] || cur == w_[1]) ? (cur == w_[0] ? w_[1] : w_[0]) : w_[0];
      mode_product(cur, sh, mt_, J_[k], k, scratch, gout);
      cur = scratch;
      which ^= 1;
    }
    return const_cast<T*>(cur);
  }

  void weights(T* xh_to_p, T* q) {
    unfolded_weights_kernel<T><<<grid(E_), 256, 0, c_.stream>>>(e_.stream().x(), xh_to_p, q, E_, bk_, beta_, eps_);
    NTFG_LAUNCHED(c_);
  }

  Context& c_;
  TuckerEngine<T>& e_;
  Cublas blas_;
  double beta_, eps_, gamma_;
  int bk_;
  int N_ = 0;
  int64_t E_ = 0, big_ = 0;
  int64_t I_[kMaxOrder] = {}, J_[kMaxOrder] = {};
  T* w_[5];
  T *mt_, *num_, *den_, *model_t_;
};

template <typename T>
static std::vector<ntfg_trace_row> tucker_mu_unfold_fit_t(Context& c, const ntfg_fit_config& cfg, uint32_t order,
                                                           const uint64_t* dims, const void* x, int dtype, int loc,
                                                           double* core, double* factors) {
  if (cfg.n_ranks != order || !cfg.ranks)
    throw Error(NTFG_ERR_SHAPE, "TuckerModel: core order does not match factor count");
  TuckerEngine<T> e(c, order, dims, cfg.ranks, cfg.beta, cfg.eps, nullptr);
  e.stream().set_x(x, dtype, loc);
  e.set_model_host(core, factors);
  double* losses = c.buf<double>("fit.losses", cfg.max_iters + 2);
  e.stream().bind_losses(losses);
  e.stream().reset_counter();
  e.stream().reset_flags();
  UnfoldTucker<T> u(c, e, order, dims, cfg.ranks, cfg.beta, cfg.eps);
  const size_t bytes = e.model_doubles() * sizeof(double);
  double* snap = c.buf<double>("tk.snap", e.model_doubles());
  LoopHooks h;
  h.fused = false;
  h.objective = [&]() { e.objective(); };
  h.snapshot = [&]() { c.d2d(snap, e.model(), bytes); };
  h.restore = [&]() {
    c.d2d(e.model(), snap, bytes);
    e.restage();
  };
  h.body = [&]() {
    u.sweep();
    e.objective();
  };
  auto tr = run_fit_loop(c, cfg, h, losses, e.stream().flags());
  e.get_model_host(core, factors);
  c.sync();
  return tr;
}

// mu_unfold_tucker_fit (unfold.cpp:199-209): run_outer_loop with the sweep as the step (eager)
void tucker_mu_unfold_fit(Context& c, const ntfg_fit_config& cfg0, uint32_t order, const uint64_t* dims,
                          const void* x, int dtype, int loc, double* core, double* factors, ntfg_trace_row* trace,
                          uint64_t* trace_len) {
  validate_config(cfg0);
  ntfg_fit_config cfg = cfg0;
  cfg.use_graphs = 0;
  c.stats = ntfg_stats{};
  std::vector<ntfg_trace_row> tr =
      cfg.precision == NTFG_F32 ? tucker_mu_unfold_fit_t<float>(c, cfg, order, dims, x, dtype, loc, core, factors)
                                : tucker_mu_unfold_fit_t<double>(c, cfg, order, dims, x, dtype, loc, core, factors);
  for (size_t i = 0; i < tr.size(); ++i) trace[i] = tr[i];
  *trace_len = tr.size();
}

void tucker_mu_unfold_sweep(Context& c, int prec, double beta, double eps, uint32_t order, const uint64_t* dims,
                            const uint64_t* ranks, const double* x, double* core, double* factors) {
  auto run = [&](auto tag) {
    using T = decltype(tag);
    TuckerEngine<T> e(c, order, dims, ranks, beta, eps, nullptr);
    e.stream().set_x(x, 0, NTFG_HOST);
    e.set_model_host(core, factors);
    e.stream().reset_flags();
    UnfoldTucker<T> u(c, e, order, dims, ranks, beta, eps);
    u.sweep();
    e.get_model_host(core, factors);
    c.sync();
  };
  if (prec == NTFG_F32) run(float{});
  else run(double{});
}

}  // namespace ntfg
