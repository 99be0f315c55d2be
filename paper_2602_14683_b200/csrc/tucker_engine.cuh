// Tucker engine: device state of one Tucker problem, B-CoMM and J-CoMM steps.
//
// Reference: src/tucker.cpp (block updates 44-88, joint-MM 92-149) and the
// contraction engine tensor.cpp:408-560.  Data flow per update:
//   Xhat:  Y = core x_0 A_0 ... x_{L-1} A_{L-1}   (small fp64 TTM chain)
//          X^(row,k) = sum_j Y(row,j) A_L(k,j)     (E-sized, CP recon kernel, H = Y)
//   core numerator (multimode contraction, tensor.cpp:421-456):
//          T(row,j_L) = sum_k P(row,k) A_L(k,j_L)  (E-sized rowgemm)
//          then T x_m A_m^T for m < L              (small chain)
//   factor n < L (fused form, tensor.cpp:514-560): T, chain over m != n,
//          then pairing with the core
//   factor L: Num(k,j) = sum_rows P(row,k) Y(row,j) (E-sized, CP contract
//          kernel case A with the Y table) -> CP finalize (MU + chi)
// Only the E-sized passes stream X / P / Q; everything else is O(E J / I_L).
#pragma once
#include <algorithm>
#include <vector>

#include "cp_engine.cuh"
#include "tucker_kernels.cuh"

namespace ntfg {

template <typename T>
class TuckerEngine {
 public:
  TuckerEngine(Context& c, uint32_t order, const uint64_t* dims, const uint64_t* ranks, double beta,
               double eps, const ntfg_shard* shard)
      : c_(c), N_(int(order)), L_(int(order) - 1), beta_(beta), eps_(eps),
        s_(c, order, dims, int64_t(ranks[order - 1]), beta, eps, shard) {
    s_.disable_tc();  // Tucker streams contract fp32 P/Q with the row-table kernels
    gamma_ = gamma_of(beta);
    I_.resize(N_);
    J_.resize(N_);
    Jtot_ = 1;
    for (int m = 0; m < N_; ++m) {
      I_[m] = int64_t(dims[m]);
      J_[m] = int64_t(ranks[m]);
      if (J_[m] < 1) throw Error(NTFG_ERR_DOMAIN, "every core rank must be >= 1");
      Jtot_ *= J_[m];
    }
    rows_ = 1;
    for (int m = 0; m < L_; ++m) rows_ *= I_[m];
    foff_.assign(N_ + 1, 0);
    for (int m = 0; m < N_; ++m) foff_[m + 1] = foff_[m] + I_[m] * J_[m];
    F_ = foff_[N_];
    const size_t B = size_t(Jtot_ + F_);
    GA_ = c_.buf<double>("tk.GA", B);
    ref_ = c_.buf<double>("tk.ref", B);
    chi1_ = c_.buf<double>("tk.chi1", B);
    chi2_ = c_.buf<double>("tk.chi2", B);
    anch_ = c_.buf<double>("tk.anchor", B);
    RP_ = pad_rank(J_[L_]);
    stageL_ = c_.buf<T>("tk.stageL", size_t(I_[L_]) * RP_);
    stageS_ = c_.buf<T>("tk.stageS", size_t(I_[L_]) * RP_);
    Y1_ = c_.buf<double>("tk.Y1", size_t(rows_ * J_[L_]));
    Y2_ = c_.buf<double>("tk.Y2", size_t(rows_ * J_[L_]));
    T1_ = c_.buf<double>("tk.T1", size_t(rows_ * J_[L_]));
    // chain scratch: largest intermediate of any chain we run
    int64_t big = std::max<int64_t>(Jtot_, rows_ * J_[L_]);
    {
      // Y chain: core with axes 0..m replaced by I
      int64_t sz = Jtot_;
      for (int m = 0; m < L_; ++m) { sz = sz / J_[m] * I_[m]; big = std::max(big, sz); }
      // contraction chains: T with axes replaced by J (any subset, ascending)
      int64_t sz2 = rows_ * J_[L_];
      for (int m = 0; m < L_; ++m) { sz2 = sz2 / I_[m] * std::max(I_[m], J_[m]); big = std::max(big, sz2); }
    }
    W1_ = c_.buf<double>("tk.W1", size_t(big));
    W2_ = c_.buf<double>("tk.W2", size_t(big));
    int64_t nb = Jtot_;
    for (int m = 0; m < N_; ++m) nb = std::max(nb, I_[m] * J_[m]);
    num_ = c_.buf<double>("tk.num", size_t(2 * nb));  // [Num | Den] packed for the allreduce
    den_ = c_.buf<double>("tk.den", size_t(nb));
  }

  CpEngine<T>& stream() { return s_; }
  double* G() const { return GA_; }
  double* A(int m) const { return GA_ + Jtot_ + foff_[m]; }
  size_t model_doubles() const { return size_t(Jtot_ + F_); }
  int64_t core_size() const { return Jtot_; }
  double* model() const { return GA_; }
  double* anchors() const { return anch_; }
  double* refs() const { return ref_; }
  int64_t factor_offset(int m) const { return foff_[m]; }

  void set_model_host(const double* core, const double* factors) {
    c_.h2d(GA_, core, size_t(Jtot_) * sizeof(double));
    c_.h2d(GA_ + Jtot_, factors, size_t(F_) * sizeof(double));
    restage();
  }
  void get_model_host(double* core, double* factors) {
    if (core) c_.d2h(core, GA_, size_t(Jtot_) * sizeof(double));
    if (factors) c_.d2h(factors, GA_ + Jtot_, size_t(F_) * sizeof(double));
  }
  void restage() { s_.stage(A(L_), stageL_); }

  // ---- small chains ---------------------------------------------------------
  void ttm(const double* in, std::vector<int64_t>& shape, int axis, const double* M, int64_t na,
           int trans, double* out) {
    int64_t outer = 1, inner = 1;
    for (int a = 0; a < axis; ++a) outer *= shape[a];
    for (size_t a = axis + 1; a < shape.size(); ++a) inner *= shape[a];
    const int64_t nb = shape[axis];
    const int64_t total = outer * na * inner;
    const int grid = int(std::min<int64_t>(ceil_div(total, 256), int64_t(c_.sm_count) * 16));
    const int ph = c_.prof_begin(2);
    const int cgrid = int(std::min<int64_t>(outer * ceil_div(inner, 32), int64_t(c_.sm_count) * 8));
    if (trans && nb >= 64 && (na == 8 || na == 16)) {  // contracting product: split-b tiles
      if (na == 8) ttm_contract_kernel<8><<<cgrid, 256, 0, c_.stream>>>(in, outer, nb, inner, M, out);
      else ttm_contract_kernel<16><<<cgrid, 256, 0, c_.stream>>>(in, outer, nb, inner, M, out);
    } else {
      ttm_kernel<<<std::max(grid, 1), 256, 0, c_.stream>>>(in, outer, nb, inner, M, na, trans, out);
    }
    NTFG_LAUNCHED(c_);
    c_.prof_end(ph);
    shape[axis] = na;
  }

  // Y = core x_0 A_0 ... x_{L-1} A_{L-1}  (shape [I_0..I_{L-1}, J_L])
  void ychain(const double* core, const double* const* fac, double* Y) {
    std::vector<int64_t> shape(J_.begin(), J_.end());
    if (L_ == 0) {
      c_.d2d(Y, core, size_t(Jtot_) * sizeof(double));
      return;
    }
    const double* cur = core;
    for (int m = 0; m < L_; ++m) {
      double* dst = (m == L_ - 1) ? Y : ((m % 2 == 0) ? W1_ : W2_);
      ttm(cur, shape, m, fac[m], I_[m], 0, dst);
      cur = dst;
    }
  }

  // T(row, j_L) = sum_k S(row, k) F_L(k, j_L)
  void rowgemm(const T* S, const double* FL) {
    s_.stage(FL, stageS_);
    const int64_t warps_needed = rows_;
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(warps_needed, 8), int64_t(c_.sm_count) * 8)));
    const int ph = c_.prof_begin(1);
    const int64_t K = I_[L_];
    bool tiled = false;
    if constexpr (sizeof(T) == 4) {
      // tiled fp32 kernel: 32-column stages, 16-byte rows, F resident in shared memory
      tiled = K % kRgCols == 0 && (reinterpret_cast<uintptr_t>(S) % 16) == 0 && size_t(K) * RP_ * 4 <= 64 * 1024;
      if (tiled) {
        const int tgrid = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows_, kRgRows), int64_t(c_.sm_count) * 2)));
        switch (RP_) {
          case 8: launch_rg<8>(tgrid, S, K); break;
          case 16: launch_rg<16>(tgrid, S, K); break;
          case 32: launch_rg<32>(tgrid, S, K); break;
          default: launch_rg<64>(tgrid, S, K); break;
        }
      }
    }
    if (!tiled) {
      switch (RP_) {
        case 8: rowgemm_kernel<T, 8><<<grid, 256, 0, c_.stream>>>(S, rows_, I_[L_], stageS_, int(J_[L_]), T1_); break;
        case 16: rowgemm_kernel<T, 16><<<grid, 256, 0, c_.stream>>>(S, rows_, I_[L_], stageS_, int(J_[L_]), T1_); break;
        case 32: rowgemm_kernel<T, 32><<<grid, 256, 0, c_.stream>>>(S, rows_, I_[L_], stageS_, int(J_[L_]), T1_); break;
        default: rowgemm_kernel<T, 64><<<grid, 256, 0, c_.stream>>>(S, rows_, I_[L_], stageS_, int(J_[L_]), T1_); break;
      }
    }
    NTFG_LAUNCHED(c_);
    c_.prof_end(ph);
  }
  template <int JP>
  void launch_rg(int grid, const T* S, int64_t K) {
    if constexpr (sizeof(T) == 4) {
      const size_t sm = RgSmem<JP>::total(K);
      static size_t attr = 0;
      if (sm > attr) {
        cuda_check(cudaFuncSetAttribute(rowgemm_tiled_kernel<JP>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)),
                   "cudaFuncSetAttribute");
        attr = sm;
      }
      rowgemm_tiled_kernel<JP><<<grid, 64 * (JP / 8), sm, c_.stream>>>(S, rows_, K, stageS_, int(J_[L_]), T1_);
    }
  }

  // multimode contraction of S against all factors -> core-shaped out
  // (reference tucker_multimode_contract, tensor.cpp:421-456)
  void contract_core(const T* S, const double* const* fac, double* out) {
    rowgemm(S, fac[L_]);
    std::vector<int64_t> shape(I_.begin(), I_.begin() + L_);
    shape.push_back(J_[L_]);
    if (L_ == 0) {
      c_.d2d(out, T1_, size_t(Jtot_) * sizeof(double));
      return;
    }
    const double* cur = T1_;
    for (int m = 0; m < L_; ++m) {
      double* dst = (m == L_ - 1) ? out : ((m % 2 == 0) ? W1_ : W2_);
      ttm(cur, shape, m, fac[m], J_[m], 1, dst);
      cur = dst;
    }
  }

  // fused factor contraction for n < L (tensor.cpp:514-560)
  void contract_factor(const T* S, const double* core, const double* const* fac, int n, double* out) {
    rowgemm(S, fac[L_]);
    std::vector<int64_t> shape(I_.begin(), I_.begin() + L_);
    shape.push_back(J_[L_]);
    const double* cur = T1_;
    int step = 0;
    for (int m = 0; m < L_; ++m) {
      if (m == n) continue;
      double* dst = (step % 2 == 0) ? W1_ : W2_;
      ttm(cur, shape, m, fac[m], J_[m], 1, dst);
      cur = dst;
      ++step;
    }
    PairParams p{};
    p.order = N_;
    p.n = n;
    p.In = I_[n];
    for (int m = 0; m < N_; ++m) p.J[m] = J_[m];
    p.S = cur;
    p.G = core;
    p.out = out;
    const int ph = c_.prof_begin(2);
    core_pair_kernel<<<int(ceil_div(I_[n] * J_[n], 128)), 128, 0, c_.stream>>>(p);
    NTFG_LAUNCHED(c_);
    c_.prof_end(ph);
  }

  // Data-parallel (mode-0 slabs): the core's and factors
  // 1..L-1's Num/Den are sums over the WHOLE tensor (tucker.cpp:44-88), so
  // each rank's slab-local sums are packed [Num | Den] and allreduced before
  // the identical MU step on every rank.  Factor 0's rows are rank-local;
  // the last factor reduces inside CpEngine::contract_and_update.
  void reduce_numden(int64_t cnt) {
    if (!s_.sharded()) return;
    c_.d2d(num_ + cnt, den_, size_t(cnt) * sizeof(double));
    s_.allreduce(num_, size_t(2 * cnt));
    c_.d2d(den_, num_ + cnt, size_t(cnt) * sizeof(double));
  }

  void mu_dense(const double* anchor, int64_t n, double* out, const double* ref, double* c1,
                double* c2) {
    mu_dense_kernel<<<int(ceil_div(n, 256)), 256, 0, c_.stream>>>(anchor, num_, den_, n, gamma_, eps_, beta_, out,
                                                                   ref, c1, c2, s_.flag_ptr());
    NTFG_LAUNCHED(c_);
  }

  // recon of (core, fac) with staged last factor -> P/Q (+objective)
  void recon(const double* core, const double* const* fac, const T* stage_last, bool pq, bool objective) {
    ychain(core, fac, Y1_);
    const double* dummy[kMaxOrder];
    for (int m = 0; m < N_; ++m) dummy[m] = A(m);
    s_.ensure_pq();
    s_.recon(dummy, stage_last, pq ? s_.p() : nullptr, pq ? s_.q_always() : nullptr, objective,
             nullptr, Y1_);
  }

  void update_last(const double* core1, const double* const* f1, const double* core2,
                   const double* const* f2, const double* anchor, const double* ref, double* c1,
                   double* c2) {
    ychain(core1, f1, Y1_);
    const double* Y2 = Y1_;
    if (core2 != core1 || f2 != f1) {
      ychain(core2, f2, Y2_);
      Y2 = Y2_;
    }
    typename CpEngine<T>::Stream st[2];
    st[0].src = s_.p();
    st[1].src = s_.q_always();
    for (int m = 0; m < N_; ++m) st[0].fac[m] = st[1].fac[m] = A(m);
    st[0].mtab = Y1_;
    st[1].mtab = Y2;
    s_.contract_and_update(L_, 2, st, false, anchor, A(L_), ref, c1, c2, stageL_);
  }

  // ---- B-CoMM (tucker.cpp:44-88) ---------------------------------------------
  void block_core(const double* anchor_core, bool objective) {
    const double* fac[kMaxOrder];
    for (int m = 0; m < N_; ++m) fac[m] = A(m);
    recon(anchor_core, fac, stageL_, true, objective);
    contract_core(s_.p(), fac, num_);
    contract_core(s_.q_always(), fac, den_);
    reduce_numden(Jtot_);
    mu_dense(anchor_core, Jtot_, G(), nullptr, nullptr, nullptr);
  }

  void block_factor(int n, const double* anchor) {
    const double* fac[kMaxOrder];
    for (int m = 0; m < N_; ++m) fac[m] = (m == n) ? anchor : A(m);
    const T* sl = stageL_;
    if (n == L_ && anchor != A(L_)) {
      s_.stage(anchor, stageS_);
      sl = stageS_;
    }
    recon(G(), fac, sl, true, false);
    if (n == L_) {
      update_last(G(), fac, G(), fac, anchor, nullptr, nullptr, nullptr);
    } else {
      contract_factor(s_.p(), G(), fac, n, num_);
      contract_factor(s_.q_always(), G(), fac, n, den_);
      if (n != 0) reduce_numden(I_[n] * J_[n]);
      mu_dense(anchor, I_[n] * J_[n], A(n), nullptr, nullptr, nullptr);
    }
  }

  void bcomm_sweep(bool objective) {
    block_core(G(), objective);
    for (int n = 0; n < N_; ++n) block_factor(n, A(n));
  }

  void bcomm_sweep_anchored(const double* anch) {
    block_core(anch, false);
    for (int n = 0; n < N_; ++n) block_factor(n, anch + Jtot_ + foff_[n]);
  }

  // ---- J-CoMM (tucker.cpp:92-149) --------------------------------------------
  void jcomm_reference(bool objective) {
    const size_t bytes = model_doubles() * sizeof(double);
    c_.d2d(ref_, GA_, bytes);
    c_.d2d(chi1_, GA_, bytes);
    c_.d2d(chi2_, GA_, bytes);
    const double* fac[kMaxOrder];
    for (int m = 0; m < N_; ++m) fac[m] = A(m);
    recon(G(), fac, stageL_, true, objective);
  }

  void fac_ptrs(double* base, const double** out) const {
    for (int m = 0; m < N_; ++m) out[m] = base + Jtot_ + foff_[m];
  }

  void jcomm_inner_core() {
    const double* f1[kMaxOrder];
    const double* f2[kMaxOrder];
    fac_ptrs(chi1_, f1);
    fac_ptrs(chi2_, f2);
    contract_core(s_.p(), f1, num_);
    contract_core(s_.q_always(), f2, den_);
    reduce_numden(Jtot_);
    mu_dense(ref_, Jtot_, G(), ref_, chi1_, chi2_);
  }

  void jcomm_inner_factor(int n) {
    const double* f1[kMaxOrder];
    const double* f2[kMaxOrder];
    fac_ptrs(chi1_, f1);
    fac_ptrs(chi2_, f2);
    const int64_t o = Jtot_ + foff_[n];
    if (n == L_) {
      update_last(chi1_, f1, chi2_, f2, ref_ + o, ref_ + o, chi1_ + o, chi2_ + o);
    } else {
      contract_factor(s_.p(), chi1_, f1, n, num_);
      contract_factor(s_.q_always(), chi2_, f2, n, den_);
      if (n != 0) reduce_numden(I_[n] * J_[n]);
      mu_dense(ref_ + o, I_[n] * J_[n], A(n), ref_ + o, chi1_ + o, chi2_ + o);
    }
  }

  void jcomm_outer(int inner, bool objective) {
    jcomm_reference(objective);
    for (int l = 0; l < inner; ++l) {
      jcomm_inner_core();
      for (int n = 0; n < N_; ++n) jcomm_inner_factor(n);
    }
  }

  void objective() {
    const double* fac[kMaxOrder];
    for (int m = 0; m < N_; ++m) fac[m] = A(m);
    recon(G(), fac, stageL_, false, true);
  }

  // ---- step-level helpers --------------------------------------------------------
  void set_ref_host(const double* core, const double* factors) {
    c_.h2d(ref_, core, size_t(Jtot_) * sizeof(double));
    c_.h2d(ref_ + Jtot_, factors, size_t(F_) * sizeof(double));
  }
  void chi_from_ref() {
    const int64_t B = int64_t(model_doubles());
    chi_all_kernel<<<int(ceil_div(B, 256)), 256, 0, c_.stream>>>(GA_, ref_, B, beta_, chi1_, chi2_, s_.flag_ptr());
    NTFG_LAUNCHED(c_);
  }
  // P~/Q~ of the reference model (make_jcomm_tucker_reference, tucker.cpp:92-98)
  void weights_of_ref() {
    const double* fac[kMaxOrder];
    fac_ptrs(ref_, fac);
    s_.stage(fac[L_], stageS_);
    recon(ref_, fac, stageS_, true, false);
  }
  double* num() const { return num_; }
  double* T1() const { return T1_; }
  int64_t rows() const { return rows_; }

 private:
  Context& c_;
  int N_, L_;
  double beta_, eps_, gamma_;
  CpEngine<T> s_;
  std::vector<int64_t> I_, J_, foff_;
  int64_t Jtot_, F_, rows_;
  int RP_;
  double *GA_, *ref_, *chi1_, *chi2_, *anch_;
  T *stageL_, *stageS_;
  double *Y1_, *Y2_, *T1_, *W1_, *W2_, *num_, *den_;
};

}  // namespace ntfg
