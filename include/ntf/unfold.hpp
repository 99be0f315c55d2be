// Drop-in for reference include/ntf/unfold.hpp (unfold.cpp): the MU-unfold
// comparison path.  unfold / refold / khatri_rao are host utilities; the CP
// and Tucker sweeps and fits run on the GPU (explicit Khatri-Rao / unfolding +
// cuBLAS GEMMs + refold, ntfg_cp_mu_unfold_* and ntfg_tucker_mu_unfold_*).
#pragma once

#include <cstddef>
#include <span>
#include <vector>

#include "ntf/ntf.hpp"

namespace ntf {

struct UnfoldedView {
    Matrix matrix;
    std::size_t mode = 0;
};

UnfoldedView unfold(const DenseTensor& t, std::size_t mode);                    // unfold.cpp (mode-n matricisation)
DenseTensor refold(const UnfoldedView& u, std::span<const std::size_t> shape);
Matrix khatri_rao(std::span<const Matrix> mats);

CpFactors mu_unfold_cp_sweep(const CpFactors& f, const DenseTensor& x, const BetaParam& p, double eps);
CpFitResult mu_unfold_cp_fit(const DenseTensor& x, CpFactors init, const FitConfig& cfg);
TuckerModel mu_unfold_tucker_sweep(const TuckerModel& m, const DenseTensor& x, const BetaParam& p, double eps);
TuckerFitResult mu_unfold_tucker_fit(const DenseTensor& x, TuckerModel init, const FitConfig& cfg);

}  // namespace ntf
