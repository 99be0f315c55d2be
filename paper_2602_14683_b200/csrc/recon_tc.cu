// K2/K5 on the tensor cores: the tcgen05/TMEM reconstruction kernel
// (recon_tc.cuh) compiled as its own translation unit.
#define NTFG_RECON_TC_IMPL
#include "recon_tc.cuh"

#include <mutex>

#include "engine.cuh"

namespace ntfg {

template <int BK, int KC, int HV>
static void launch_hv(int grid, cudaStream_t stream, const ReconParams<float>& p, int RP) {
  static std::once_flag once;
  std::call_once(once, [] {
    cuda_check(cudaFuncSetAttribute(recon_tc_kernel<BK, KC, HV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(232448 - 1536)),
               "cudaFuncSetAttribute");
  });
  recon_tc_kernel<BK, KC, HV><<<grid, kRcThreads, rc_smem(RP), stream>>>(p, RP, rc_stages(RP));
}

template <int BK, int KC>
static void launch_kc(int grid, cudaStream_t stream, const ReconParams<float>& p, int RP) {
  if ((p.R & 3) != 0) launch_hv<BK, KC, 0>(grid, stream, p, RP);
  else if (p.hfac32 && !p.htab) launch_hv<BK, KC, 2>(grid, stream, p, RP);
  else launch_hv<BK, KC, 1>(grid, stream, p, RP);
}

template <int BK>
static void launch_bk(int grid, cudaStream_t stream, const ReconParams<float>& p, int RP) {
  switch (int(p.g.K / kRcCols)) {
    case 1: launch_kc<BK, 1>(grid, stream, p, RP); break;
    case 2: launch_kc<BK, 2>(grid, stream, p, RP); break;
    case 3: launch_kc<BK, 3>(grid, stream, p, RP); break;
    default: launch_kc<BK, 4>(grid, stream, p, RP); break;
  }
}

void recon_tc_launch(int grid, cudaStream_t stream, const ReconParams<float>& p, int RP, int bk) {
  switch (bk) {
    case kBeta1: launch_bk<kBeta1>(grid, stream, p, RP); break;
    case kBetaHalf: launch_bk<kBetaHalf>(grid, stream, p, RP); break;
    case kBeta3Half: launch_bk<kBeta3Half>(grid, stream, p, RP); break;
    case kBeta0: launch_bk<kBeta0>(grid, stream, p, RP); break;
    default: launch_bk<kBetaGeneric>(grid, stream, p, RP); break;
  }
}

}  // namespace ntfg
