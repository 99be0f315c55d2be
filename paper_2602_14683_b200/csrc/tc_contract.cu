// K3 on the tensor cores: the tcgen05/TMEM/TMA contraction kernel
// (tc_contract.cuh) compiled as its own translation unit.
#define NTFG_TC_CONTRACT_IMPL
#include "tc_contract.cuh"

#include <mutex>

#include "engine.cuh"

namespace ntfg {

template <int N>
static void launch_instance(int grid, cudaStream_t stream, const TcMaps& maps, const TcParams& p) {
  static std::once_flag once;
  std::call_once(once, [] {
    cuda_check(cudaFuncSetAttribute(tc_contract_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(kTcSmemMax)),
               "cudaFuncSetAttribute");
  });
  tc_contract_kernel<N><<<grid, tc_threads<N>(), p.lay.total, stream>>>(maps, p);
}

void tc_contract_launch(int grid, cudaStream_t stream, const TcMaps& maps, const TcParams& p) {
  if (p.N == 16) launch_instance<16>(grid, stream, maps, p);
  else if (p.N == 32) launch_instance<32>(grid, stream, maps, p);
  else launch_instance<64>(grid, stream, maps, p);
}

}  // namespace ntfg
