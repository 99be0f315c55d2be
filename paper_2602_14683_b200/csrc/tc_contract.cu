// K3 on the tensor cores: the tcgen05/TMEM/TMA contraction kernel
// (tc_contract.cuh) compiled as its own translation unit.
#define NTFG_TC_CONTRACT_IMPL
#include "tc_contract.cuh"

#include <cstdlib>
#include <mutex>

#include "engine.cuh"

namespace ntfg {

template <int N, bool SB>
static void launch_instance(int grid, cudaStream_t stream, const TcMaps& maps, const TcParams& p) {
  static std::once_flag once;
  std::call_once(once, [] {
    cuda_check(cudaFuncSetAttribute(tc_contract_kernel<N, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(kTcSmemMax)),
               "cudaFuncSetAttribute");
  });
  tc_contract_kernel<N, SB><<<grid, tc_threads<N>(), p.lay.total, stream>>>(maps, p);
}

// bf16 hi/lo B tiles of every 16-row block of the fastest off-mode's fp32 factor copy, in the
// K-major core-matrix layout the MMA reads (same offsets as the B producers' stores)
static __global__ void stage_btiles_kernel(const float* f0, const float* f1, int ns, int runst, int N, uint32_t b_tile,
                                           unsigned char* out) {
  const int total = ns * runst * 2 * N;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int r = i % N, kg = (i / N) & 1, blk = (i / (2 * N)) % runst, s = i / (2 * N * runst);
    const float* f = (s ? f1 : f0) + size_t(blk * 16 + kg * 8) * N + r;
    uint32_t h[4], l[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) bf16_split_pair_fast(f[size_t(2 * e) * N], f[size_t(2 * e + 1) * N], h[e], l[e]);
    unsigned char* tile = out + size_t((s * runst + blk) * 2) * b_tile;
    const uint32_t off = uint32_t(r / 8) * kTcBSbo + uint32_t(kg) * 128 + uint32_t(r % 8) * 16;
    *reinterpret_cast<uint4*>(tile + off) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(tile + b_tile + off) = make_uint4(l[0], l[1], l[2], l[3]);
  }
}

void tc_contract_launch(int grid, cudaStream_t stream, const TcMaps& maps, const TcParams& pin) {
  TcParams p = pin;
  // static B tiles (tc_contract.cuh, TcParams::sb): fast-gather shapes whose runs of the fastest
  // off-mode are at least 8 stages long (shorter runs would mean a segment drain every few stages)
  static const bool sb_off = [] { const char* e = std::getenv("NTFG_TC_STATIC_B"); return e && e[0] == '0'; }();
  p.sb = 0;
  p.sb_runst = 0;
  // (at N <= 32 the producer warps kept up, so the gain there is only the saved SM work: C2 step
  // 317 -> 322 outer it/s on the same box; at N = 64 it removes the bottleneck)
  if (!sb_off && p.gfast && p.btiles && p.fmode >= 0 && !p.ablate) {
    const int64_t If = p.g.dims[p.fmode];
    if (If % kTcRows == 0 && If / kTcRows >= 8) {
      p.sb = 1;
      p.sb_runst = int(If / kTcRows);
      const int total = p.ns * p.sb_runst * 2 * p.N;
      stage_btiles_kernel<<<(total + 255) / 256, 256, 0, stream>>>(p.fac32[0][p.fmode], p.fac32[p.ns > 1 ? 1 : 0][p.fmode],
                                                                  p.ns, p.sb_runst, p.N, p.lay.b_tile, p.btiles);
    }
  }
  if (p.sb) {
    if (p.N == 16) launch_instance<16, true>(grid, stream, maps, p);
    else if (p.N == 32) launch_instance<32, true>(grid, stream, maps, p);
    else launch_instance<64, true>(grid, stream, maps, p);
  } else {
    if (p.N == 16) launch_instance<16, false>(grid, stream, maps, p);
    else if (p.N == 32) launch_instance<32, false>(grid, stream, maps, p);
    else launch_instance<64, false>(grid, stream, maps, p);
  }
}

}  // namespace ntfg
