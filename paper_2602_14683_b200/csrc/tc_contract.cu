// K3 on the tensor cores: the tcgen05/TMEM/TMA contraction kernel
// (tc_contract.cuh) compiled as its own translation unit.
#define NTFG_TC_CONTRACT_IMPL
#include "tc_contract.cuh"

#include <algorithm>
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

// One staging launch per contraction: blocks [0, nb32) write the fp32 zero-padded copies of every
// factor of every stream ([I_m][R] fp64 -> [I_m][N] fp32: B-operand gathers, the case-B epilogue's last
// factor, the epilogue's run scales); blocks [nb32, ...) build, straight from the fp64 factor, the bf16
// hi/lo B tiles of every 16-row block of the fastest off-mode in the K-major core-matrix layout the MMA
// reads (same offsets as the generic path's producer stores; float(x) is the value the fp32 copy holds).
struct BtStage {
  const double* src[2];
  int ns, runst, N, R;
  uint32_t b_tile;
  unsigned char* out;
};
static __global__ void stage_factors_kernel(const F32Stage a, const int nb32, const BtStage b) {
  if (int(blockIdx.x) < nb32) {
    const int64_t tot = a.off[a.order];
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < tot * a.ns; i += int64_t(nb32) * blockDim.x) {
      const int s = int(i / tot);
      const int64_t e = i - s * tot;
      int m = 0;
      while (e >= a.off[m + 1]) ++m;
      const int64_t l = e - a.off[m];
      const int64_t row = l / a.N;
      const int r = int(l - row * a.N);
      a.dst[s][m][l] = r < a.R ? float(a.src[s][m][row * a.R + r]) : 0.f;
    }
    return;
  }
  const int nbt = int(gridDim.x) - nb32;
  const int total = b.ns * b.runst * 2 * b.N;
  for (int i = (int(blockIdx.x) - nb32) * blockDim.x + threadIdx.x; i < total; i += nbt * blockDim.x) {
    const int r = i % b.N, kg = (i / b.N) & 1, blk = (i / (2 * b.N)) % b.runst, s = i / (2 * b.N * b.runst);
    const double* f = b.src[s] + size_t(blk * 16 + kg * 8) * b.R + r;
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = r < b.R ? float(f[size_t(e) * b.R]) : 0.f;
    uint32_t h[4], l[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) bf16_split_pair_fast(v[2 * e], v[2 * e + 1], h[e], l[e]);
    unsigned char* tile = b.out + size_t((s * b.runst + blk) * 2) * b.b_tile;
    const uint32_t off = uint32_t(r / 8) * kTcBSbo + uint32_t(kg) * 128 + uint32_t(r % 8) * 16;
    *reinterpret_cast<uint4*>(tile + off) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(tile + b.b_tile + off) = make_uint4(l[0], l[1], l[2], l[3]);
  }
}

void tc_contract_launch(int grid, cudaStream_t stream, const TcMaps& maps, const TcParams& pin, const F32Stage& fs) {
  TcParams p = pin;
  // static B tiles (tc_contract.cuh, TcParams::sb): fast-gather shapes whose runs of the fastest
  // off-mode are at least 8 stages long (shorter runs would mean a segment drain every few stages)
  // (at N <= 32 the producer warps kept up, so the gain there is only the saved SM work: C2 step
  // 317 -> 322 outer it/s on the same box; at N = 64 it removes the bottleneck)
  static const bool sb_off = [] { const char* e = std::getenv("NTFG_TC_STATIC_B"); return e && e[0] == '0'; }();
  p.sb = 0;
  p.sb_runst = 0;
  BtStage bt{};
  int nbt = 0;
  if (!sb_off && p.gfast && p.btiles && p.fmode >= 0 && !p.ablate) {
    const int64_t If = p.g.dims[p.fmode];
    if (If % kTcRows == 0 && If / kTcRows >= 8) {
      p.sb = 1;
      p.sb_runst = int(If / kTcRows);
      bt.src[0] = p.mfac[0][p.fmode];
      bt.src[1] = p.mfac[p.ns > 1 ? 1 : 0][p.fmode];
      bt.ns = p.ns;
      bt.runst = p.sb_runst;
      bt.N = p.N;
      bt.R = p.R;
      bt.b_tile = p.lay.b_tile;
      bt.out = p.btiles;
      nbt = (p.ns * p.sb_runst * 2 * p.N + 255) / 256;
    }
  }
  const int64_t n32 = fs.off[fs.order] * fs.ns;
  const int nb32 = int(std::min<int64_t>((n32 + 255) / 256, 1024));
  stage_factors_kernel<<<nb32 + nbt, 256, 0, stream>>>(fs, nb32, bt);
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
