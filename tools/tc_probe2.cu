// Probe 2: can one TMA box land a whole 16-row x 512-column bf16 stage in the
// canonical MN-major SW128 layout ([ko][row][64]) using a tensor map whose
// dims are (k_inner, rows, k_outer) with strides (K*2 bytes, 128 bytes)?
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "../paper_2602_14683_b200/csrc/tc_common.cuh"
using namespace ntfg;
constexpr int ROWS = 16, KC = 512;
__global__ void k3(const __grid_constant__ CUtensorMap tmap, unsigned short* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); }
  tc::fence_barrier_init();
  __syncthreads();
  if (threadIdx.x == 0) {
    tc::expect_tx(&bar, ROWS * KC * 2);
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
                 :: "r"(tc::saddr(smem)), "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(0), "r"(0), "r"(0), "r"(tc::saddr(&bar)) : "memory");
  }
  tc::wait(&bar, 0);
  for (int i = threadIdx.x; i < ROWS * KC; i += blockDim.x) out[i] = reinterpret_cast<unsigned short*>(smem)[i];
}
int main() {
  std::vector<unsigned short> a(ROWS * KC);
  for (int i = 0; i < ROWS * KC; ++i) a[i] = (unsigned short)i;
  unsigned short *da, *dout;
  cudaMalloc(&da, a.size() * 2); cudaMalloc(&dout, a.size() * 2);
  cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice);
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap map;
  const cuuint64_t dims[3] = {64, ROWS, KC / 64};
  const cuuint64_t strides[2] = {KC * 2, 128};
  const cuuint32_t box[3] = {64, ROWS, KC / 64};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = ((Encode)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, da, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode (non-monotonic strides) -> %d\n", int(r));
  if (r != CUDA_SUCCESS) return 0;
  cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
  k3<<<1, 128, 20000>>>(map, dout);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<unsigned short> o(a.size());
  cudaMemcpy(o.data(), dout, o.size() * 2, cudaMemcpyDeviceToHost);
  // expected canonical: smem [ko][row][ki] with 128B swizzle: chunk (16B) index xor (row % 8)
  int bad = 0;
  for (int ko = 0; ko < KC / 64; ++ko)
    for (int row = 0; row < ROWS; ++row)
      for (int ki = 0; ki < 64; ++ki) {
        const int chunk = ki / 8, within = ki % 8;
        const int sidx = (ko * ROWS + row) * 64 + ((chunk ^ (row % 8)) * 8) + within;
        if (o[sidx] != a[row * KC + ko * 64 + ki]) ++bad;
      }
  printf("layout mismatches %d of %d -> %s\n", bad, ROWS * KC, bad ? "FAIL" : "PASS");
  return 0;
}
