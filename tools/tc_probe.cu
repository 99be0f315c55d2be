// Probe: one tcgen05.mma (kind::f16, bf16 inputs, fp32 accumulate in TMEM)
// with A = a TMA-loaded MN-major SWIZZLE_128B tile and B = a hand-written
// K-major no-swizzle tile, D = A(128 x 16) * B(16 x 32) -> compare to CPU.
// Validates the descriptor encodings used by tc_contract.cuh.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2602_14683_b200/csrc/tc_common.cuh"

using namespace ntfg;

constexpr int ROWS = 16, KCOLS = 512, N = 32;

__global__ void probe_kernel(const __grid_constant__ CUtensorMap tmap, const float* bmat /*[16][32]*/, int mtile,
                             float* out /*[128][32]*/) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* a_tile = smem;                 // 16 rows x 512 k bf16 = 16KB, 8 ko blocks of 2KB
  unsigned char* b_tile = smem + 16384;         // 1KB
  __shared__ uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  if (tid == 0) {
    tc::mbar_init(&bar_tma, 1);
    tc::mbar_init(&bar_mma, 1);
  }
  tc::fence_barrier_init();
  __syncthreads();
  if (warp == 0) tc::tmem_alloc(&tmem_base, 64);
  // B tile: element (n, k) at (n/8)*256 + (k/8)*128 + (n%8)*16 + (k%8)*2
  for (int idx = tid; idx < N * ROWS; idx += blockDim.x) {
    const int n = idx / ROWS, k = idx % ROWS;
    __nv_bfloat16 v = __float2bfloat16_rn(bmat[k * N + n]);
    *reinterpret_cast<__nv_bfloat16*>(b_tile + (n / 8) * 256 + (k / 8) * 128 + (n % 8) * 16 + (k % 8) * 2) = v;
  }
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    tc::expect_tx(&bar_tma, ROWS * KCOLS * 2);
    for (int ko = 0; ko < KCOLS / 64; ++ko) tc::tma_load_5d(a_tile + ko * 2048, &tmap, 0, ko, 0, 0, 0, &bar_tma);
    tc::wait(&bar_tma, 0);
    tc::fence_after_sync();
    const uint64_t adesc = tc::desc_mn_sw128(a_tile + mtile * 2 * 2048, 2048, 1024);
    const uint64_t bdesc = tc::desc_k_interleave(b_tile, 128, 256);
    tc::mma_bf16(tmem, adesc, bdesc, tc::idesc_bf16_f32(128, N, true, false), false);
    tc::commit(&bar_mma);
  }
  __syncwarp();
  tc::wait(&bar_mma, 0);
  tc::fence_after_sync();
  if (warp < 4) {
    uint32_t r[32];
    tc::tmem_ld32(tmem + ((warp * 32) << 16), r);
    for (int c = 0; c < 32; ++c) out[(warp * 32 + (tid % 32)) * N + c] = __uint_as_float(r[c]);
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 64);
}

int main() {
  std::vector<float> a(ROWS * KCOLS), b(ROWS * N);
  for (int i = 0; i < ROWS * KCOLS; ++i) a[i] = float((i * 37 % 101) - 50) / 16.0f;
  for (int i = 0; i < ROWS * N; ++i) b[i] = float((i * 13 % 29) - 14) / 8.0f;
  std::vector<__nv_bfloat16> ah(ROWS * KCOLS);
  for (int i = 0; i < ROWS * KCOLS; ++i) ah[i] = __float2bfloat16_rn(a[i]);
  __nv_bfloat16* da;
  float *db, *dout;
  cudaMalloc(&da, ah.size() * 2);
  cudaMalloc(&db, b.size() * 4);
  cudaMalloc(&dout, 128 * N * 4);
  cudaMemcpy(da, ah.data(), ah.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap tmap;
  if (!tc::make_plane_map(&tmap, da, KCOLS, ROWS, 1, 1, 16, 1)) { printf("tmap failed\n"); return 1; }
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  int worst = 0;
  for (int mtile = 0; mtile < 4; ++mtile) {
    probe_kernel<<<1, 128, 32768>>>(tmap, db, mtile, dout);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<float> out(128 * N);
    cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    double maxerr = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < ROWS; ++k)
          ref += double(__bfloat162float(ah[k * KCOLS + mtile * 128 + m])) *
                 double(__bfloat162float(__float2bfloat16_rn(b[k * N + n])));
        const double err = std::fabs(ref - out[m * N + n]);
        maxerr = std::max(maxerr, err);
        if (err > 1e-3 * (1 + std::fabs(ref))) {
          if (bad < 5) printf("mtile %d m %d n %d got %f want %f\n", mtile, m, n, out[m * N + n], ref);
          ++bad;
        }
      }
    printf("mtile %d: bad %d maxerr %g\n", mtile, bad, maxerr);
    worst += bad;
  }
  printf(worst == 0 ? "PROBE PASS\n" : "PROBE FAIL\n");
  return worst == 0 ? 0 : 1;
}
