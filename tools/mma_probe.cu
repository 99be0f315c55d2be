// Probe: issue cost of tcgen05.mma as a function of how often the accumulator
// tile D changes between consecutive instructions (K3 cycles 4-8 accumulators
// per 16-row stage, 3 MMAs each).  One CTA, one issuing thread, zeroed smem.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_probe tools/mma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include "../paper_2602_14683_b200/csrc/tc_common.cuh"
using namespace ntfg;

struct Cfg {
  int kind;    // 0 bf16 (K = 16), 1 tf32 (K = 8)
  int N;       // UMMA N
  int a_mn;    // A MN-major SW128 (K3) or K-major interleave
  int ntile;   // distinct accumulators cycled
  int per_d;   // consecutive MMAs per accumulator before switching
  int count;   // total MMAs
  int same_ab; // 1: every MMA uses the same A/B descriptors
};

__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, bool acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(uint32_t(acc)));
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n" : "=r"(pred));
  return pred != 0;
}

template <bool CONV>
__global__ void probe(Cfg c, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) tc::mbar_init(&bar, 1);
  tc::fence_barrier_init();
  tc::fence_proxy_async();
  if (threadIdx.x < 32) tc::tmem_alloc(&tmem_base, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (CONV ? threadIdx.x < 32 : threadIdx.x == 0) {
    const uint32_t tmem = CONV ? __shfl_sync(0xffffffffu, tmem_base, 0) : tmem_base;
    uint32_t idesc;
    if (c.kind == 0) idesc = tc::idesc_bf16_f32(128, c.N, c.a_mn, false);
    else idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(c.N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    unsigned char* a0 = smem;
    unsigned char* a1 = smem + 16384;
    unsigned char* b0 = smem + 32768;
    unsigned char* b1 = smem + 49152;
    uint64_t ad[2], bd[2];
    if (c.a_mn) {
      ad[0] = tc::desc_mn_sw128(a0, 2048, 1024);
      ad[1] = tc::desc_mn_sw128(a1, 2048, 1024);
    } else {
      ad[0] = tc::desc_k_interleave(a0, 128, 256);
      ad[1] = tc::desc_k_interleave(a1, 128, 256);
    }
    bd[0] = tc::desc_k_interleave(b0, 128, 272);
    bd[1] = tc::desc_k_interleave(b1, 128, 272);
    for (int rep = 0; rep < 2; ++rep) {  // rep 0 warms up
      const unsigned long long t0 = clock64();
      int i = 0;
      while (i < c.count) {
        for (int t = 0; t < c.ntile; ++t) {
          const uint32_t d = tmem + uint32_t(t * c.N);
          int k3 = 0;
          for (int k = 0; k < c.per_d; ++k, ++i) {
            const int ai = c.same_ab ? 0 : (k3 == 2);
            const int bi = c.same_ab ? 0 : (k3 == 1);
            k3 = k3 == 2 ? 0 : k3 + 1;
            const bool acc = i >= c.ntile * c.per_d;
            if (!CONV || elect_one()) {
              if (c.kind == 0) tc::mma_bf16(d, ad[ai], bd[bi], idesc, acc);
              else mma_tf32(d, ad[ai], bd[bi], idesc, acc);
            }
          }
        }
      }
      const unsigned long long t1 = clock64();
      if (!CONV || elect_one()) tc::commit(&bar);
      tc::wait(&bar, rep & 1);
      const unsigned long long t2 = clock64();
      if (threadIdx.x == 0) {
        out[rep * 2] = t1 - t0;
        out[rep * 2 + 1] = t2 - t0;
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tmem_base, 512);
}


// straight-line: UNR back-to-back MMAs on one accumulator (or alternating two), uniform operands
template <int UNR, int ND>
__global__ void probe2(int kind, int N, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) tc::mbar_init(&bar, 1);
  tc::fence_barrier_init();
  tc::fence_proxy_async();
  if (threadIdx.x < 32) tc::tmem_alloc(&tmem_base, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (threadIdx.x < 32) {
    const uint32_t tmem = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint32_t idesc = kind == 0 ? tc::idesc_bf16_f32(128, N, true, false)
                                     : ((1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24));
    const uint64_t ad = kind == 0 ? tc::desc_mn_sw128(smem, 2048, 1024) : tc::desc_k_interleave(smem, 128, 256);
    const uint64_t bd = tc::desc_k_interleave(smem + 32768, 128, 272);
    for (int rep = 0; rep < 2; ++rep) {
      const unsigned long long t0 = clock64();
      for (int it = 0; it < 40; ++it) {
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < UNR; ++k) {
            const uint32_t d = tmem + uint32_t((k % ND) * N);
            if (kind == 0) tc::mma_bf16(d, ad, bd, idesc, true);
            else mma_tf32(d, ad, bd, idesc, true);
          }
        }
        __syncwarp();
      }
      const unsigned long long t1 = clock64();
      if (elect_one()) tc::commit(&bar);
      tc::wait(&bar, rep & 1);
      const unsigned long long t2 = clock64();
      if (threadIdx.x == 0) {
        out[rep * 2] = t1 - t0;
        out[rep * 2 + 1] = t2 - t0;
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tmem_base, 512);
}

template <int UNR, int ND>
void run2(int kind, int N, unsigned long long* d) {
  cudaFuncSetAttribute(probe2<UNR, ND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  probe2<UNR, ND><<<1, 128, 100 * 1024>>>(kind, N, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error: %s\n", cudaGetErrorString(e)); exit(1); }
  unsigned long long h[4];
  cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("straight %s N=%3d unroll=%d nd=%d | issue %7.1f | complete %7.1f clk/MMA\n", kind ? "tf32" : "bf16", N, UNR, ND,
         double(h[2]) / (40 * UNR), double(h[3]) / (40 * UNR));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  cudaFuncSetAttribute(probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const Cfg cfgs[] = {
      // kind N a_mn ntile per_d count same
      {0, 64, 1, 1, 1, 960, 1},   {0, 64, 1, 1, 1, 960, 0},   {0, 64, 1, 4, 1, 960, 0},  {0, 64, 1, 4, 3, 960, 0},
      {0, 64, 1, 4, 6, 960, 0},   {0, 64, 1, 4, 12, 960, 0},  {0, 64, 1, 4, 24, 960, 0}, {0, 64, 1, 2, 3, 960, 0},
      {0, 64, 0, 1, 1, 960, 0},   {0, 64, 0, 4, 3, 960, 0},   {0, 64, 0, 4, 12, 960, 0},
      {0, 32, 1, 1, 1, 960, 0},   {0, 32, 1, 8, 3, 960, 0},   {0, 32, 1, 8, 6, 960, 0},  {0, 32, 1, 8, 12, 960, 0},
      {0, 32, 1, 4, 3, 960, 0},   {0, 128, 1, 1, 1, 960, 0},  {0, 128, 1, 2, 3, 960, 0}, {0, 128, 1, 2, 12, 960, 0},
      {0, 256, 1, 1, 1, 960, 0},  {0, 256, 1, 2, 3, 960, 0},
      {1, 128, 0, 1, 1, 960, 0},  {1, 128, 0, 2, 24, 960, 0}, {1, 128, 0, 2, 12, 960, 0}, {1, 64, 0, 1, 1, 960, 0},
      {1, 256, 0, 1, 1, 960, 0},
  };
  for (int kind = 0; kind < 2; ++kind)
    for (int N : {32, 64, 128, 256}) {
      run2<24, 1>(kind, N, d);
      run2<24, 2>(kind, N, d);
      if (N <= 128) run2<24, 4>(kind, N, d);
    }
  if (getenv("PROBE_SHORT")) return 0;
  printf("kind N a_mn ntile per_d same | issue clk/MMA | complete clk/MMA\n");
  for (int conv = 0; conv < 2; ++conv)
  for (const Cfg& c : cfgs) {
    if (conv) probe<true><<<1, 128, 100 * 1024>>>(c, d);
    else probe<false><<<1, 128, 100 * 1024>>>(c, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error: %s\n", cudaGetErrorString(e));
      return 1;
    }
    unsigned long long h[4];
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("conv=%d %s N=%3d a_mn=%d ntile=%d per_d=%2d same=%d | %7.1f | %7.1f\n", conv, c.kind ? "tf32" : "bf16", c.N, c.a_mn,
           c.ntile, c.per_d, c.same_ab, double(h[2]) / c.count, double(h[3]) / c.count);
  }
  return 0;
}
