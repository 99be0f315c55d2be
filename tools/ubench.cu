// Microbenchmarks that decide the design of the CP streaming passes on B200:
//   1. FFMA (3-register form) vs FFMA2 (packed) vs DFMA issue throughput,
//   2. streaming read bandwidth with 64/128-bit loads,
//   3. the "thread owns k, broadcast row-vector" accumulation loop used by
//      the contraction kernel (R = 32, two k per thread), scalar vs packed.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench ubench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int CH>
__global__ void ffma_kernel(float* out, int iters, float a, float b) {
  float acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3f + c;
  float m = a, n = b + threadIdx.x * 1e-7f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fmaf(acc[c], m, n);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.f) out[threadIdx.x] = s;
}

template <int CH>
__global__ void ffma2_kernel(float* out, int iters, float a, float b) {
  float2 acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = make_float2(threadIdx.x * 1e-3f + c, c * 0.5f);
  float2 m = make_float2(a, a), n = make_float2(b + threadIdx.x * 1e-7f, b);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = __ffma2_rn(acc[c], m, n);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c].x + acc[c].y;
  if (s == 12345.f) out[threadIdx.x] = s;
}

template <int CH>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  double m = a, n = b + threadIdx.x * 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], m, n);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void read64_kernel(const float2* __restrict__ p, size_t n, float* out) {
  float s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float2 v = __ldg(p + i);
    s += v.x + v.y;
  }
  if (s == 12345.f) out[0] = s;
}

__global__ void read128_kernel(const float4* __restrict__ p, size_t n, float* out) {
  float s = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    float4 v0 = __ldg(p + i), v1 = __ldg(p + i + stride), v2 = __ldg(p + i + 2 * stride), v3 = __ldg(p + i + 3 * stride);
    s += v0.x + v1.y + v2.z + v3.w;
  }
  for (; i < n; i += stride) { float4 v = __ldg(p + i); s += v.x; }
  if (s == 12345.f) out[0] = s;
}

// rows x K row-major fp32 stream; each thread owns two consecutive k and
// accumulates G[k][r] += S[row][k] * M[row][r] with M broadcast from smem.
template <int R, bool PACKED>
__global__ void __launch_bounds__(256) gacc_kernel(const float* __restrict__ S, int rows, int K,
                                                   const float* __restrict__ M, float* out) {
  __shared__ __align__(16) float sm[16][R];
  const int k0 = 2 * threadIdx.x;
  float2 g[R];
#pragma unroll
  for (int r = 0; r < R; ++r) g[r] = make_float2(0.f, 0.f);
  const int rows_per_block = (rows + gridDim.x - 1) / gridDim.x;
  const int rbeg = blockIdx.x * rows_per_block;
  const int rend = min(rows, rbeg + rows_per_block);
  for (int rb = rbeg; rb < rend; rb += 16) {
    __syncthreads();
    for (int t = threadIdx.x; t < 16 * R; t += blockDim.x) {
      int rr = t / R, r = t % R;
      sm[rr][r] = (rb + rr < rend) ? M[(size_t)(rb + rr) * R + r] : 0.f;
    }
    __syncthreads();
    float2 sv[16];
#pragma unroll
    for (int rr = 0; rr < 16; ++rr) {
      int row = min(rb + rr, rend - 1);
      sv[rr] = *reinterpret_cast<const float2*>(S + (size_t)row * K + k0);
    }
#pragma unroll
    for (int rr = 0; rr < 16; ++rr) {
#pragma unroll
      for (int r = 0; r < R; r += 4) {
        float4 m4 = *reinterpret_cast<const float4*>(&sm[rr][r]);
        if (PACKED) {
          g[r + 0] = __ffma2_rn(sv[rr], make_float2(m4.x, m4.x), g[r + 0]);
          g[r + 1] = __ffma2_rn(sv[rr], make_float2(m4.y, m4.y), g[r + 1]);
          g[r + 2] = __ffma2_rn(sv[rr], make_float2(m4.z, m4.z), g[r + 2]);
          g[r + 3] = __ffma2_rn(sv[rr], make_float2(m4.w, m4.w), g[r + 3]);
        } else {
          g[r + 0].x = fmaf(sv[rr].x, m4.x, g[r + 0].x); g[r + 0].y = fmaf(sv[rr].y, m4.x, g[r + 0].y);
          g[r + 1].x = fmaf(sv[rr].x, m4.y, g[r + 1].x); g[r + 1].y = fmaf(sv[rr].y, m4.y, g[r + 1].y);
          g[r + 2].x = fmaf(sv[rr].x, m4.z, g[r + 2].x); g[r + 2].y = fmaf(sv[rr].y, m4.z, g[r + 2].y);
          g[r + 3].x = fmaf(sv[rr].x, m4.w, g[r + 3].x); g[r + 3].y = fmaf(sv[rr].y, m4.w, g[r + 3].y);
        }
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) s += g[r].x + g[r].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  printf("device %s SMs %d clock %d kHz\n", prop.name, prop.multiProcessorCount, prop.clockRate);
  const int sms = prop.multiProcessorCount;
  float* outf; double* outd; CK(cudaMalloc(&outf, 1 << 24)); CK(cudaMalloc(&outd, 1 << 24));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  const int iters = 4096, threads = 256, blocks = sms * 8;
  auto rate = [&](double ops, float ms_) { return ops / (ms_ * 1e-3) / 1e12; };
  for (int rep = 0; rep < 2; ++rep) {
    ffma_kernel<8><<<blocks, threads>>>(outf, iters, 0.999f, 1e-3f);
    CK(cudaEventRecord(e0)); ffma_kernel<8><<<blocks, threads>>>(outf, iters, 0.999f, 1e-3f); CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA  : %.1f T FMA/s (%.3f ms)\n", rate((double)blocks * threads * iters * 8, ms), ms);
    ffma2_kernel<8><<<blocks, threads>>>(outf, iters, 0.999f, 1e-3f);
    CK(cudaEventRecord(e0)); ffma2_kernel<8><<<blocks, threads>>>(outf, iters, 0.999f, 1e-3f); CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA2 : %.1f T FMA/s (%.3f ms)\n", rate((double)blocks * threads * iters * 16, ms), ms);
    dfma_kernel<8><<<blocks, threads>>>(outd, iters / 4, 0.999, 1e-3);
    CK(cudaEventRecord(e0)); dfma_kernel<8><<<blocks, threads>>>(outd, iters / 4, 0.999, 1e-3); CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA  : %.2f T FMA/s (%.3f ms)\n", rate((double)blocks * threads * (iters / 4) * 8, ms), ms);
  }
  size_t bytes = size_t(2) << 30;
  float* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 0, bytes));
  for (int rep = 0; rep < 3; ++rep) {
    CK(cudaEventRecord(e0)); read64_kernel<<<sms * 8, 256>>>((const float2*)buf, bytes / 8, outf); CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("read64 : %.0f GB/s\n", bytes / (ms * 1e-3) / 1e9);
    CK(cudaEventRecord(e0)); read128_kernel<<<sms * 8, 256>>>((const float4*)buf, bytes / 16, outf); CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("read128: %.0f GB/s\n", bytes / (ms * 1e-3) / 1e9);
  }
  // G-accumulation loop: 512 x 512 rows, K = 512 (one C2 mode pass, one stream)
  const int rows = 262144, K = 512, R = 32;
  float* M; CK(cudaMalloc(&M, (size_t)rows * R * 4)); CK(cudaMemset(M, 0, (size_t)rows * R * 4));
  for (int grid : {sms, sms * 2, sms * 4}) {
    for (int rep = 0; rep < 2; ++rep) {
      gacc_kernel<32, false><<<grid, 256>>>(buf, rows, K, M, outf);
      CK(cudaEventRecord(e0)); gacc_kernel<32, false><<<grid, 256>>>(buf, rows, K, M, outf); CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      double ent = (double)rows * K;
      printf("gacc scalar grid %d: %.3f ms, %.0f GB/s, %.1f T FMA/s\n", grid, ms, ent * 4 / (ms * 1e-3) / 1e9, rate(ent * R, ms));
      gacc_kernel<32, true><<<grid, 256>>>(buf, rows, K, M, outf);
      CK(cudaEventRecord(e0)); gacc_kernel<32, true><<<grid, 256>>>(buf, rows, K, M, outf); CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      printf("gacc packed grid %d: %.3f ms, %.0f GB/s, %.1f T FMA/s\n", grid, ms, ent * 4 / (ms * 1e-3) / 1e9, rate(ent * R, ms));
    }
  }
  CK(cudaDeviceSynchronize());
  printf("done\n");
  return 0;
}
