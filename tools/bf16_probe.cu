// Checks that bf16 hi/lo planes survive the fp64 round trip used by the
// step-level API: v = hi + lo  ->  split(v) == (hi, lo) bit for bit.
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
__global__ void k(int n, int* bad_dbl, int* bad_flt, unsigned seed) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned s = seed ^ (i * 2654435761u);
  s = s * 1664525u + 1013904223u;
  float p = 0.001f + float(s >> 8) / float(1u << 24) * 100.f;
  __nv_bfloat16 h = __float2bfloat16_rn(p);
  __nv_bfloat16 l = __float2bfloat16_rn(p - __bfloat162float(h));
  double v = double(__bfloat162float(h)) + double(__bfloat162float(l));
  __nv_bfloat16 h2 = __double2bfloat16(v);
  __nv_bfloat16 l2 = __double2bfloat16(v - double(__bfloat162float(h2)));
  if (__bfloat16_as_ushort(h2) != __bfloat16_as_ushort(h) || __bfloat16_as_ushort(l2) != __bfloat16_as_ushort(l)) atomicAdd(bad_dbl, 1);
  float f = float(v);
  __nv_bfloat16 h3 = __float2bfloat16_rn(f);
  __nv_bfloat16 l3 = __float2bfloat16_rn(f - __bfloat162float(h3));
  if (__bfloat16_as_ushort(h3) != __bfloat16_as_ushort(h) || __bfloat16_as_ushort(l3) != __bfloat16_as_ushort(l)) atomicAdd(bad_flt, 1);
}
int main() {
  int *d; cudaMalloc(&d, 8); cudaMemset(d, 0, 8);
  int n = 1 << 24;
  k<<<n / 256, 256>>>(n, d, d + 1, 12345u);
  int h[2]; cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("bad double-path %d float-path %d of %d\n", h[0], h[1], n);
  return 0;
}
