// Achievable HBM bandwidth for the hot kernels' traffic mixes at the c5 size (4 Gi elements): plain
// grid-stride streaming kernels, 16-byte accesses, two iterations in flight per thread.
//   u16 -> f32  read 2 B, write 4 B per element (the decompressor's mix, 1:2)
//   f32 -> u16  read 4 B, write 2 B per element (the quantiser's mix, 2:1)
//   f32 copy    1:1 (the MEASURED_PEAKS.json recipe)
// Prints one JSON line: GB/s of read + write bytes, best and median of the repetitions.
#include <cstdio>
#include <cstdint>
#include <algorithm>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s: %s\n",#x,cudaGetErrorString(e)); return 1;}}while(0)

__global__ void k_u16_f32(const uint4* __restrict__ a, float4* __restrict__ b, size_t n8) {
  const size_t st = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n8; i += st) {
    const uint4 v = __ldcs(a + i);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    float f[8];
#pragma unroll
    for (int k = 0; k < 4; k++) { f[2 * k] = (float)(w[k] & 0xffffu); f[2 * k + 1] = (float)(w[k] >> 16); }
    __stcs(b + 2 * i, make_float4(f[0], f[1], f[2], f[3]));
    __stcs(b + 2 * i + 1, make_float4(f[4], f[5], f[6], f[7]));
  }
}
__global__ void k_f32_u16(const float4* __restrict__ a, uint4* __restrict__ b, size_t n8) {
  const size_t st = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n8; i += st) {
    const float4 p = __ldcs(a + 2 * i), q = __ldcs(a + 2 * i + 1);
    const float f[8] = {p.x, p.y, p.z, p.w, q.x, q.y, q.z, q.w};
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; k++) w[k] = ((uint32_t)f[2 * k] & 0xffffu) | ((uint32_t)f[2 * k + 1] << 16);
    __stcs(b + i, make_uint4(w[0], w[1], w[2], w[3]));
  }
}
__global__ void k_copy4(const float4* __restrict__ a, float4* __restrict__ b, size_t n4) {
  const size_t st = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += st) __stcs(b + i, __ldcs(a + i));
}
template <class F> void timeit(F f, int reps, float& best, float& med) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 3; w++) f();
  std::vector<float> t;
  for (int r = 0; r < reps; r++) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); t.push_back(ms);
  }
  std::sort(t.begin(), t.end()); best = t[0]; med = t[t.size() / 2];
}
int main() {
  int sms = 148; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t n = (size_t)1024 * 2048 * 2048, n8 = n / 8;
  void *x, *y;
  CK(cudaMalloc(&x, n * 4)); CK(cudaMalloc(&y, n * 4));
  CK(cudaMemset(x, 0, n * 4)); CK(cudaMemset(y, 0, n * 4));
  const int blocks = sms * 8, thr = 256, reps = 10;
  float b1, m1, b2, m2, b3, m3;
  timeit([&] { k_u16_f32<<<blocks, thr>>>((const uint4*)x, (float4*)y, n8); }, reps, b1, m1);
  timeit([&] { k_f32_u16<<<blocks, thr>>>((const float4*)y, (uint4*)x, n8); }, reps, b2, m2);
  timeit([&] { k_copy4<<<blocks, thr>>>((const float4*)x, (float4*)y, n / 4); }, reps, b3, m3);
  CK(cudaDeviceSynchronize());
  const double B = 6.0 * n, C = 8.0 * n;
  printf("{\"n\": %zu, \"u16_to_f32_1to2\": {\"best_gbs\": %.1f, \"median_gbs\": %.1f, \"ms\": %.3f}, "
         "\"f32_to_u16_2to1\": {\"best_gbs\": %.1f, \"median_gbs\": %.1f, \"ms\": %.3f}, "
         "\"copy_f32_1to1\": {\"best_gbs\": %.1f, \"median_gbs\": %.1f, \"ms\": %.3f}}\n",
         n, B / b1 / 1e6, B / m1 / 1e6, m1, B / b2 / 1e6, B / m2 / 1e6, m2, C / b3 / 1e6, C / m3 / 1e6, m3);
  return 0;
}
