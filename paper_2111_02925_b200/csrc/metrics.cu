// libsz3g -- distortion metrics of a reconstruction (NEXT-3): "The bit rate equals
// bits/cr ... PSNR is inversely proportional to the mean square error of decompress data and original
// data in logarithmic scale"; SPEC S:545 PSNR = 20 log10(range) - 10 log10(MSE).  One read of x and x'
// gives max |x - x'|, sum (x - x')^2 (fp64) and the number of elements above a bound; the caller forms
// MSE, PSNR (with the value range of x, e.g. from sz3g_regression_analyze), ratio and bit rate.
// Elements whose x and x' are bitwise identical contribute 0 (so preserved NaN / Inf outliers count as
// exact); otherwise the fp64 difference is used as is.  Deterministic: per-CTA partials in a fixed
// grid, reduced in a fixed order by a second 1-CTA kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>

#include "../../include/sz3g.h"
#include "ptx.cuh"

namespace {

std::atomic<uint64_t> g_me_launches{0};
constexpr int ME_T = 256;

template <typename T>
struct Bits;
template <>
struct Bits<float> { using type = uint32_t; };
template <>
struct Bits<double> { using type = uint64_t; };

template <typename T>
__device__ __forceinline__ void acc(T a, T b, double eb, double& mx, double& sq, double& cnt) {
  using B = typename Bits<T>::type;
  B ba, bb;
  memcpy(&ba, &a, sizeof(T));
  memcpy(&bb, &b, sizeof(T));
  if (ba == bb) return;
  const double d = (double)a - (double)b;
  const double ad = fabs(d);
  mx = (ad > mx || ad != ad) ? ad : mx;   // NaN sticks
  sq += d * d;
  cnt += (ad > eb || ad != ad) ? 1.0 : 0.0;
}

template <typename T>
__global__ void __launch_bounds__(ME_T) k_error_partials(const T* __restrict__ x, const T* __restrict__ y, uint64_t n,
                                                         double eb, double* __restrict__ part) {
  double mx = 0.0, sq = 0.0, cnt = 0.0;
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  constexpr int V = 16 / sizeof(T);
  const bool al = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;
  uint64_t done = 0;
  if (al) {
    const uint4* xv = reinterpret_cast<const uint4*>(x);
    const uint4* yv = reinterpret_cast<const uint4*>(y);
    const uint64_t nv = n / V;
    for (uint64_t v = tid; v < nv; v += nth) {
      const uint4 a = __ldcs(xv + v), b = __ldcs(yv + v);
      const T* pa = reinterpret_cast<const T*>(&a);
      const T* pb = reinterpret_cast<const T*>(&b);
#pragma unroll
      for (int c = 0; c < V; c++) acc<T>(pa[c], pb[c], eb, mx, sq, cnt);
    }
    done = nv * V;
  }
  for (uint64_t e = done + tid; e < n; e += nth) acc<T>(x[e], y[e], eb, mx, sq, cnt);
  // block reduction in a fixed order
  __shared__ double s[3][ME_T / 32];
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double m2 = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = (m2 > mx || m2 != m2) ? m2 : mx;
    sq += __shfl_xor_sync(0xffffffffu, sq, o);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { s[0][w] = mx; s[1][w] = sq; s[2][w] = cnt; }
  SZ3G_SYNCTHREADS();
  if (threadIdx.x == 0) {
    for (int i = 1; i < ME_T / 32; i++) {
      mx = (s[0][i] > mx || s[0][i] != s[0][i]) ? s[0][i] : mx;
      sq += s[1][i];
      cnt += s[2][i];
    }
    part[3 * blockIdx.x] = mx;
    part[3 * blockIdx.x + 1] = sq;
    part[3 * blockIdx.x + 2] = cnt;
  }
}

__global__ void k_error_final(const double* __restrict__ part, uint32_t nb, double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  double mx = 0.0, sq = 0.0, cnt = 0.0;
  for (uint32_t i = 0; i < nb; i++) {
    mx = (part[3 * i] > mx || part[3 * i] != part[3 * i]) ? part[3 * i] : mx;
    sq += part[3 * i + 1];
    cnt += part[3 * i + 2];
  }
  out[0] = mx;
  out[1] = sq;
  out[2] = cnt;
}

uint32_t me_blocks(uint64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((n + 4095) / 4096, (uint64_t)sms * 4));
}

}  // namespace

uint64_t sz3g_metrics_launch_count_internal() { return g_me_launches.load(); }

extern "C" {

uint64_t sz3g_error_stats_scratch_bytes(uint64_t n) { return 3ull * 8 * me_blocks(n); }

int sz3g_error_stats(const sz3g_grid* grid, const void* x, const void* y, double eb, double* d_out, void* scratch,
                     sz3g_stream_t stream) {
  if (!grid || !d_out || !scratch) return SZ3G_EINVAL;
  if (grid->dtype != SZ3G_F32 && grid->dtype != SZ3G_F64) return SZ3G_EUNSUPPORTED;
  const uint64_t n = grid->dims[0] * grid->dims[1] * grid->dims[2];
  if (n > 0 && (!x || !y)) return SZ3G_EINVAL;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const uint32_t nb = me_blocks(n);
  double* part = static_cast<double*>(scratch);
  if (n == 0) {
    cudaMemsetAsync(d_out, 0, 3 * sizeof(double), st);
  } else {
    if (grid->dtype == SZ3G_F32)
      k_error_partials<float><<<nb, ME_T, 0, st>>>((const float*)x, (const float*)y, n, eb, part);
    else
      k_error_partials<double><<<nb, ME_T, 0, st>>>((const double*)x, (const double*)y, n, eb, part);
    k_error_final<<<1, 32, 0, st>>>(part, nb, d_out);
  }
  if (cudaGetLastError() != cudaSuccess) return SZ3G_ECUDA;
  g_me_launches.fetch_add(n == 0 ? 0 : 2, std::memory_order_relaxed);
  return SZ3G_OK;
}

}  // extern "C"
