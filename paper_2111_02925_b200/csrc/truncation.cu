// libsz3g -- SZ3-Truncation (NEXT-2): "Given the target bytes k as input parameter, it keeps k
// most-significant bytes of each floating-point data while discarding the rest of the bytes"
// (PAPER.md P:848-850).  Definition: oracle/DEFINITION.md T1-T2 -- the stream holds, element after
// element, the k most-significant bytes of the IEEE-754 pattern, most significant first;
// decompression zero-fills the rest.  C ABI: sz3g_truncation_compress / _decompress (include/sz3g.h).
//
// A pure streaming transform (HBM-bound: s + k bytes per element).  One thread owns groups of 16
// consecutive elements: the group's input is 16 s bytes (s/4 x 16-byte loads) and its output exactly
// 16 k bytes (k x 16-byte stores), so every access is a full 16-byte vector for any k.  The byte
// shuffle is done in registers with compile-time indices (K and T are template parameters).  Grid:
// a multiple of the SM count, grid-stride over groups; the tail (n mod 16) goes element by element.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>

#include "../../include/sz3g.h"
#include "ptx.cuh"

namespace {

std::atomic<uint64_t> g_tr_launches{0};

template <int S>
struct Word;
template <>
struct Word<4> { using type = uint32_t; };
template <>
struct Word<8> { using type = uint64_t; };

// 16 elements -> 16 K bytes (4 K words)
template <int S, int K>
__device__ __forceinline__ void pack16(const typename Word<S>::type (&v)[16], uint32_t (&o)[4 * K]) {
#pragma unroll
  for (int w = 0; w < 4 * K; w++) o[w] = 0u;
#pragma unroll
  for (int i = 0; i < 16; i++) {
#pragma unroll
    for (int j = 0; j < K; j++) {
      const int p = i * K + j;
      const uint32_t byte = (uint32_t)(v[i] >> (8 * (S - 1 - j))) & 0xffu;
      o[p >> 2] |= byte << (8 * (p & 3));
    }
  }
}

template <int S, int K>
__device__ __forceinline__ void unpack16(const uint32_t (&o)[4 * K], typename Word<S>::type (&v)[16]) {
  using W = typename Word<S>::type;
#pragma unroll
  for (int i = 0; i < 16; i++) {
    W x = 0;
#pragma unroll
    for (int j = 0; j < K; j++) {
      const int p = i * K + j;
      x |= (W)((o[p >> 2] >> (8 * (p & 3))) & 0xffu) << (8 * (S - 1 - j));
    }
    v[i] = x;
  }
}

template <int S, int K>
__global__ void __launch_bounds__(256) k_trunc_compress(const uint8_t* __restrict__ x, uint64_t n,
                                                        uint8_t* __restrict__ out) {
  using W = typename Word<S>::type;
  const uint64_t ng = n / 16;
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t g = tid; g < ng; g += nth) {
    W v[16];
    const uint4* src = reinterpret_cast<const uint4*>(x + g * 16 * S);
#pragma unroll
    for (int q = 0; q < S; q++) {   // 16 S bytes = S uint4
      const uint4 u = __ldcs(src + q);
      const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int t = 0; t < 4; t++) {
        const int word = 4 * q + t;   // 32-bit word index inside the group
        if constexpr (S == 4) v[word] = (W)w4[t];
        else if (word & 1) v[word >> 1] |= (W)w4[t] << 32;
        else v[word >> 1] = (W)w4[t];
      }
    }
    uint32_t o[4 * K];
    pack16<S, K>(v, o);
    uint4* dst = reinterpret_cast<uint4*>(out + g * 16 * K);
#pragma unroll
    for (int q = 0; q < K; q++) __stcs(dst + q, make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]));
  }
  // tail: fewer than 16 elements
  for (uint64_t e = ng * 16 + tid; e < n; e += nth) {
    W v = 0;
    for (int b = 0; b < S; b++) v |= (W)x[e * S + b] << (8 * b);
    for (int j = 0; j < K; j++) out[e * K + j] = (uint8_t)(v >> (8 * (S - 1 - j)));
  }
}

template <int S, int K>
__global__ void __launch_bounds__(256) k_trunc_decompress(const uint8_t* __restrict__ in, uint64_t n,
                                                          uint8_t* __restrict__ x) {
  using W = typename Word<S>::type;
  __shared__ uint4 s_stage[8 * 32 * S];
  const uint64_t ng = n / 16;
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  // gb = the warp's first group (warp-uniform, nth is a multiple of 32)
  const int lane = threadIdx.x & 31;
  for (uint64_t gb = tid - lane; gb < ng; gb += nth) {
    const uint64_t g = gb + lane;
    uint4 q4[S];
    if (g < ng) {
      uint32_t o[4 * K];
      const uint4* src = reinterpret_cast<const uint4*>(in + g * 16 * K);
#pragma unroll
      for (int q = 0; q < K; q++) {
        const uint4 u = __ldcs(src + q);
        o[4 * q] = u.x; o[4 * q + 1] = u.y; o[4 * q + 2] = u.z; o[4 * q + 3] = u.w;
      }
      W v[16];
      unpack16<S, K>(o, v);
#pragma unroll
      for (int q = 0; q < S; q++) {
        uint32_t w4[4];
#pragma unroll
        for (int t = 0; t < 4; t++) {
          const int word = 4 * q + t;
          if (S == 4) w4[t] = (uint32_t)v[word];
          else w4[t] = (uint32_t)(v[word >> 1] >> (32 * (word & 1)));
        }
        q4[q] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
      }
    }
    if (gb + 32 <= ng) {
      // the warp's 32 groups are consecutive: stage them in shared memory and store 512 contiguous
      // bytes per instruction (a lane's own 16 S bytes touch S different 128-B lines per instruction).
      // 16-byte slot i holds (lane i / S, part i % S), swizzled by (i / 8) & 3 against bank conflicts
      uint4* st = s_stage + (threadIdx.x >> 5) * 32 * S;
#pragma unroll
      for (int q = 0; q < S; q++) {
        const int i = lane * S + q;
        st[i ^ ((i >> 3) & 3)] = q4[q];
      }
      SZ3G_SYNCWARP();
      uint4* dst = reinterpret_cast<uint4*>(x + gb * 16 * S);
#pragma unroll
      for (int q = 0; q < S; q++) {
        const int i = q * 32 + lane;
        __stcs(dst + i, st[i ^ ((i >> 3) & 3)]);
      }
      SZ3G_SYNCWARP();
    } else if (g < ng) {
      uint4* dst = reinterpret_cast<uint4*>(x + g * 16 * S);
#pragma unroll
      for (int q = 0; q < S; q++) __stcs(dst + q, q4[q]);
    }
  }
  for (uint64_t e = ng * 16 + tid; e < n; e += nth) {
    W v = 0;
    for (int j = 0; j < K; j++) v |= (W)in[e * K + j] << (8 * (S - 1 - j));
    for (int b = 0; b < S; b++) x[e * S + b] = (uint8_t)(v >> (8 * b));
  }
}

int sm_count_tr() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

unsigned tr_grid(uint64_t n) {
  const uint64_t groups = std::max<uint64_t>(1, n / 16);
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((groups + 255) / 256, (uint64_t)sm_count_tr() * 8));
}

template <int S, int K>
void launch_c(const void* x, uint64_t n, uint8_t* out, cudaStream_t st) {
  k_trunc_compress<S, K><<<tr_grid(n), 256, 0, st>>>(static_cast<const uint8_t*>(x), n, out);
}
template <int S, int K>
void launch_d(const uint8_t* in, uint64_t n, void* x, cudaStream_t st) {
  k_trunc_decompress<S, K><<<tr_grid(n), 256, 0, st>>>(in, n, static_cast<uint8_t*>(x));
}

template <int S, int... Ks>
bool dispatch_c(int k, const void* x, uint64_t n, uint8_t* out, cudaStream_t st) {
  bool done = false;
  ((k == Ks ? (launch_c<S, Ks>(x, n, out, st), done = true) : false), ...);
  return done;
}
template <int S, int... Ks>
bool dispatch_d(int k, const uint8_t* in, uint64_t n, void* x, cudaStream_t st) {
  bool done = false;
  ((k == Ks ? (launch_d<S, Ks>(in, n, x, st), done = true) : false), ...);
  return done;
}

int tr_check() {
  if (cudaGetLastError() != cudaSuccess) return SZ3G_ECUDA;
  g_tr_launches.fetch_add(1, std::memory_order_relaxed);
  return SZ3G_OK;
}

int tr_validate(const sz3g_grid* grid, uint32_t k, const void* a, const void* b) {
  if (!grid) return SZ3G_EINVAL;
  if (grid->dtype != SZ3G_F32 && grid->dtype != SZ3G_F64) return SZ3G_EUNSUPPORTED;
  const uint32_t s = grid->dtype == SZ3G_F32 ? 4u : 8u;
  if (k < 1 || k > s) return SZ3G_ERANGE;
  if (grid->dims[0] * grid->dims[1] * grid->dims[2] == 0) return SZ3G_OK;   // nothing to touch
  if (!a || !b) return SZ3G_EINVAL;
  if ((reinterpret_cast<uintptr_t>(a) & 15) || (reinterpret_cast<uintptr_t>(b) & 15)) return SZ3G_EINVAL;
  return SZ3G_OK;
}

}  // namespace

uint64_t sz3g_truncation_launch_count_internal() { return g_tr_launches.load(); }

extern "C" {

int sz3g_truncation_compress(const sz3g_grid* grid, const void* x, uint32_t k, uint8_t* out,
                             sz3g_stream_t stream) {
  const int rc = tr_validate(grid, k, x, out);
  if (rc) return rc;
  const uint64_t n = grid->dims[0] * grid->dims[1] * grid->dims[2];
  if (n == 0) return SZ3G_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool ok = grid->dtype == SZ3G_F32 ? dispatch_c<4, 1, 2, 3, 4>((int)k, x, n, out, st)
                                          : dispatch_c<8, 1, 2, 3, 4, 5, 6, 7, 8>((int)k, x, n, out, st);
  return ok ? tr_check() : SZ3G_ERANGE;
}

int sz3g_truncation_decompress(const sz3g_grid* grid, const uint8_t* in, uint32_t k, void* x_out,
                               sz3g_stream_t stream) {
  const int rc = tr_validate(grid, k, in, x_out);
  if (rc) return rc;
  const uint64_t n = grid->dims[0] * grid->dims[1] * grid->dims[2];
  if (n == 0) return SZ3G_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool ok = grid->dtype == SZ3G_F32 ? dispatch_d<4, 1, 2, 3, 4>((int)k, in, n, x_out, st)
                                          : dispatch_d<8, 1, 2, 3, 4, 5, 6, 7, 8>((int)k, in, n, x_out, st);
  return ok ? tr_check() : SZ3G_ERANGE;
}

}  // extern "C"
