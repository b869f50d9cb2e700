// libsz3g -- coefficient-code delta coding (NEXT-3; oracle/DEFINITION.md C1-C2, reading G25).
// The G1 coefficient codes (int32 [NB][4]) are differenced along the block order per channel, zigzag-
// mapped, and clipped to uint16 symbols with an escape (65535) whose full value goes to a position-
// ordered escape list; the symbols (channel-major [4][NB]) are then Huffman-coded like the element
// codes (sz3g_huffman_*).  The inverse resolves escapes by rank and takes running sums per channel.
//
// Work decomposition: tiles of CT = 2048 consecutive positions of one channel (index ch * NB + b),
// one CTA per tile.  Encode: (1) escapes per tile, (2) exclusive scan of the tile counts (one CTA),
// (3) symbols + escapes at tile offset + in-tile rank (block scan).  Decode: (1) escapes per tile and
// the tile's sum of deltas, (2) scans of both (one CTA, the delta sums segmented per channel),
// (3) in-tile scan of the deltas + the tile's offset -> int32 codes.  Scratch: 2 x 8 bytes per tile.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>

#include "../../include/sz3g.h"
#include "ptx.cuh"

namespace {

std::atomic<uint64_t> g_cc_launches{0};
constexpr int CC_T = 256, CC_PER = 8, CT = CC_T * CC_PER;   // tile = 2048 positions of one channel
constexpr uint32_t ESC = 65535;

__device__ __forceinline__ uint64_t zigzag(int64_t d) { return d >= 0 ? (uint64_t)d * 2 : (uint64_t)(-(d + 1)) * 2 + 1; }
__device__ __forceinline__ int64_t unzigzag(uint64_t z) { return (z & 1) ? -(int64_t)(z >> 1) - 1 : (int64_t)(z >> 1); }

// block-wide exclusive scan (CC_T threads) of a 64-bit value; returns the block total
template <typename V>
__device__ V block_scan_excl(V v, V& excl, V* s_w) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  V x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const V y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[w] = x;
  SZ3G_SYNCTHREADS();
  V before = 0, total = 0;
  for (int i = 0; i < CC_T / 32; i++) {
    if (i < w) before += s_w[i];
    total += s_w[i];
  }
  excl = before + x - v;
  SZ3G_SYNCTHREADS();
  return total;
}

struct TileGeo {
  uint32_t ch;      // channel
  uint64_t b0, b1;  // block range of the tile
};
__device__ __forceinline__ TileGeo tile_geo(uint64_t tile, uint64_t nb, uint64_t tpc) {
  TileGeo t;
  t.ch = (uint32_t)(tile / tpc);
  t.b0 = (tile - (uint64_t)t.ch * tpc) * CT;
  t.b1 = min(nb, t.b0 + CT);
  return t;
}

__device__ __forceinline__ uint64_t enc_z(const int32_t* __restrict__ coef, uint64_t b, uint32_t ch) {
  const int64_t v = coef[4 * b + ch];
  const int64_t p = b ? (int64_t)coef[4 * (b - 1) + ch] : 0;
  return zigzag(v - p);
}

// ---------------------------------------------------------------- encode
__global__ void __launch_bounds__(CC_T) k_cc_enc_count(const int32_t* __restrict__ coef, uint64_t nb, uint64_t tpc,
                                                       uint64_t* __restrict__ tcount) {
  __shared__ uint64_t s_w[CC_T / 32];
  const TileGeo t = tile_geo(blockIdx.x, nb, tpc);
  uint64_t cnt = 0;
  for (uint64_t b = t.b0 + threadIdx.x; b < t.b1; b += CC_T) cnt += enc_z(coef, b, t.ch) >= ESC ? 1 : 0;
  uint64_t ex;
  const uint64_t tot = block_scan_excl<uint64_t>(cnt, ex, s_w);
  if (threadIdx.x == 0) tcount[blockIdx.x] = tot;
}

// one CTA: exclusive scan of n values in place; total to v[n] (and *total if given)
__global__ void __launch_bounds__(CC_T) k_cc_scan(uint64_t* __restrict__ v, uint64_t n, uint64_t* total) {
  __shared__ uint64_t s_w[CC_T / 32];
  __shared__ uint64_t s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  SZ3G_SYNCTHREADS();
  for (uint64_t b = 0; b < n; b += CC_T) {
    const uint64_t i = b + threadIdx.x;
    const uint64_t x = i < n ? v[i] : 0;
    uint64_t ex;
    const uint64_t tot = block_scan_excl<uint64_t>(x, ex, s_w);
    const uint64_t c = s_carry;
    if (i < n) v[i] = c + ex;
    SZ3G_SYNCTHREADS();
    if (threadIdx.x == 0) s_carry = c + tot;
    SZ3G_SYNCTHREADS();
  }
  if (threadIdx.x == 0) {
    v[n] = s_carry;
    if (total) *total = s_carry;
  }
}

__global__ void __launch_bounds__(CC_T) k_cc_enc_write(const int32_t* __restrict__ coef, uint64_t nb, uint64_t tpc,
                                                       const uint64_t* __restrict__ toff, uint16_t* __restrict__ sym,
                                                       uint64_t* __restrict__ esc, uint64_t cap) {
  __shared__ uint64_t s_w[CC_T / 32];
  const TileGeo t = tile_geo(blockIdx.x, nb, tpc);
  // thread j owns positions b0 + j*CC_PER .. (contiguous, so in-tile ranks follow position order)
  const uint64_t q0 = t.b0 + (uint64_t)threadIdx.x * CC_PER;
  uint64_t z[CC_PER];
  uint64_t cnt = 0;
#pragma unroll
  for (int k = 0; k < CC_PER; k++) {
    const uint64_t b = q0 + k;
    z[k] = b < t.b1 ? enc_z(coef, b, t.ch) : 0;
    cnt += (b < t.b1 && z[k] >= ESC) ? 1 : 0;
  }
  uint64_t ex;
  block_scan_excl<uint64_t>(cnt, ex, s_w);
  uint64_t pos = toff[blockIdx.x] + ex;
#pragma unroll
  for (int k = 0; k < CC_PER; k++) {
    const uint64_t b = q0 + k;
    if (b >= t.b1) break;
    const bool e = z[k] >= ESC;
    sym[(uint64_t)t.ch * nb + b] = e ? (uint16_t)ESC : (uint16_t)z[k];
    if (e) {
      if (pos < cap) esc[pos] = z[k];
      pos++;
    }
  }
}

// ---------------------------------------------------------------- decode
// (1) escapes per tile
__global__ void __launch_bounds__(CC_T) k_cc_dec_count(const uint16_t* __restrict__ sym, uint64_t nb, uint64_t tpc,
                                                       uint64_t* __restrict__ tcount) {
  __shared__ uint64_t s_w[CC_T / 32];
  const TileGeo t = tile_geo(blockIdx.x, nb, tpc);
  uint64_t cnt = 0;
  for (uint64_t b = t.b0 + threadIdx.x; b < t.b1; b += CC_T) cnt += sym[(uint64_t)t.ch * nb + b] == ESC ? 1 : 0;
  uint64_t ex;
  const uint64_t tot = block_scan_excl<uint64_t>(cnt, ex, s_w);
  if (threadIdx.x == 0) tcount[blockIdx.x] = tot;
}

// the tile's deltas (escapes resolved): per-thread values, in position order
__device__ __forceinline__ void dec_deltas(const uint16_t* __restrict__ sym, uint64_t nb, const TileGeo& t,
                                           const uint64_t* __restrict__ esc, uint64_t nesc, uint64_t eoff,
                                           int64_t (&d)[CC_PER], uint64_t* s_w, bool& bad) {
  const uint64_t q0 = t.b0 + (uint64_t)threadIdx.x * CC_PER;
  uint32_t s[CC_PER];
  uint64_t cnt = 0;
#pragma unroll
  for (int k = 0; k < CC_PER; k++) {
    const uint64_t b = q0 + k;
    s[k] = b < t.b1 ? sym[(uint64_t)t.ch * nb + b] : 0u;
    cnt += s[k] == ESC ? 1 : 0;
  }
  uint64_t ex;
  block_scan_excl<uint64_t>(cnt, ex, s_w);
  uint64_t pos = eoff + ex;
#pragma unroll
  for (int k = 0; k < CC_PER; k++) {
    uint64_t z = s[k];
    if (s[k] == ESC) {
      if (pos < nesc) z = esc[pos];
      else bad = true;
      pos++;
    }
    d[k] = unzigzag(z);
  }
}

// (1b) sum of the tile's deltas (needs the escape offsets: run after the count scan)
__global__ void __launch_bounds__(CC_T) k_cc_dec_sums(const uint16_t* __restrict__ sym, uint64_t nb, uint64_t tpc,
                                                      const uint64_t* __restrict__ esc, uint64_t nesc,
                                                      const uint64_t* __restrict__ eoff, uint64_t* __restrict__ tsum,
                                                      int32_t* status) {
  __shared__ uint64_t s_w[CC_T / 32];
  const TileGeo t = tile_geo(blockIdx.x, nb, tpc);
  int64_t d[CC_PER];
  bool bad = false;
  dec_deltas(sym, nb, t, esc, nesc, eoff[blockIdx.x], d, s_w, bad);
  uint64_t loc = 0;
#pragma unroll
  for (int k = 0; k < CC_PER; k++) loc += (uint64_t)d[k];
  uint64_t ex;
  const uint64_t tot = block_scan_excl<uint64_t>(loc, ex, s_w);
  if (threadIdx.x == 0) tsum[blockIdx.x] = tot;
  if (bad) atomicOr(status, (int)SZ3G_STATUS_BAD_HUFFMAN);
}

// (2b) one CTA: exclusive scan of the tile sums segmented per channel (tpc tiles per channel)
__global__ void __launch_bounds__(CC_T) k_cc_scan_seg(uint64_t* __restrict__ v, uint64_t tpc) {
  __shared__ uint64_t s_w[CC_T / 32];
  __shared__ uint64_t s_carry;
  for (int ch = 0; ch < 4; ch++) {
    if (threadIdx.x == 0) s_carry = 0;
    SZ3G_SYNCTHREADS();
    uint64_t* w = v + (uint64_t)ch * tpc;
    for (uint64_t b = 0; b < tpc; b += CC_T) {
      const uint64_t i = b + threadIdx.x;
      const uint64_t x = i < tpc ? w[i] : 0;
      uint64_t ex;
      const uint64_t tot = block_scan_excl<uint64_t>(x, ex, s_w);
      const uint64_t c = s_carry;
      if (i < tpc) w[i] = c + ex;
      SZ3G_SYNCTHREADS();
      if (threadIdx.x == 0) s_carry = c + tot;
      SZ3G_SYNCTHREADS();
    }
  }
}

// (3) codes = tile offset + in-tile running sum
__global__ void __launch_bounds__(CC_T) k_cc_dec_write(const uint16_t* __restrict__ sym, uint64_t nb, uint64_t tpc,
                                                       const uint64_t* __restrict__ esc, uint64_t nesc,
                                                       const uint64_t* __restrict__ eoff,
                                                       const uint64_t* __restrict__ toff, int32_t* __restrict__ coef) {
  __shared__ uint64_t s_w[CC_T / 32];
  const TileGeo t = tile_geo(blockIdx.x, nb, tpc);
  int64_t d[CC_PER];
  bool bad = false;
  dec_deltas(sym, nb, t, esc, nesc, eoff[blockIdx.x], d, s_w, bad);
  uint64_t loc = 0;
#pragma unroll
  for (int k = 0; k < CC_PER; k++) loc += (uint64_t)d[k];
  uint64_t ex;
  block_scan_excl<uint64_t>(loc, ex, s_w);
  uint64_t acc = toff[blockIdx.x] + ex;
  const uint64_t q0 = t.b0 + (uint64_t)threadIdx.x * CC_PER;
#pragma unroll
  for (int k = 0; k < CC_PER; k++) {
    const uint64_t b = q0 + k;
    acc += (uint64_t)d[k];
    if (b < t.b1) coef[4 * b + t.ch] = (int32_t)(int64_t)acc;
  }
}

int cc_check(int nl) {
  if (cudaGetLastError() != cudaSuccess) return SZ3G_ECUDA;
  g_cc_launches.fetch_add((uint64_t)nl, std::memory_order_relaxed);
  return SZ3G_OK;
}

}  // namespace

uint64_t sz3g_coefcode_launch_count_internal() { return g_cc_launches.load(); }

extern "C" {

uint64_t sz3g_coef_delta_scratch_bytes(uint64_t nb) {
  const uint64_t tpc = (nb + CT - 1) / CT;
  return 8ull * (2 * (4 * tpc + 1) + 2);
}

int sz3g_coef_delta_encode(const int32_t* coef, uint64_t nb, uint16_t* sym, uint64_t* escapes, uint64_t esc_cap,
                           uint64_t* d_nesc, void* scratch, sz3g_stream_t stream) {
  if (!d_nesc || (nb > 0 && (!coef || !sym || !scratch))) return SZ3G_EINVAL;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (nb == 0) {
    cudaMemsetAsync(d_nesc, 0, 8, st);
    return cudaGetLastError() == cudaSuccess ? SZ3G_OK : SZ3G_ECUDA;
  }
  const uint64_t tpc = (nb + CT - 1) / CT, nt = 4 * tpc;
  uint64_t* tcount = static_cast<uint64_t*>(scratch);
  k_cc_enc_count<<<(unsigned)nt, CC_T, 0, st>>>(coef, nb, tpc, tcount);
  k_cc_scan<<<1, CC_T, 0, st>>>(tcount, nt, d_nesc);
  k_cc_enc_write<<<(unsigned)nt, CC_T, 0, st>>>(coef, nb, tpc, tcount, sym, escapes, esc_cap);
  return cc_check(3);
}

int sz3g_coef_delta_decode(const uint16_t* sym, uint64_t nb, const uint64_t* escapes, uint64_t nesc, int32_t* coef,
                           void* scratch, int32_t* d_status, sz3g_stream_t stream) {
  if (nb == 0) return SZ3G_OK;
  if (!sym || !coef || !scratch || !d_status || (nesc > 0 && !escapes)) return SZ3G_EINVAL;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const uint64_t tpc = (nb + CT - 1) / CT, nt = 4 * tpc;
  uint64_t* eoff = static_cast<uint64_t*>(scratch);
  uint64_t* tsum = eoff + nt + 1;
  k_cc_dec_count<<<(unsigned)nt, CC_T, 0, st>>>(sym, nb, tpc, eoff);
  k_cc_scan<<<1, CC_T, 0, st>>>(eoff, nt, nullptr);
  k_cc_dec_sums<<<(unsigned)nt, CC_T, 0, st>>>(sym, nb, tpc, escapes, nesc, eoff, tsum, d_status);
  k_cc_scan_seg<<<1, CC_T, 0, st>>>(tsum, tpc);
  k_cc_dec_write<<<(unsigned)nt, CC_T, 0, st>>>(sym, nb, tpc, escapes, nesc, eoff, tsum, coef);
  return cc_check(5);
}

}  // extern "C"
