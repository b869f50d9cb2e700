// libsz3g -- the encoder stage after the quantiser (NEXT-1): Huffman codebook from the merged
// histogram, GPU encode / decode of the uint16 codes (App. A
// P:948-957).  C ABI in include/sz3g.h (sz3g_huffman_*).  The definition the kernels reproduce is
// oracle/DEFINITION.md H1-H5: optimal length-limited code lengths by package-merge with a fixed tie
// rule, canonical codewords, chunks of C codes each packed MSB-first into whole 32-bit words.
//
// Kernels:
//   k_huff_codebook   ONE CTA (1024 threads): compact the active symbols, LSD radix sort by
//                     (count, symbol), package-merge with every level merged in parallel by
//                     merge-path partitions, leaf counts per level, lengths, canonical codewords
//                     (per-length ranks with warp match + block scans), the decoder's 12-bit LUT.
//   k_huff_chunk_words  one warp per chunk: words of the chunk (sum of code lengths / 32, ceil).
//   k_scan_*          exclusive scan of the chunk word counts -> chunk offsets (3 phases).
//   k_huff_encode     one warp per chunk: lanes own 64 consecutive codes, warp scan of their bit
//                     counts, each lane packs its bits into whole words of a shared-memory image of
//                     the chunk (first / last word by atomicOr), the image is copied out coalesced.
//   k_huff_decode     one thread per chunk: 64-bit bit window, 12-bit LUT in shared memory,
//                     canonical search for longer codes, 8 codes per 16-byte store.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>

#include "../../include/sz3g.h"

namespace {

constexpr int HF_THREADS = 512;         // codebook CTA (16 x 512 radix counters = 32 KiB smem)
constexpr int HF_WARPS = HF_THREADS / 32;
constexpr int HF_LUT_BITS = 12;         // decoder first-level table
constexpr int HF_MAXL = 32;             // array bound for per-length tables (max_len <= 24 supported)
constexpr int HF_MAX_LEN_LIMIT = 24;

// ------------------------------------------------------------------------------------------------
// Device table layout (sz3g_huffman_dtable_bytes): lut[4096] u32 ((len << 16) | symbol, 0 = longer
// code), first[32] u32, count[32] u32, base[32] u32, syms[nsym] u16 (symbols of codes longer than the
// LUT, ordered by (length, codeword)).
struct DTab {
  uint32_t lut[1 << HF_LUT_BITS];
  uint32_t first[HF_MAXL];
  uint32_t count[HF_MAXL];
  uint32_t base[HF_MAXL];
};
size_t dtable_bytes(uint32_t nsym) { return sizeof(DTab) + 2ull * nsym; }

// scratch layout of the codebook kernel (sz3g_huffman_scratch_bytes)
struct CbScratch {
  uint64_t* keys0;    // [nsym] sort ping
  uint64_t* keys1;    // [nsym] sort pong
  uint64_t* listA;    // [2 nsym] merged list of the level below
  uint64_t* listB;    // [2 nsym] merged list being built
  uint64_t* pk;       // [max_len][nsym] package weights of each level
};
size_t cb_scratch_bytes(uint32_t nsym, uint32_t max_len) {
  return 8ull * nsym * (2 + 4 + (size_t)max_len) + 256;
}
__host__ __device__ inline CbScratch cb_carve(void* base, uint32_t nsym) {
  uint64_t* p = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(base) + 15) & ~uintptr_t(15));
  CbScratch s;
  s.keys0 = p;
  s.keys1 = p + nsym;
  s.listA = p + 2ull * nsym;
  s.listB = p + 4ull * nsym;
  s.pk = p + 6ull * nsym;
  return s;
}

// block-wide exclusive scan of one uint32 per thread (HF_THREADS threads); returns the total
__device__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp, uint32_t& excl) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t t = lane < HF_WARPS ? s_warp[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    s_warp[lane] = t;   // inclusive totals per warp
  }
  __syncthreads();
  const uint32_t before = w ? s_warp[w - 1] : 0u;
  excl = before + x - v;
  const uint32_t total = s_warp[HF_WARPS - 1];
  __syncthreads();
  return total;
}

// number of leaves among the first k items of merge(leaves[0..n), pk[0..np)), a leaf before a
// package of equal weight (merge-path partition)
__device__ __forceinline__ uint32_t merge_split(const uint64_t* __restrict__ leaves, uint32_t n,
                                                const uint64_t* __restrict__ pk, uint32_t np, uint32_t k) {
  uint32_t lo = k > np ? k - np : 0u, hi = min(k, n);
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    // leaf mid is among the first k iff fewer than k - mid packages are strictly lighter
    if (pk[k - mid - 1] >= leaves[mid]) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(HF_THREADS, 1)
    k_huff_codebook(const int64_t* __restrict__ hist, uint32_t nsym, uint32_t max_len, uint8_t* __restrict__ lens,
                    uint32_t* __restrict__ cws, DTab* __restrict__ dt, void* scratch, int32_t* status) {
  __shared__ uint32_t s_cnt[16 * HF_THREADS];   // radix digit counts [digit][thread]; reused below
  __shared__ uint32_t s_warp[32];
  __shared__ uint32_t s_bad, s_bits;
  __shared__ uint32_t s_c[HF_MAXL + 1];         // leaves per level
  __shared__ uint32_t s_np[HF_MAXL + 1];        // packages per level
  __shared__ uint32_t s_blc[HF_MAXL + 1];       // symbols per length
  __shared__ uint32_t s_first[HF_MAXL + 1];
  const int tid = threadIdx.x;
  const CbScratch S = cb_carve(scratch, nsym);
  if (tid == 0) { s_bad = 0; s_bits = 0; }
  for (uint32_t s = tid; s < nsym; s += HF_THREADS) { lens[s] = 0; cws[s] = 0; }
  for (uint32_t i = tid; i < (1u << HF_LUT_BITS); i += HF_THREADS) dt->lut[i] = 0;
  if (tid < HF_MAXL) { dt->first[tid] = 0; dt->count[tid] = 0; dt->base[tid] = 0; }
  __syncthreads();

  // (A) compact active symbols, in symbol order: key = (count << 16) | symbol
  const uint32_t per = (nsym + HF_THREADS - 1) / HF_THREADS;
  const uint32_t s0 = min(nsym, tid * per), s1 = min(nsym, s0 + per);
  uint32_t mine = 0;
  uint64_t kmax = 0;
  for (uint32_t s = s0; s < s1; s++) {
    const int64_t c = hist[s];
    if (c > 0) mine++;
    if (c < 0 || (uint64_t)c >= (1ull << 47)) atomicOr(&s_bad, 1u);
  }
  uint32_t excl;
  const uint32_t n = block_excl_scan(mine, s_warp, excl);
  for (uint32_t s = s0, o = excl; s < s1; s++) {
    const int64_t c = hist[s];
    if (c > 0) {
      const uint64_t key = ((uint64_t)c << 16) | s;
      S.keys0[o++] = key;
      kmax = max(kmax, key);
    }
  }
  // highest key bit -> number of 4-bit radix passes
  {
    const uint32_t hb = kmax ? 64u - (uint32_t)__clzll((long long)kmax) : 0u;
    atomicMax(&s_bits, hb);
  }
  __syncthreads();
  const bool bad = s_bad || n == 0 || (max_len < 32 && (1ull << max_len) < n);
  if (bad) {
    if (tid == 0) atomicOr(status, (int)SZ3G_STATUS_BAD_HUFFMAN);
    return;
  }
  if (n == 1) {   // one symbol -> length 1, codeword 0
    if (tid == 0) {
      const uint32_t sym = (uint32_t)(S.keys0[0] & 0xffffu);
      lens[sym] = 1;
      cws[sym] = 0;
      dt->first[1] = 0;
      dt->count[1] = 1;
      for (uint32_t i = 0; i < (1u << (HF_LUT_BITS - 1)); i++) dt->lut[i] = (1u << 16) | sym;
    }
    return;
  }

  // (B) stable LSD radix sort of the n keys, 4 bits per pass (ascending count, then symbol)
  uint64_t* src = S.keys0;
  uint64_t* dst = S.keys1;
  const uint32_t iper = (n + HF_THREADS - 1) / HF_THREADS;
  const uint32_t i0 = min(n, tid * iper), i1 = min(n, i0 + iper);
  for (uint32_t sh = 0; sh < s_bits; sh += 4) {
    uint32_t cnt[16];
#pragma unroll
    for (int d = 0; d < 16; d++) cnt[d] = 0;
    for (uint32_t i = i0; i < i1; i++) cnt[(src[i] >> sh) & 15u]++;
#pragma unroll
    for (int d = 0; d < 16; d++) s_cnt[d * HF_THREADS + tid] = cnt[d];
    __syncthreads();
    // exclusive scan over (digit, thread) in digit-major order: thread t owns entries [16t, 16t + 16)
    uint32_t loc[16], sum = 0;
#pragma unroll
    for (int e = 0; e < 16; e++) { loc[e] = sum; sum += s_cnt[16 * tid + e]; }
    uint32_t base;
    block_excl_scan(sum, s_warp, base);
#pragma unroll
    for (int e = 0; e < 16; e++) s_cnt[16 * tid + e] = base + loc[e];
    __syncthreads();
    uint32_t off[16];
#pragma unroll
    for (int d = 0; d < 16; d++) off[d] = s_cnt[d * HF_THREADS + tid];
    for (uint32_t i = i0; i < i1; i++) {
      const uint64_t k = src[i];
      const uint32_t d = (uint32_t)(k >> sh) & 15u;
      uint32_t o = 0;
#pragma unroll
      for (int e = 0; e < 16; e++) if (e == (int)d) o = off[e]++;
      dst[o] = k;
    }
    __syncthreads();
    uint64_t* t = src; src = dst; dst = t;
  }
  // sorted keys in src; leaf weights in listA (level max_len list)
  uint64_t* leaves = dst;   // reuse the other sort buffer for the leaf weights
  for (uint32_t i = tid; i < n; i += HF_THREADS) leaves[i] = src[i] >> 16;
  for (uint32_t i = tid; i < n; i += HF_THREADS) S.listA[i] = leaves[i];
  __syncthreads();

  // (C) package-merge: list[l] = merge(leaves, packages of list[l + 1]), l = max_len - 1 .. 1
  uint64_t* A = S.listA;
  uint64_t* B = S.listB;
  uint32_t lenA = n;
  if (tid == 0) s_np[max_len] = 0;
  for (uint32_t l = max_len - 1; l >= 1; l--) {
    uint64_t* pk = S.pk + (size_t)l * nsym;
    const uint32_t np = lenA / 2;
    if (tid == 0) s_np[l] = np;
    for (uint32_t j = tid; j < np; j += HF_THREADS) pk[j] = A[2 * j] + A[2 * j + 1];
    __syncthreads();
    const uint32_t tot = n + np;
    const uint32_t oper = (tot + HF_THREADS - 1) / HF_THREADS;
    const uint32_t k0 = min(tot, tid * oper), k1 = min(tot, k0 + oper);
    if (k0 < k1) {
      uint32_t a = merge_split(leaves, n, pk, np, k0), b = k0 - a;
      for (uint32_t k = k0; k < k1; k++) {
        if (b >= np || (a < n && leaves[a] <= pk[b])) B[k] = leaves[a++];
        else B[k] = pk[b++];
      }
    }
    __syncthreads();
    uint64_t* t = A; A = B; B = t;
    lenA = tot;
    if (l == 1) break;
  }
  // (D) leaves among the selected prefix m of each level: m = 2n - 2 at level 1, then twice the
  // packages taken at the level above
  if (tid == 0) {
    uint64_t m = 2ull * n - 2;
    for (uint32_t l = 1; l <= max_len; l++) {
      const uint32_t np = s_np[l];
      const uint64_t tot = (uint64_t)n + np;
      const uint32_t k = (uint32_t)(m < tot ? m : tot);
      const uint32_t c = np ? merge_split(leaves, n, S.pk + (size_t)l * nsym, np, k) : k;
      s_c[l] = c;
      m = 2 * (m - c);
    }
  }
  if (tid <= HF_MAXL) s_blc[tid] = 0;
  __syncthreads();
  // (E) lengths of the sorted leaves: len(i) = #{l : i < c[l]}
  for (uint32_t i = tid; i < n; i += HF_THREADS) {
    uint32_t L = 0;
    for (uint32_t l = 1; l <= max_len; l++) L += i < s_c[l] ? 1u : 0u;
    lens[(uint32_t)(src[i] & 0xffffu)] = (uint8_t)L;
    atomicAdd(&s_blc[L], 1u);
  }
  __syncthreads();
  // (F) canonical codewords: first code per length (DEFLATE form of H3), then per-symbol rank
  // among the symbols of its length in symbol order
  if (tid == 0) {
    uint32_t code = 0, cum = 0;
    s_blc[0] = 0;
    for (uint32_t L = 1; L <= max_len; L++) {
      code = (code + s_blc[L - 1]) << 1;
      s_first[L] = code;
      dt->first[L] = code;
      dt->count[L] = s_blc[L];
      dt->base[L] = cum;
      if (L > HF_LUT_BITS) cum += s_blc[L];
    }
  }
  __syncthreads();
  uint32_t* s_run = s_cnt;            // running count per length over earlier rounds
  uint32_t* s_wl = s_cnt + 64;        // [HF_WARPS][32 lengths] counts of the current round
  for (int i = tid; i < 64 + HF_WARPS * 32; i += HF_THREADS) s_cnt[i] = 0;
  __syncthreads();
  const int lane = tid & 31, wid = tid >> 5;
  uint16_t* syms = reinterpret_cast<uint16_t*>(dt + 1);
  for (uint32_t r0 = 0; r0 < nsym; r0 += HF_THREADS) {
    const uint32_t s = r0 + tid;
    const uint32_t L = s < nsym ? lens[s] : 0u;
    const uint32_t peers = __match_any_sync(0xffffffffu, L);
    const uint32_t rank_w = __popc(peers & ((1u << lane) - 1u));
    if (lane == 31 - __clz(peers)) s_wl[wid * 32 + L] = __popc(peers);   // the group's highest lane
    __syncthreads();
    if (L > 0) {
      uint32_t before = s_run[L];
      for (int w = 0; w < wid; w++) before += s_wl[w * 32 + L];
      const uint32_t cw = s_first[L] + before + rank_w;
      cws[s] = cw;
      if (L <= HF_LUT_BITS) {
        const uint32_t lo = cw << (HF_LUT_BITS - L), cnt = 1u << (HF_LUT_BITS - L);
        for (uint32_t e = 0; e < cnt; e++) dt->lut[lo + e] = (L << 16) | s;
      } else {
        syms[dt->base[L] + (cw - s_first[L])] = (uint16_t)s;
      }
    }
    __syncthreads();
    if (tid < 32) {   // fold this round's per-warp counts into the running counts, clear them
      uint32_t add = 0;
      for (int w = 0; w < HF_WARPS; w++) { add += s_wl[w * 32 + tid]; s_wl[w * 32 + tid] = 0; }
      s_run[tid] += add;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------------------
// encode
__global__ void __launch_bounds__(256) k_huff_chunk_words(const uint16_t* __restrict__ codes, uint64_t n,
                                                          uint32_t chunk, const uint8_t* __restrict__ lens,
                                                          uint64_t* __restrict__ words, uint64_t nch,
                                                          int32_t* status) {
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (uint64_t c = warp; c < nch; c += nw) {
    const uint64_t e0 = c * chunk, e1 = min(n, e0 + chunk);
    uint64_t bits = 0;
    bool miss = false;
    for (uint64_t e = e0 + lane; e < e1; e += 32) {
      const uint32_t L = __ldg(lens + codes[e]);
      bits += L;
      miss |= L == 0;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) bits += __shfl_xor_sync(0xffffffffu, bits, o);
    if (__any_sync(0xffffffffu, miss) && lane == 0) atomicOr(status, (int)SZ3G_STATUS_BAD_HUFFMAN);
    if (lane == 0) words[c] = (bits + 31) / 32;
  }
}

// exclusive scan of v[0..m) in place, v[m] <- total.  Phase 1: per-block sums of 4096 items.
constexpr int SCAN_T = 512, SCAN_PER = 8, SCAN_TILE = SCAN_T * SCAN_PER;
__global__ void __launch_bounds__(SCAN_T) k_scan_sums(const uint64_t* __restrict__ v, uint64_t m,
                                                      uint64_t* __restrict__ sums) {
  __shared__ uint64_t s[SCAN_T / 32];
  const uint64_t b0 = (uint64_t)blockIdx.x * SCAN_TILE;
  uint64_t acc = 0;
  for (int k = 0; k < SCAN_PER; k++) {
    const uint64_t i = b0 + (uint64_t)k * SCAN_T + threadIdx.x;
    if (i < m) acc += v[i];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int w = 0; w < SCAN_T / 32; w++) t += s[w];
    sums[blockIdx.x] = t;
  }
}

// Phase 2 (one CTA): exclusive scan of the block sums (sequential chunks of SCAN_T), total at sums[nb]
__global__ void __launch_bounds__(SCAN_T) k_scan_top(uint64_t* __restrict__ sums, uint64_t nb) {
  __shared__ uint64_t s_w[SCAN_T / 32];
  __shared__ uint64_t s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (uint64_t b = 0; b < nb; b += SCAN_T) {
    const uint64_t i = b + threadIdx.x;
    const uint64_t v = i < nb ? sums[i] : 0;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[w] = x;
    __syncthreads();
    uint64_t before = 0;
    for (int k = 0; k < w; k++) before += s_w[k];
    const uint64_t carry = s_carry;
    if (i < nb) sums[i] = carry + before + x - v;
    __syncthreads();
    if (threadIdx.x == SCAN_T - 1) s_carry = carry + before + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[nb] = s_carry;
}

// Phase 3: exclusive scan inside each block + the block's offset; v[m] <- total
__global__ void __launch_bounds__(SCAN_T) k_scan_apply(uint64_t* __restrict__ v, uint64_t m,
                                                       const uint64_t* __restrict__ sums, uint64_t nb) {
  __shared__ uint64_t s_w[SCAN_T / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t b0 = (uint64_t)blockIdx.x * SCAN_TILE + (uint64_t)threadIdx.x * SCAN_PER;
  uint64_t loc[SCAN_PER], sum = 0;
#pragma unroll
  for (int k = 0; k < SCAN_PER; k++) {
    const uint64_t i = b0 + k;
    const uint64_t x = i < m ? v[i] : 0;
    loc[k] = sum;
    sum += x;
  }
  uint64_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[w] = x;
  __syncthreads();
  uint64_t before = sums[blockIdx.x];
  for (int k = 0; k < w; k++) before += s_w[k];
  before += x - sum;
#pragma unroll
  for (int k = 0; k < SCAN_PER; k++) {
    const uint64_t i = b0 + k;
    if (i < m) v[i] = before + loc[k];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) v[m] = sums[nb];
}

// One warp per chunk (chunk <= 32 * 64 codes).  Lane l owns codes [l*per, (l+1)*per) of the chunk.
constexpr int ENC_WARPS = 4, ENC_PER = 64, ENC_MAX_CHUNK = 32 * ENC_PER;   // 4 x 6 KiB chunk images
constexpr int ENC_WORDS = ENC_MAX_CHUNK * HF_MAX_LEN_LIMIT / 32 + 1;
__global__ void __launch_bounds__(ENC_WARPS * 32) k_huff_encode(const uint16_t* __restrict__ codes, uint64_t n,
                                                                uint32_t chunk, const uint8_t* __restrict__ lens,
                                                                const uint32_t* __restrict__ cws,
                                                                const uint64_t* __restrict__ offs, uint64_t nch,
                                                                uint32_t* __restrict__ payload, uint64_t cap,
                                                                int32_t* status) {
  __shared__ uint32_t s_img[ENC_WARPS][ENC_WORDS];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  uint32_t* img = s_img[wl];
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t per = (chunk + 31) / 32;
  for (uint64_t c = gw; c < nch; c += nw) {
    const uint64_t e0 = c * chunk, e1 = min(n, e0 + chunk);
    const uint64_t w0 = offs[c], nwords = offs[c + 1] - w0;
    if (offs[c + 1] > cap) {   // capacity exceeded: nothing of this chunk is written
      if (lane == 0) atomicOr(status, (int)SZ3G_STATUS_PAYLOAD_OVERFLOW);
      continue;
    }
    for (uint32_t i = lane; i < nwords; i += 32) img[i] = 0u;
    __syncwarp();
    const uint64_t a0 = min(e1, e0 + (uint64_t)lane * per), a1 = min(e1, a0 + per);
    uint32_t bits = 0;
    for (uint64_t e = a0; e < a1; e++) bits += __ldg(lens + codes[e]);
    uint32_t incl = bits;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t b0 = incl - bits;   // first bit of this lane inside the chunk
    // pack: the buffer starts with the (b0 % 32) bits of the previous lane as zeros, so every emitted
    // word is a whole word of the chunk image; the first and the last are shared -> atomicOr
    uint64_t buf = 0;
    uint32_t nbuf = b0 & 31u, wi = b0 >> 5;
    bool first = true;
    for (uint64_t e = a0; e < a1; e++) {
      const uint32_t q = codes[e];
      const uint32_t L = __ldg(lens + q), cw = __ldg(cws + q);
      buf = (buf << L) | cw;
      nbuf += L;
      if (nbuf >= 32) {
        const uint32_t word = (uint32_t)(buf >> (nbuf - 32));
        if (first) atomicOr(&img[wi], word);
        else img[wi] = word;
        first = false;
        wi++;
        nbuf -= 32;
      }
    }
    if (nbuf > 0 && bits > 0) atomicOr(&img[wi], (uint32_t)(buf << (32 - nbuf)));
    __syncwarp();
    for (uint32_t i = lane; i < nwords; i += 32) payload[w0 + i] = img[i];
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------------------------
// decode: one thread per chunk
__global__ void __launch_bounds__(256) k_huff_decode(const uint32_t* __restrict__ payload,
                                                     const uint64_t* __restrict__ offs, uint64_t n, uint32_t chunk,
                                                     const DTab* __restrict__ dt, uint32_t max_len,
                                                     uint16_t* __restrict__ codes, uint64_t nch, int32_t* status) {
  __shared__ uint32_t s_lut[1 << HF_LUT_BITS];
  __shared__ uint32_t s_first[HF_MAXL], s_count[HF_MAXL], s_base[HF_MAXL];
  for (int i = threadIdx.x; i < (1 << HF_LUT_BITS); i += blockDim.x) s_lut[i] = dt->lut[i];
  if (threadIdx.x < HF_MAXL) {
    s_first[threadIdx.x] = dt->first[threadIdx.x];
    s_count[threadIdx.x] = dt->count[threadIdx.x];
    s_base[threadIdx.x] = dt->base[threadIdx.x];
  }
  __syncthreads();
  const uint16_t* syms = reinterpret_cast<const uint16_t*>(dt + 1);
  const uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (c >= nch) return;
  const uint64_t e0 = c * chunk, e1 = min(n, e0 + chunk);
  const uint32_t* p = payload + offs[c];
  const uint32_t* pend = payload + offs[c + 1];
  uint64_t win = 0;     // left-aligned bit window (zeros past the end of the chunk)
  uint32_t avail = 0;
  uint64_t consumed = 0;
  bool bad = false;
  uint32_t pack[4];
  uint32_t npk = 0;
  const bool vec = ((e0 & 7) == 0);   // 16-byte stores from an 8-code aligned start
  for (uint64_t e = e0; e < e1; e++) {
    if (avail <= 32) {
      const uint32_t w = p < pend ? *p : 0u;
      if (p < pend) p++;
      win |= (uint64_t)w << (32 - avail);
      avail += 32;
    }
    const uint32_t top = (uint32_t)(win >> 40);   // 24 bits
    uint32_t ent = s_lut[top >> (24 - HF_LUT_BITS)];
    uint32_t L, sym;
    if (ent) {
      L = ent >> 16;
      sym = ent & 0xffffu;
    } else {
      sym = 0;
      L = 0;
      for (uint32_t l = HF_LUT_BITS + 1; l <= max_len; l++) {
        const uint32_t code = top >> (24 - l);
        if (code - s_first[l] < s_count[l]) {
          sym = syms[s_base[l] + code - s_first[l]];
          L = l;
          break;
        }
      }
      if (L == 0) { bad = true; L = 1; }
    }
    win <<= L;
    avail -= L;
    consumed += L;
    if (vec) {
      const uint32_t slot = npk >> 1;
      if (npk & 1) pack[slot] |= sym << 16;
      else pack[slot] = sym;
      if (++npk == 8) {
        *reinterpret_cast<uint4*>(codes + e - 7) = make_uint4(pack[0], pack[1], pack[2], pack[3]);
        npk = 0;
      }
    } else {
      codes[e] = (uint16_t)sym;
    }
  }
  if (vec) {   // tail (fewer than 8 codes)
    for (uint32_t k = 0; k < npk; k++) codes[e1 - npk + k] = (uint16_t)(pack[k >> 1] >> (16 * (k & 1)));
  }
  // consumed more bits than the chunk holds?
  if (bad || consumed > (offs[c + 1] - offs[c]) * 32) atomicOr(status, (int)SZ3G_STATUS_BAD_HUFFMAN);
}

std::atomic<uint64_t> g_hf_launches{0};

int hf_check(int nl) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return SZ3G_ECUDA;
  g_hf_launches.fetch_add((uint64_t)nl, std::memory_order_relaxed);
  return SZ3G_OK;
}

int sm_count_hf() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

}  // namespace

// launches of this translation unit (folded into sz3g_launch_count)
uint64_t sz3g_huffman_launch_count_internal() { return g_hf_launches.load(); }

extern "C" {

uint64_t sz3g_huffman_scratch_bytes(uint32_t nsym, uint32_t max_len) { return cb_scratch_bytes(nsym, max_len); }
uint64_t sz3g_huffman_dtable_bytes(uint32_t nsym) { return dtable_bytes(nsym); }
uint64_t sz3g_huffman_encode_scratch_bytes(uint64_t n, uint32_t chunk) {
  const uint64_t nch = chunk ? (n + chunk - 1) / chunk : 0;
  return 8 * ((nch + SCAN_TILE - 1) / SCAN_TILE + 2);
}

int sz3g_huffman_codebook(const int64_t* hist, uint32_t nsym, uint32_t max_len, uint8_t* lengths,
                          uint32_t* codewords, void* dtable, void* scratch, int32_t* d_status,
                          sz3g_stream_t stream) {
  if (!hist || !lengths || !codewords || !dtable || !scratch || !d_status) return SZ3G_EINVAL;
  if (nsym < 1 || nsym > 65536) return SZ3G_ERANGE;
  if (max_len < 1 || max_len > HF_MAX_LEN_LIMIT) return SZ3G_ERANGE;
  if (reinterpret_cast<uintptr_t>(dtable) & 15) return SZ3G_EINVAL;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  k_huff_codebook<<<1, HF_THREADS, 0, st>>>(hist, nsym, max_len, lengths, codewords,
                                            reinterpret_cast<DTab*>(dtable), scratch, d_status);
  return hf_check(1);
}

int sz3g_huffman_encode(const uint16_t* codes, uint64_t n, uint32_t chunk, const uint8_t* lengths,
                        const uint32_t* codewords, uint64_t* chunk_offsets, uint32_t* payload,
                        uint64_t payload_cap_words, void* scratch, int32_t* d_status, sz3g_stream_t stream) {
  if ((n > 0 && !codes) || !lengths || !codewords || !chunk_offsets || !d_status) return SZ3G_EINVAL;
  if (chunk < 1 || chunk > ENC_MAX_CHUNK) return SZ3G_ERANGE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const uint64_t nch = (n + chunk - 1) / chunk;
  if (nch == 0) {
    cudaMemsetAsync(chunk_offsets, 0, 8, st);
    return cudaGetLastError() == cudaSuccess ? SZ3G_OK : SZ3G_ECUDA;
  }
  if (!payload || !scratch) return SZ3G_EINVAL;
  const int sms = sm_count_hf();
  const unsigned gw = (unsigned)std::min<uint64_t>((nch * 32 + 255) / 256, (uint64_t)sms * 16);
  k_huff_chunk_words<<<gw, 256, 0, st>>>(codes, n, chunk, lengths, chunk_offsets, nch, d_status);
  const uint64_t nb = (nch + SCAN_TILE - 1) / SCAN_TILE;
  uint64_t* sums = reinterpret_cast<uint64_t*>(scratch);
  k_scan_sums<<<(unsigned)nb, SCAN_T, 0, st>>>(chunk_offsets, nch, sums);
  k_scan_top<<<1, SCAN_T, 0, st>>>(sums, nb);
  k_scan_apply<<<(unsigned)nb, SCAN_T, 0, st>>>(chunk_offsets, nch, sums, nb);
  const unsigned ge = (unsigned)std::min<uint64_t>((nch + ENC_WARPS - 1) / ENC_WARPS, (uint64_t)sms * 8);
  k_huff_encode<<<ge, ENC_WARPS * 32, 0, st>>>(codes, n, chunk, lengths, codewords, chunk_offsets, nch, payload,
                                               payload_cap_words, d_status);
  return hf_check(5);
}

int sz3g_huffman_decode(const uint32_t* payload, const uint64_t* chunk_offsets, uint64_t n, uint32_t chunk,
                        const void* dtable, uint32_t max_len, uint16_t* codes, int32_t* d_status,
                        sz3g_stream_t stream) {
  if (n == 0) return SZ3G_OK;
  if (!payload || !chunk_offsets || !dtable || !codes || !d_status) return SZ3G_EINVAL;
  if (chunk < 1 || max_len < 1 || max_len > HF_MAX_LEN_LIMIT) return SZ3G_ERANGE;
  if (reinterpret_cast<uintptr_t>(codes) & 15) return SZ3G_EINVAL;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const uint64_t nch = (n + chunk - 1) / chunk;
  k_huff_decode<<<(unsigned)((nch + 255) / 256), 256, 0, st>>>(payload, chunk_offsets, n, chunk,
                                                               reinterpret_cast<const DTab*>(dtable), max_len,
                                                               codes, nch, d_status);
  return hf_check(1);
}

}  // extern "C"
