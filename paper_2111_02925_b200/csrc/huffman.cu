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
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "../../include/sz3g.h"
#include "ptx.cuh"

namespace {

constexpr int HF_THREADS = 512;         // codebook CTA (16 x 512 radix counters = 32 KiB smem)
constexpr int HF_WARPS = HF_THREADS / 32;
constexpr int HF_LUT_BITS = 12;         // decoder first-level table
constexpr int HF_MAXL = 32;             // array bound for per-length tables
constexpr int HF_MAX_LEN_LIMIT = 16;    // format limit (G20): two codes fit in one 32-bit refill

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
  SZ3G_SYNCTHREADS();
  if (w == 0) {
    uint32_t t = lane < HF_WARPS ? s_warp[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    s_warp[lane] = t;   // inclusive totals per warp
  }
  SZ3G_SYNCTHREADS();
  const uint32_t before = w ? s_warp[w - 1] : 0u;
  excl = before + x - v;
  const uint32_t total = s_warp[HF_WARPS - 1];
  SZ3G_SYNCTHREADS();
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
  const bool from_len = hist == nullptr;   // lengths given (a stored canonical codebook): (F) and (G) only
  uint16_t* syms0 = reinterpret_cast<uint16_t*>(dt + 1);   // long-code symbol table: zeroed, so every
  for (uint32_t s = tid; s < nsym; s += HF_THREADS) {         // byte of the decode table is defined
    if (!from_len) lens[s] = 0;
    cws[s] = 0;
    syms0[s] = 0;
  }
  for (uint32_t i = tid; i < (1u << HF_LUT_BITS); i += HF_THREADS) dt->lut[i] = 0;
  if (tid < HF_MAXL) { dt->first[tid] = 0; dt->count[tid] = 0; dt->base[tid] = 0; }
  if (tid <= HF_MAXL) s_blc[tid] = 0;
  SZ3G_SYNCTHREADS();
  if (from_len) {
    // validate: every length <= max_len, at least one symbol, Kraft sum <= 1 (sum 2^(max_len - L) <= 2^max_len)
    __shared__ unsigned long long s_kraft;
    if (tid == 0) s_kraft = 0;
    SZ3G_SYNCTHREADS();
    unsigned long long kr = 0;
    for (uint32_t s = tid; s < nsym; s += HF_THREADS) {
      const uint32_t L = lens[s];
      if (L > max_len) atomicOr(&s_bad, 1u);
      else if (L) {
        kr += 1ull << (max_len - L);
        atomicAdd(&s_blc[L], 1u);
      }
    }
    atomicAdd(&s_kraft, kr);
    SZ3G_SYNCTHREADS();
    uint32_t nact = 0;
    for (int L = 1; L <= HF_MAXL; L++) nact += s_blc[L];
    if (s_bad || nact == 0 || s_kraft > (1ull << max_len)) {
      if (tid == 0) atomicOr(status, (int)SZ3G_STATUS_BAD_HUFFMAN);
      return;
    }
  } else {

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
  SZ3G_SYNCTHREADS();
  const bool bad = s_bad || n == 0 || (max_len < 32 && (1ull << max_len) < n);
  if (bad) {
    if (tid == 0) atomicOr(status, (int)SZ3G_STATUS_BAD_HUFFMAN);
    return;
  }
  if (n == 1) {   // one symbol -> length 1, codeword 0
    if (tid == 0) {
      const uint32_t sym = (uint32_t)(S.keys0[0] & 0xffffu);
      lens[sym] = 1;
      cws[sym] = 1u << 24;   // length 1, codeword 0
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
    SZ3G_SYNCTHREADS();
    // exclusive scan over (digit, thread) in digit-major order: thread t owns entries [16t, 16t + 16)
    uint32_t loc[16], sum = 0;
#pragma unroll
    for (int e = 0; e < 16; e++) { loc[e] = sum; sum += s_cnt[16 * tid + e]; }
    uint32_t base;
    block_excl_scan(sum, s_warp, base);
#pragma unroll
    for (int e = 0; e < 16; e++) s_cnt[16 * tid + e] = base + loc[e];
    SZ3G_SYNCTHREADS();
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
    SZ3G_SYNCTHREADS();
    uint64_t* t = src; src = dst; dst = t;
  }
  // sorted keys in src; leaf weights in listA (level max_len list)
  uint64_t* leaves = dst;   // reuse the other sort buffer for the leaf weights
  for (uint32_t i = tid; i < n; i += HF_THREADS) leaves[i] = src[i] >> 16;
  for (uint32_t i = tid; i < n; i += HF_THREADS) S.listA[i] = leaves[i];
  SZ3G_SYNCTHREADS();

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
    SZ3G_SYNCTHREADS();
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
    SZ3G_SYNCTHREADS();
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
  SZ3G_SYNCTHREADS();
  // (E) lengths of the sorted leaves: len(i) = #{l : i < c[l]}
  for (uint32_t i = tid; i < n; i += HF_THREADS) {
    uint32_t L = 0;
    for (uint32_t l = 1; l <= max_len; l++) L += i < s_c[l] ? 1u : 0u;
    lens[(uint32_t)(src[i] & 0xffffu)] = (uint8_t)L;
    atomicAdd(&s_blc[L], 1u);
  }
  }   // !from_len
  SZ3G_SYNCTHREADS();
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
  SZ3G_SYNCTHREADS();
  uint32_t* s_run = s_cnt;            // running count per length over earlier rounds
  uint32_t* s_wl = s_cnt + 64;        // [HF_WARPS][32 lengths] counts of the current round
  for (int i = tid; i < 64 + HF_WARPS * 32; i += HF_THREADS) s_cnt[i] = 0;
  SZ3G_SYNCTHREADS();
  const int lane = tid & 31, wid = tid >> 5;
  uint16_t* syms = reinterpret_cast<uint16_t*>(dt + 1);
  for (uint32_t r0 = 0; r0 < nsym; r0 += HF_THREADS) {
    const uint32_t s = r0 + tid;
    const uint32_t L = s < nsym ? lens[s] : 0u;
    const uint32_t peers = __match_any_sync(0xffffffffu, L);
    const uint32_t rank_w = __popc(peers & ((1u << lane) - 1u));
    if (lane == 31 - __clz(peers)) s_wl[wid * 32 + L] = __popc(peers);   // the group's highest lane
    SZ3G_SYNCTHREADS();
    if (L > 0) {
      uint32_t before = s_run[L];
      for (int w = 0; w < wid; w++) before += s_wl[w * 32 + L];
      const uint32_t cw = s_first[L] + before + rank_w;
      cws[s] = (L << 24) | cw;   // packed: length in the top 8 bits
      if (L <= HF_LUT_BITS) {
        const uint32_t lo = cw << (HF_LUT_BITS - L), cnt = 1u << (HF_LUT_BITS - L);
        for (uint32_t e = 0; e < cnt; e++) dt->lut[lo + e] = (L << 16) | s;
      } else {
        syms[dt->base[L] + (cw - s_first[L])] = (uint16_t)s;
      }
    }
    SZ3G_SYNCTHREADS();
    if (tid < 32) {   // fold this round's per-warp counts into the running counts, clear them
      uint32_t add = 0;
      for (int w = 0; w < HF_WARPS; w++) { add += s_wl[w * 32 + tid]; s_wl[w * 32 + tid] = 0; }
      s_run[tid] += add;
    }
    SZ3G_SYNCTHREADS();
  }
}

// ------------------------------------------------------------------------------------------------
// encode
constexpr uint32_t ENC_MAX_CHUNK_W = 2048;   // the format's chunk (k_huff_chunk_words fast path)

__global__ void __launch_bounds__(256) k_huff_chunk_words(const uint16_t* __restrict__ codes, uint64_t n,
                                                          uint32_t chunk, const uint32_t* __restrict__ tab,
                                                          uint32_t nsym, uint64_t* __restrict__ words, uint64_t nch,
                                                          int32_t* status, uint64_t c_begin) {
  const uint64_t warp = c_begin + ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5);
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  const bool vec = (chunk % 8 == 0) && ((reinterpret_cast<uintptr_t>(codes) & 15) == 0);
  for (uint64_t c = warp; c < nch; c += nw) {
    const uint64_t e0 = c * chunk, e1 = min(n, e0 + chunk);
    uint64_t bits = 0;
    bool miss = false;
    auto add = [&](uint32_t q) {
      const uint32_t L = q < nsym ? (__ldg(tab + q) >> 24) : 0u;
      bits += L;
      miss |= L == 0;
    };
    if (vec && chunk == ENC_MAX_CHUNK_W && e1 - e0 == ENC_MAX_CHUNK_W) {
      // full 2048-code chunk: the lane's 8 loads are issued together (one DRAM latency per chunk)
      const uint4* g = reinterpret_cast<const uint4*>(codes + e0) + lane;
      uint4 u[8];
#pragma unroll
      for (int k = 0; k < 8; k++) u[k] = __ldcs(g + 32 * k);
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const uint32_t w[4] = {u[k].x, u[k].y, u[k].z, u[k].w};
#pragma unroll
        for (int h = 0; h < 8; h++) add((w[h >> 1] >> (16 * (h & 1))) & 0xffffu);
      }
    } else if (vec) {   // 8 codes per 16-byte load (the chunk start is 16-byte aligned)
      const uint4* g = reinterpret_cast<const uint4*>(codes + e0);
      const uint32_t m = (uint32_t)(e1 - e0);
      for (uint32_t i = lane; 8 * i < m; i += 32) {
        const uint4 u = __ldg(g + i);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
        if (8 * i + 8 <= m) {
#pragma unroll
          for (int h = 0; h < 8; h++) add((w[h >> 1] >> (16 * (h & 1))) & 0xffffu);
        } else {
          for (uint32_t h = 0; 8 * i + h < m; h++) add((w[h >> 1] >> (16 * (h & 1))) & 0xffffu);
        }
      }
    } else {
      for (uint64_t e = e0 + lane; e < e1; e += 32) add(codes[e]);
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
  SZ3G_SYNCTHREADS();
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
  SZ3G_SYNCTHREADS();
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
    SZ3G_SYNCTHREADS();
    uint64_t before = 0;
    for (int k = 0; k < w; k++) before += s_w[k];
    const uint64_t carry = s_carry;
    if (i < nb) sums[i] = carry + before + x - v;
    SZ3G_SYNCTHREADS();
    if (threadIdx.x == SCAN_T - 1) s_carry = carry + before + x;
    SZ3G_SYNCTHREADS();
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
  SZ3G_SYNCTHREADS();
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

// One warp per chunk (chunk <= 32 * 64 codes).  The chunk's codes are staged in shared memory with
// coalesced 16-byte loads (uint4 i stored at slot i ^ ((i >> 3) & 7): conflict-free both when the
// warp writes consecutive uint4 and when lane l reads its own 8 consecutive uint4).  Lane l owns codes
// [64 l, 64 l + 64) of the chunk: their bit count, a warp scan for the lane's first bit, then the
// lane packs whole words of the chunk image (its first and last word shared -> atomicOr).  One
// lookup per code in the packed table (length << 24 | codeword).
constexpr int ENC_WARPS = 4, ENC_PER = 64, ENC_MAX_CHUNK = 32 * ENC_PER;   // 4 x (4 KiB image + 4 KiB codes)
constexpr int ENC_WORDS = ENC_MAX_CHUNK * HF_MAX_LEN_LIMIT / 32 + 1;
__device__ __forceinline__ uint32_t swz(uint32_t i) { return i ^ ((i >> 3) & 7u); }

struct Packer {
  uint64_t buf;
  uint32_t nbuf, wi;
  bool first;
  __device__ __forceinline__ void put(uint32_t t, uint32_t* img) {
    const uint32_t L = t >> 24;
    buf = (buf << L) | (t & 0xffffffu);
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
};

__global__ void __launch_bounds__(ENC_WARPS * 32) k_huff_encode(const uint16_t* __restrict__ codes, uint64_t n,
                                                                uint32_t chunk, const uint32_t* __restrict__ tab,
                                                                uint32_t nsym, const uint64_t* __restrict__ offs,
                                                                uint64_t nch, uint32_t* __restrict__ payload,
                                                                uint64_t cap, int32_t* status, uint64_t c_begin) {
  __shared__ uint32_t s_img[ENC_WARPS][ENC_WORDS];
  __shared__ uint4 s_codes[ENC_WARPS][ENC_MAX_CHUNK / 8];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  uint32_t* img = s_img[wl];
  uint4* sc = s_codes[wl];
  const uint64_t gw = c_begin + ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5);
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const bool vec = (chunk == ENC_MAX_CHUNK) && ((reinterpret_cast<uintptr_t>(codes) & 15) == 0);
  const uint32_t per = vec ? ENC_PER : (chunk + 31) / 32;
  const uint32_t* __restrict__ tb = tab;
  const uint32_t ns = nsym;
  // codes >= nsym were flagged BAD_HUFFMAN by k_huff_chunk_words; clamping (instead of a guard) keeps
  // the lookup branch-free and the table pointer in a register
  const uint32_t smax = ns - 1;
  auto look = [tb, smax](uint32_t q) -> uint32_t { return __ldg(tb + min(q, smax)); };
  for (uint64_t c = gw; c < nch; c += nw) {
    const uint64_t e0 = c * chunk, e1 = min(n, e0 + chunk);
    const uint64_t w0 = offs[c], nwords = offs[c + 1] - w0;
    if (offs[c + 1] > cap) {   // capacity exceeded: nothing of this chunk is written
      if (lane == 0) atomicOr(status, (int)SZ3G_STATUS_PAYLOAD_OVERFLOW);
      continue;
    }
    for (uint32_t i = lane; i < nwords; i += 32) img[i] = 0u;
    const uint32_t m = (uint32_t)(e1 - e0);
    const uint32_t a0 = min(m, (uint32_t)lane * per), a1 = min(m, a0 + per);
    const bool fullc = vec && m == ENC_MAX_CHUNK;
    uint32_t bits = 0;
    if (vec) {
      const uint4* g = reinterpret_cast<const uint4*>(codes + e0);
      for (uint32_t i = lane; i < ENC_MAX_CHUNK / 8; i += 32)
        sc[swz(i)] = 8 * i < m ? __ldg(g + i) : make_uint4(0, 0, 0, 0);
      SZ3G_SYNCWARP();
    }
    if (fullc) {
#pragma unroll 2
      for (uint32_t v = 0; v < ENC_PER / 8; v++) {
        const uint4 u = sc[swz(lane * 8 + v)];
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int h = 0; h < 8; h++) bits += look((w[h >> 1] >> (16 * (h & 1))) & 0xffffu) >> 24;
      }
    } else if (vec) {
      for (uint32_t e = a0; e < a1; e++) {
        const uint4 u = sc[swz(e >> 3)];
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
        bits += look((w[(e & 7) >> 1] >> (16 * (e & 1))) & 0xffffu) >> 24;
      }
    } else {
      for (uint32_t e = a0; e < a1; e++) bits += look(codes[e0 + e]) >> 24;
    }
    uint32_t incl = bits;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t b0 = incl - bits;   // first bit of this lane inside the chunk
    SZ3G_SYNCWARP();                      // the image is zeroed before any lane writes into it
    // pack: the buffer starts with the (b0 % 32) bits of the previous lane as zeros, so every emitted
    // word is a whole word of the chunk image; the first and the last are shared -> atomicOr
    Packer pk{0, b0 & 31u, b0 >> 5, true};
    if (fullc) {
#pragma unroll 2
      for (uint32_t v = 0; v < ENC_PER / 8; v++) {
        const uint4 u = sc[swz(lane * 8 + v)];
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
        uint32_t t[8];
#pragma unroll
        for (int h = 0; h < 8; h++) t[h] = look((w[h >> 1] >> (16 * (h & 1))) & 0xffffu);
#pragma unroll
        for (int h = 0; h < 8; h++) pk.put(t[h], img);
      }
    } else if (vec) {
      for (uint32_t e = a0; e < a1; e++) {
        const uint4 u = sc[swz(e >> 3)];
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
        pk.put(look((w[(e & 7) >> 1] >> (16 * (e & 1))) & 0xffffu), img);
      }
    } else {
      for (uint32_t e = a0; e < a1; e++) pk.put(look(codes[e0 + e]), img);
    }
    if (pk.nbuf > 0 && bits > 0) atomicOr(&img[pk.wi], (uint32_t)(pk.buf << (32 - pk.nbuf)));
    SZ3G_SYNCWARP();
    for (uint32_t i = lane; i < nwords; i += 32) payload[w0 + i] = img[i];
    SZ3G_SYNCWARP();
  }
}

// ------------------------------------------------------------------------------------------------
// Full-chunk fast path (chunk = 2048 codes, 16-byte aligned codes): the bulk of every field.
//
// The codes of a field concentrate around the radius (the histogram's mass is near R), so each CTA
// stages a window of EW_TW table entries centred on nsym / 2 in shared memory and looks codes up there;
// a group of 8 codes with any code outside the window takes the global table for that group (warp
// vote).  One warp per chunk; chunks are loaded one chunk ahead into registers with coalesced 16-byte
// loads (load v of lane l = uint4 32 v + l of the chunk).
//
// k_huff_chunk_words_full: the bit count of every group of 64 consecutive codes (uint4 8 g .. 8 g + 7
// of the chunk) from a byte table of lengths -- the 8-lane sums of the coalesced layout -- then the
// chunk's word count and, per group g, its first bit inside the chunk (u16, `loff`).
// k_huff_encode_full: lane g owns group g (its 64 codes restaged through shared memory) and its first
// bit is known from `loff`, so it packs its codes MSB-first straight into the chunk image at their
// final place: pairs of codes are joined into one <= 32-bit unit and appended to a 64-bit accumulator,
// every completed word is stored.  A lane that does not start on a word boundary stores its first word
// with the previous lane's bits as zeros; after a warp barrier the previous lane ORs its partial last
// word into it.  No atomics, no zeroing.  The image sits at word (w0 mod 4) so that it leaves with 16-byte stores.
// A chunk holding a code without a codeword is flagged (BAD_HUFFMAN) and gets 0 words.
constexpr int EW_TW = 8192, EW_WARPS = 16, EW_CHUNK = 2048;
constexpr int EW_IMG = ENC_WORDS + 3;   // 1028 words per warp (a <= 3 words of alignment + 1025)

__device__ __forceinline__ uint32_t ew_lo(uint32_t nsym) { return nsym > EW_TW ? nsym / 2 - EW_TW / 2 : 0u; }

// 8 codes of a uint4 -> idx - lo packed per half word; true if every code is inside the window.  A code
// below lo borrows from the next half (or wraps the top half), which makes that half >= EW_TW: the
// window test catches every case (lo <= 65536 - EW_TW - 1).
__device__ __forceinline__ bool ew_in_window(const uint4 u, uint32_t lo2, uint32_t (&d)[4]) {
  d[0] = u.x - lo2; d[1] = u.y - lo2; d[2] = u.z - lo2; d[3] = u.w - lo2;
  constexpr uint32_t oor = ((~(uint32_t)(EW_TW - 1)) & 0xffffu) * 0x10001u;
  return ((d[0] | d[1] | d[2] | d[3]) & oor) == 0u;
}

// coalesced: load v of lane l is uint4 v * 32 + l of the chunk
__device__ __forceinline__ void ew_load_chunk(const uint16_t* __restrict__ codes, uint64_t c, int lane, uint4 (&u)[8]) {
  const uint4* g = reinterpret_cast<const uint4*>(codes + c * EW_CHUNK) + lane;
#pragma unroll
  for (int v = 0; v < 8; v++) u[v] = __ldcs(g + 32 * v);
}

// stage the loaded chunk in shared memory (uint4 i at slot swz(i)) and read back the lane's own 64
// consecutive codes (uint4 8 l .. 8 l + 7): conflict-free both ways
__device__ __forceinline__ void ew_restage(const uint4 (&nx)[8], uint4* st, int lane, uint4 (&u)[8]) {
#pragma unroll
  for (int v = 0; v < 8; v++) st[swz(v * 32 + lane)] = nx[v];
  SZ3G_SYNCWARP();
#pragma unroll
  for (int v = 0; v < 8; v++) u[v] = st[swz(lane * 8 + v)];
  SZ3G_SYNCWARP();
}

__global__ void __launch_bounds__(EW_WARPS * 32, 1) k_huff_chunk_words_full(const uint16_t* __restrict__ codes,
                                                                            uint64_t nfull,
                                                                            const uint32_t* __restrict__ tab,
                                                                            uint32_t nsym,
                                                                            uint64_t* __restrict__ words,
                                                                            uint16_t* __restrict__ loff,
                                                                            int32_t* status) {
  // byte table (4 symbols per bank word: few bank conflicts for codes concentrated near R): the code
  // length, or 0x80 for a symbol without a codeword (OR-accumulated into the miss flag)
  __shared__ uint8_t s_len[EW_TW];
  const uint32_t lo = ew_lo(nsym), lo2 = lo | (lo << 16);
  for (uint32_t i = threadIdx.x; i < EW_TW; i += blockDim.x) {
    const uint32_t L = lo + i < nsym ? __ldg(tab + lo + i) >> 24 : 0u;
    s_len[i] = (uint8_t)(L ? L : 0x80u);
  }
  SZ3G_SYNCTHREADS();
  const int lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * EW_WARPS;
  uint64_t c = (uint64_t)blockIdx.x * EW_WARPS + (threadIdx.x >> 5);
  if (c >= nfull) return;
  uint4 nx[8];
  ew_load_chunk(codes, c, lane, nx);
  for (; c < nfull; c += nw) {
    uint4 u[8];
#pragma unroll
    for (int v = 0; v < 8; v++) u[v] = nx[v];
    // unconditional prefetch (the last iteration reloads its own chunk): a predicated load would be
    // merged into the live registers and waited for at once
    ew_load_chunk(codes, c + nw < nfull ? c + nw : c, lane, nx);
    uint32_t sv[8], miss = 0;   // sv[v]: bits of the lane's uint4 32 v + lane
#pragma unroll
    for (int v = 0; v < 8; v++) {
      uint32_t d[4];
      sv[v] = 0;
      if (__all_sync(0xffffffffu, ew_in_window(u[v], lo2, d))) {
#pragma unroll
        for (int k = 0; k < 4; k++) {
          const uint32_t la = s_len[d[k] & 0xffffu], lb = s_len[d[k] >> 16];
          sv[v] += la + lb;
          miss |= la | lb;
        }
      } else {
        const uint32_t w[4] = {u[v].x, u[v].y, u[v].z, u[v].w};
#pragma unroll
        for (int h = 0; h < 8; h++) {
          const uint32_t q = (w[h >> 1] >> (16 * (h & 1))) & 0xffffu;
          const uint32_t L = q < nsym ? __ldg(tab + q) >> 24 : 0u;
          sv[v] += L;
          miss |= L ? 0u : 0x80u;
        }
      }
    }
    // uint4 32 v + l belongs to group 4 v + l / 8, so group 4 v + s is the sum of sv[v] over the 8
    // lanes of segment s.  Butterfly reduce-scatter inside the segment (7 shuffles): afterwards lane l
    // holds the sum for v = l & 7, i.e. group 4 (l & 7) + l / 8; one more shuffle gives lane g group g.
    uint32_t r4[4], r2[2];
    {
      const bool hb = (lane >> 2) & 1;
#pragma unroll
      for (int j = 0; j < 4; j++)
        r4[j] = (hb ? sv[j + 4] : sv[j]) + __shfl_xor_sync(0xffffffffu, hb ? sv[j] : sv[j + 4], 4);
    }
    {
      const bool hb = (lane >> 1) & 1;
#pragma unroll
      for (int j = 0; j < 2; j++)
        r2[j] = (hb ? r4[j + 2] : r4[j]) + __shfl_xor_sync(0xffffffffu, hb ? r4[j] : r4[j + 2], 2);
    }
    const bool hb0 = lane & 1;
    const uint32_t fin = (hb0 ? r2[1] : r2[0]) + __shfl_xor_sync(0xffffffffu, hb0 ? r2[0] : r2[1], 1);
    const uint32_t mine = __shfl_sync(0xffffffffu, fin, 8 * (lane & 3) + (lane >> 2));
    const bool bad = __any_sync(0xffffffffu, (miss & 0x80u) != 0);
    uint32_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    loff[c * 32 + lane] = bad ? (uint16_t)0 : (uint16_t)(incl - mine);
    if (lane == 31) {
      if (bad) atomicOr(status, (int)SZ3G_STATUS_BAD_HUFFMAN);
      words[c] = bad ? 0 : (incl + 31) / 32;
    }
  }
}

__global__ void __launch_bounds__(EW_WARPS * 32, 1) k_huff_encode_full(const uint16_t* __restrict__ codes,
                                                                       uint64_t nfull,
                                                                       const uint32_t* __restrict__ tab,
                                                                       uint32_t nsym,
                                                                       const uint64_t* __restrict__ offs,
                                                                       const uint16_t* __restrict__ loff,
                                                                       uint32_t* __restrict__ payload, uint64_t cap,
                                                                       int32_t* status) {
  extern __shared__ __align__(16) uint32_t esm[];
  uint32_t* s_tab = esm;                                   // [EW_TW] (L << 16) | codeword
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  uint32_t* img = esm + EW_TW + wl * EW_IMG;
  const uint32_t lo = ew_lo(nsym), lo2 = lo | (lo << 16), smax = nsym - 1;
  for (uint32_t i = threadIdx.x; i < EW_TW; i += blockDim.x) {
    const uint32_t t = lo + i < nsym ? __ldg(tab + lo + i) : 0u;
    s_tab[i] = ((t >> 24) << 16) | (t & 0xffffu);
  }
  SZ3G_SYNCTHREADS();
  const uint64_t nw = (uint64_t)gridDim.x * EW_WARPS;
  uint64_t c = (uint64_t)blockIdx.x * EW_WARPS + wl;
  if (c >= nfull) return;
  const bool vec_out = (reinterpret_cast<uintptr_t>(payload) & 15) == 0;
  uint4 nx[8];
  ew_load_chunk(codes, c, lane, nx);
  uint64_t nw0 = offs[c], nw1 = offs[c + 1];
  uint32_t nb0 = loff[c * 32 + lane];
  for (; c < nfull; c += nw) {
    uint4 u[8];
    const uint64_t w0 = nw0, w1 = nw1;
    const uint32_t b0 = nb0;
    const uint32_t a = (uint32_t)(w0 & 3u);
    ew_restage(nx, reinterpret_cast<uint4*>(img), lane, u);   // the image is free until packing
    {   // unconditional prefetch of the next chunk and its offsets (the last iteration reloads its own)
      const uint64_t cn = c + nw < nfull ? c + nw : c;
      ew_load_chunk(codes, cn, lane, nx);
      nw0 = offs[cn];
      nw1 = offs[cn + 1];
      nb0 = loff[cn * 32 + lane];
    }
    // pack: the accumulator starts with (b0 mod 32) zero bits (the previous lane's part of the first word)
    const uint32_t sh = b0 & 31u;
    uint32_t* dst = img + a + (b0 >> 5);
    uint64_t acc = 0;
    uint32_t nb = sh, wi = 0;
#pragma unroll
    for (int v = 0; v < 8; v++) {
      uint32_t d[4], e[8];
      if (__all_sync(0xffffffffu, ew_in_window(u[v], lo2, d))) {
#pragma unroll
        for (int k = 0; k < 4; k++) {
          e[2 * k] = s_tab[d[k] & 0xffffu];
          e[2 * k + 1] = s_tab[d[k] >> 16];
        }
      } else {
        const uint32_t w[4] = {u[v].x, u[v].y, u[v].z, u[v].w};
#pragma unroll
        for (int h = 0; h < 8; h++) {   // codes >= nsym are flagged by the size pass; clamp like it
          const uint32_t t = __ldg(tab + min((w[h >> 1] >> (16 * (h & 1))) & 0xffffu, smax));
          e[h] = ((t >> 24) << 16) | (t & 0xffffu);
        }
      }
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const uint32_t ea = e[2 * k], eb = e[2 * k + 1];
        const uint32_t lb = eb >> 16;
        const uint32_t pl = (ea >> 16) + lb;                              // <= 32 bits
        const uint32_t pv = ((ea & 0xffffu) << lb) | (eb & 0xffffu);
        acc = (acc << pl) | pv;
        nb += pl;
        if (nb >= 32) {
          nb -= 32;
          dst[wi++] = (uint32_t)(acc >> nb);
        }
      }
    }
    // the partial last word continues in the next lane, which has stored its part there (its first
    // word, the upper bits zero); lane 31's is the chunk's zero-padded last word
    SZ3G_SYNCWARP();
    const uint32_t nhead = (nb && lane < 31) ? dst[wi] : 0u;
    SZ3G_SYNCWARP();
    if (nb) dst[wi] = (uint32_t)(acc << (32 - nb)) | nhead;
    SZ3G_SYNCWARP();
    // out
    const uint32_t nwords = (uint32_t)(w1 - w0);
    if (w1 > cap) {
      if (lane == 0) atomicOr(status, (int)SZ3G_STATUS_PAYLOAD_OVERFLOW);
    } else {
      uint32_t* gout = payload + (w0 - a);    // 16-byte aligned when payload is
      const uint32_t e_ = a + nwords, v0 = (a + 3) >> 2, v1 = e_ >> 2;
      if (vec_out && v0 <= v1) {
        for (uint32_t k = v0 + lane; k < v1; k += 32)
          reinterpret_cast<uint4*>(gout)[k] = reinterpret_cast<const uint4*>(img)[k];
        if (lane < 4 * v0 - a) gout[a + lane] = img[a + lane];               // head words
        if (lane < e_ - 4 * v1) gout[4 * v1 + lane] = img[4 * v1 + lane];    // tail words
      } else {
        for (uint32_t i = a + lane; i < e_; i += 32) gout[i] = img[i];
      }
    }
    SZ3G_SYNCWARP();
  }
}

size_t ew_smem_bytes() { return 4ull * (EW_TW + EW_WARPS * EW_IMG); }


// ------------------------------------------------------------------------------------------------
// decode: one thread per chunk, warp-synchronous staging.  Lane l of a warp decodes chunk
// (warp base + l), one code per step.  Codes are at most 16 bits, so a round of 32 steps consumes at
// most 16 payload words per lane: at the start of every round the warp tops up, with coalesced
// 64-byte loads (half a warp per chunk), the per-lane ring of 32 words in shared memory (rows padded
// to 33 words: no bank conflicts when every lane reads its own row).  Lanes refill their 64-bit bit
// window from their ring once per pair of codes (a pair needs <= 32 bits).  Decoded codes go to a
// per-lane row of 32 codes in shared memory, written out after each round with one coalesced
// 64-byte store per chunk.  Codes longer than the 12-bit LUT take a branch-free canonical length
// search (3 compares), guarded by a warp vote.
constexpr int DEC_WARPS = 8, DEC_ROUND = 32, RING = 32, RING_P = RING + 1, OUT_P = DEC_ROUND / 2 + 1;

struct DecLane {
  uint64_t win;      // left-aligned bit window (zeros past the end of the chunk)
  uint32_t avail;    // valid bits in win
  uint32_t r;        // next word (relative to the chunk start) to append to the window
  uint32_t filled;   // words [0, filled) of the chunk have been staged into the ring
  uint32_t nwords;   // words of this chunk
  uint32_t consumed; // bits decoded (steps before the chunk end)
};

__device__ __forceinline__ uint32_t dec_one(DecLane& d, const uint32_t* s_lut, const uint32_t* s_ljl,
                                            const uint32_t* s_first, const uint32_t* s_base,
                                            const uint16_t* __restrict__ syms, uint32_t maxl, bool& bad,
                                            bool active) {
  const uint32_t top = (uint32_t)(d.win >> 48);   // next 16 bits
  const uint32_t ent = s_lut[top >> (16 - HF_LUT_BITS)];
  uint32_t L = ent >> 16, sym = ent & 0xffffu;
  if (__any_sync(0xffffffffu, ent == 0u)) {
    if (ent == 0u) {   // canonical: the smallest l > 12 whose left-justified limit exceeds top
      L = HF_LUT_BITS + 1 + (top >= s_ljl[13] ? 1u : 0u) + (top >= s_ljl[14] ? 1u : 0u) + (top >= s_ljl[15] ? 1u : 0u);
      if (L > maxl || top >= s_ljl[L]) { bad |= active; L = 1; sym = 0; }
      else sym = syms[s_base[L] + (top >> (16 - L)) - s_first[L]];
    }
  }
  d.win <<= L;
  d.avail -= L;
  d.consumed += active ? L : 0u;   // steps past the end of a short chunk do not count
  return sym;
}

__device__ __forceinline__ void dec_refill(DecLane& d, const uint32_t* ring) {
  if (d.avail <= 32) {
    const uint32_t w = d.r < d.nwords ? ring[d.r % RING] : 0u;
    d.win |= (uint64_t)w << (32 - d.avail);
    d.avail += 32;
    d.r++;
  }
}

__global__ void __launch_bounds__(DEC_WARPS * 32) k_huff_decode(const uint32_t* __restrict__ payload,
                                                                const uint64_t* __restrict__ offs, uint64_t n,
                                                                uint32_t chunk, const DTab* __restrict__ dt,
                                                                uint32_t max_len, uint16_t* __restrict__ codes,
                                                                uint64_t nch, int32_t* status, uint64_t c_begin) {
  extern __shared__ __align__(16) uint32_t dsm[];
  uint32_t* s_lut = dsm;                                  // 4096
  uint32_t* s_first = s_lut + (1 << HF_LUT_BITS);         // 32
  uint32_t* s_base = s_first + HF_MAXL;
  uint32_t* s_ljl = s_base + HF_MAXL;
  uint32_t* s_ring = s_ljl + HF_MAXL;                     // [DEC_WARPS][32 lanes][RING_P]
  uint32_t* s_out = s_ring + DEC_WARPS * 32 * RING_P;     // [DEC_WARPS][32 lanes][OUT_P]
  for (int i = threadIdx.x; i < (1 << HF_LUT_BITS); i += blockDim.x) s_lut[i] = dt->lut[i];
  if (threadIdx.x < HF_MAXL) {
    const uint32_t l = threadIdx.x;
    s_first[l] = dt->first[l];
    s_base[l] = dt->base[l];
    // left-justified (16-bit) limit of length l; lengths above max_len are unreachable
    s_ljl[l] = (l >= 1 && l <= max_len) ? (uint32_t)(((uint64_t)dt->first[l] + dt->count[l]) << (16 - l))
                                        : (l > max_len ? 0x10000u : 0u);
  }
  SZ3G_SYNCTHREADS();
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  uint32_t* ring_w = s_ring + wl * 32 * RING_P;
  uint32_t* ring = ring_w + lane * RING_P;
  uint32_t* out_w = s_out + wl * 32 * OUT_P;
  uint32_t* out = out_w + lane * OUT_P;
  const uint16_t* syms = reinterpret_cast<const uint16_t*>(dt + 1);
  const uint64_t cbase = c_begin + ((uint64_t)blockIdx.x * DEC_WARPS + wl) * 32;
  if (cbase >= nch) return;
  const uint64_t c = cbase + lane;
  const bool live = c < nch;
  const uint64_t cc = live ? c : nch - 1;
  const uint64_t e0 = cc * chunk;
  const uint32_t m = live ? (uint32_t)(min(n, e0 + chunk) - e0) : 0u;
  const uint64_t w0 = offs[cc];
  DecLane d;
  d.nwords = live ? (uint32_t)(offs[cc + 1] - w0) : 0u;
  d.win = 0;
  d.avail = 0;
  d.r = 0;
  d.filled = 0;
  d.consumed = 0;
  bool bad = false;
  const uint32_t steps = __reduce_max_sync(0xffffffffu, m);
  const int half = lane >> 4, hl = lane & 15;
  for (uint32_t e = 0; e < steps; e += DEC_ROUND) {
    // (1) top up every ring that holds fewer than 16 unread words (the first round: 32, since the
    // window is primed with 2 words first): 16 words per lane, 2 lanes per pass.  A fill overwrites
    // words [filled - 32, filled - 16), all consumed since filled < r + 16.
    for (int pass = 0; pass < (e == 0 ? 2 : 1); pass++) {
      const bool need = d.filled < d.r + 16 + (e == 0 ? 16u : 0u) && d.filled < d.nwords;
      if (__any_sync(0xffffffffu, need)) {
        // pass j serves chunk 2j + half: all 16 loads are issued before any store
        uint32_t v[16];
#pragma unroll
        for (int j = 0; j < 16; j++) {
          const int src = 2 * j + half;
          const bool nd = __shfl_sync(0xffffffffu, need, src);
          const uint32_t fl = __shfl_sync(0xffffffffu, d.filled, src);
          const uint32_t nw = __shfl_sync(0xffffffffu, d.nwords, src);
          const uint64_t gw = __shfl_sync(0xffffffffu, w0, src);
          const uint32_t wi = fl + hl;
          v[j] = (nd && wi < nw) ? __ldg(payload + gw + wi) : 0u;
        }
#pragma unroll
        for (int j = 0; j < 16; j++) {
          const int src = 2 * j + half;
          const bool nd = __shfl_sync(0xffffffffu, need, src);
          const uint32_t fl = __shfl_sync(0xffffffffu, d.filled, src);
          if (nd) ring_w[src * RING_P + (fl + hl) % RING] = v[j];
        }
        if (need) d.filled += 16;
      }
      SZ3G_SYNCWARP();
    }
    if (e == 0) {   // prime the window: 64 bits
      dec_refill(d, ring);
      dec_refill(d, ring);
    }
    // (2) 32 steps: 16 pairs of codes
    if (__all_sync(0xffffffffu, e + DEC_ROUND <= m)) {
      // every lane decodes 32 real codes this round: no per-code bookkeeping; both codes of a pair go
      // through the LUT and one warp vote per pair catches codes longer than the LUT -- the pair is then
      // decoded again, code by code, from the saved window
#pragma unroll 4
      for (int h = 0; h < DEC_ROUND; h += 2) {
        const uint64_t win0 = d.win;
        const uint32_t top1 = (uint32_t)(win0 >> 48);
        const uint32_t ea = s_lut[top1 >> (16 - HF_LUT_BITS)];
        const uint32_t La = ea >> 16;
        const uint64_t win1 = win0 << La;
        const uint32_t eb = s_lut[(uint32_t)(win1 >> 48) >> (16 - HF_LUT_BITS)];
        const uint32_t Lb = eb >> 16;
        uint32_t a, b;
        if (__any_sync(0xffffffffu, ea == 0u || eb == 0u)) {
          a = dec_one(d, s_lut, s_ljl, s_first, s_base, syms, max_len, bad, true);
          b = dec_one(d, s_lut, s_ljl, s_first, s_base, syms, max_len, bad, true);
        } else {
          a = ea & 0xffffu;
          b = eb & 0xffffu;
          d.win = win1 << Lb;
          d.avail -= La + Lb;
          d.consumed += La + Lb;
        }
        dec_refill(d, ring);
        out[h >> 1] = a | (b << 16);
      }
    } else {
#pragma unroll 4
      for (int h = 0; h < DEC_ROUND; h += 2) {
        const uint32_t a = dec_one(d, s_lut, s_ljl, s_first, s_base, syms, max_len, bad, e + h < m);
        const uint32_t b = dec_one(d, s_lut, s_ljl, s_first, s_base, syms, max_len, bad, e + h + 1 < m);
        dec_refill(d, ring);
        out[h >> 1] = a | (b << 16);
      }
    }
    SZ3G_SYNCWARP();
    // (3) write the round's codes: one chunk row (64 B) per half-warp pass
    for (int j = 0; j < 32; j += 2) {
      const int src = j + half;
      const uint32_t mj = __shfl_sync(0xffffffffu, m, src);
      const uint64_t ej = __shfl_sync(0xffffffffu, e0, src);
      const uint32_t k = e + 2 * hl;   // first code of this lane's word
      const uint32_t v = out_w[src * OUT_P + hl];
      if (k + 1 < mj && ((ej & 1) == 0)) {
        *reinterpret_cast<uint32_t*>(codes + ej + k) = v;
      } else {
        if (k < mj) codes[ej + k] = (uint16_t)v;
        if (k + 1 < mj) codes[ej + k + 1] = (uint16_t)(v >> 16);
      }
    }
    SZ3G_SYNCWARP();
  }
  if (live && (bad || d.consumed > d.nwords * 32u)) atomicOr(status, (int)SZ3G_STATUS_BAD_HUFFMAN);
}

size_t dec_smem_bytes() {
  return 4ull * ((1 << HF_LUT_BITS) + 3 * HF_MAXL + DEC_WARPS * 32 * (RING_P + OUT_P));
}

// ------------------------------------------------------------------------------------------------
// Full-chunk decoder (chunk = 2048 codes, 16-byte aligned payload and codes): one chunk per lane, as
// k_huff_decode, but each lane streams its own payload words through a private ring in
// shared memory (16 words) filled by cp.async (asynchronous global -> shared copies, zero-filled past
// the end of the payload) every 8 codes, so no cooperative top-up and no registers waiting on loads.  Per pair of codes: two 12-bit LUT lookups from the 64-bit window and ONE warp vote
// for codes longer than the LUT (then the pair is decoded code by code with the canonical search).  The
// window takes one ring word whenever it holds <= 32 bits (predicated).  A round's 32 codes stay in
// registers and leave through a swizzled shared-memory stage with 16-byte stores (4 lanes per 64-byte
// chunk row).
constexpr int DF_ROUND = 32, DF_RING = 16, DF_RING_W = 20;   // ring: 16 words, 80-byte row stride
#ifndef SZ3G_DF_DIRECT
#define SZ3G_DF_DIRECT 0   // 1: a round's codes leave with the lane's own 16-byte stores (no staging)
#endif
#ifndef SZ3G_DF_TMA
#define SZ3G_DF_TMA 1      // a round's codes leave by one 2D TMA store per warp (else staged 16-byte stores)
#endif
// Two shapes (the launch picks one, sz3g_huffman_decode):
//  * WARPS = 32, one CTA per SM, persistent (a grid of #SMs CTAs; warp wl of CTA b takes the groups of 32
//    chunks b * 32 + wl, + 32 * gridDim.x, ...): one copy of the tables per SM, built once, and the
//    smallest shared-memory footprint per warp (161 KB for 32 warps against 4 x 54 KB);
//  * WARPS = 8, up to 4 CTAs per SM, one group per warp: fields with fewer groups than 32 per SM would
//    leave SMs idle with the 32-warp CTA.
constexpr int DF_BIG = 32, DF_SMALL = 8;
#ifndef SZ3G_DF_PREF
#define SZ3G_DF_PREF 1   // the window's next ring word loaded one refill ahead, by the taking lanes only
#endif
__host__ __device__ constexpr size_t df_smem_core_bytes(int warps) {   // LUT, per-length tables, rings
  return 4ull * ((1 << HF_LUT_BITS) + 3 * HF_MAXL) + 4ull * warps * 32 * DF_RING_W;
}

struct DfLane {
  uint32_t hi, lo;  // left-aligned 64-bit bit window (hi = its upper 32 bits)
  uint32_t avail;   // valid bits in the window
  uint32_t rp4;     // 4 x (next ring word to read), counted from the aligned chunk start (ring byte = rp4 mod 64)
  uint32_t fp4;     // 4 x (ring words requested so far; 16-byte copies of 4 words)
  uint32_t wn;      // SZ3G_DF_PREF: ring word rp4 / 4, loaded ahead
};

__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

#ifndef SZ3G_DF_CG
#define SZ3G_DF_CG 1        // ring copies bypass L1 (cp.async.cg; .ca measured 5.6 against 4.6 ms on c5)
#endif
#ifndef SZ3G_DF_CARVE
#define SZ3G_DF_CARVE -1    // >= 0: cudaFuncAttributePreferredSharedMemoryCarveout of the decoder (percent)
#endif
#ifndef SZ3G_DF_IMAD
#define SZ3G_DF_IMAD 1
#endif
// shared address of the 12-bit LUT entry indexed by the window's top bits
__device__ __forceinline__ uint32_t df_lut_addr(uint32_t hi, uint32_t k_hi, uint32_t k4, uint32_t lut_sh) {
  if (SZ3G_DF_IMAD) return __umulhi(hi, k_hi) * k4 + lut_sh;   // (hi >> 20) * 4 + base
  return lut_sh + ((hi >> (32 - HF_LUT_BITS)) << 2);
}

// 16 bytes of the lane's payload from byte fp4 of its aligned start pl (lim4 = payload bytes from pl,
// clamped to 2^30), zero-filled past the end of the payload; 32-bit arithmetic only
__device__ __forceinline__ void df_copy16(uint32_t s_dst, const uint8_t* __restrict__ pl, uint32_t fp4,
                                          uint32_t lim4) {
  const uint32_t bytes = fp4 >= lim4 ? 0u : min(16u, lim4 - fp4);
  const uint8_t* src = pl + (fp4 < lim4 ? fp4 : 0u);
  if (SZ3G_DF_CG)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s_dst), "l"(src), "r"(bytes) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(s_dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void df_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void df_wait2() {
  asm volatile("cp.async.wait_group 2;\n" ::: "memory");
  sz3g::ptx::chaos_delay();
}

// top the ring up towards DF_RING = 16 words ahead of the read position (<= K copies of 4 words) and
// wait for the copies requested before the previous call.  Every quarter round (8 codes, <= 4 words
// read) calls it with K = 1: with g = requested - read at a call, the next call sees g' >=
// min(g + 4, 13) - 4 >= min(g, 9), and g starts at 14 (16 words, 2 of them in the primed window); the
// words requested before the previous call reach >= g_prev - 4 >= 5 >= 4 words past the read position.
template <int K>
__device__ __forceinline__ void df_topup(DfLane& d, uint32_t s_ring, const uint8_t* __restrict__ pl, uint32_t lim4) {
#pragma unroll
  for (int k = 0; k < K; k++) {
    if (d.fp4 + 16 <= d.rp4 + 4 * DF_RING) {
      df_copy16(s_ring + (d.fp4 & (4 * DF_RING - 1)), pl, d.fp4, lim4);
      d.fp4 += 16;
    }
  }
  df_commit();
  df_wait2();
}

// append one ring word when the window holds <= 32 bits (then every valid bit is in hi and lo = 0):
// branch-free, a 32-bit shared address, clamped funnel shifts (a shift by 32 gives 0)
__device__ __forceinline__ void df_refill(DfLane& d, uint32_t s_ring) {
  const bool take = d.avail <= 32u;
  const uint32_t w = SZ3G_DF_PREF ? d.wn : lds32(s_ring + (d.rp4 & (4 * DF_RING - 1)));
  const uint32_t add_hi = __funnelshift_rc(w, 0u, d.avail);          // w >> avail (0 at avail = 32)
  const uint32_t new_lo = __funnelshift_lc(0u, w, 32u - d.avail);    // w << (32 - avail) (0 at avail = 0)
  d.hi |= add_hi;   // 0 unless take: the clamped shift by avail >= 33 gives 0
  d.lo = take ? new_lo : d.lo;
  d.avail += take ? 32u : 0u;
  d.rp4 += take ? 4u : 0u;
  if (SZ3G_DF_PREF)   // the next word, by the taking lanes only (predicated load, off the decode chain)
    asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p ld.shared.u32 %0, [%1];\n}"
                 : "+r"(d.wn)
                 : "r"(s_ring + (d.rp4 & (4 * DF_RING - 1))), "r"((uint32_t)take));
}

// shift the window left by L (<= 16) bits
__device__ __forceinline__ void df_shift(DfLane& d, uint32_t L) {
  d.hi = __funnelshift_l(d.lo, d.hi, L);
  d.lo <<= L;
  d.avail -= L;
}

// one code, any length (LUT, else the canonical search of k_huff_decode's dec_one)
__device__ __forceinline__ uint32_t df_code(DfLane& d, uint32_t s_lut, const uint32_t* s_ljl,
                                            const uint32_t* s_first, const uint32_t* s_base,
                                            const uint16_t* __restrict__ syms, uint32_t maxl, bool& bad) {
  const uint32_t top = d.hi >> 16;
  const uint32_t ent = lds32(s_lut + 4u * (top >> (16 - HF_LUT_BITS)));
  uint32_t L = ent >> 16, sym = ent & 0xffffu;
  if (ent == 0u) {
    L = HF_LUT_BITS + 1 + (top >= s_ljl[13] ? 1u : 0u) + (top >= s_ljl[14] ? 1u : 0u) + (top >= s_ljl[15] ? 1u : 0u);
    if (L > maxl || top >= s_ljl[L]) { bad = true; L = 1; sym = 0; }
    else sym = syms[s_base[L] + (top >> (16 - L)) - s_first[L]];
  }
  df_shift(d, L);
  return sym;
}

#ifndef SZ3G_DF_QUARTER
#define SZ3G_DF_QUARTER 1   // TMA-store path: quarter rounds in a rolled loop (see the kernel)
#endif
#ifndef SZ3G_DF_SLOW_CALL
#define SZ3G_DF_SLOW_CALL 0   // 1: the pair slow path out of line (a call): c5 4.36 -> 4.21 ms (fewer i-cache
                              // misses), but c2 (3.9% of codes longer than 12 bits) 0.41 -> 0.55 ms: off
#endif
// both codes of a pair, any length (the slow path): (hi, lo, avail | bad << 31, a | b << 16)
__device__ __noinline__ uint4 df_slow_pair(uint32_t hi, uint32_t lo, uint32_t avail, uint32_t lut_sh,
                                           const uint32_t* s_ljl, const uint32_t* s_first, const uint32_t* s_base,
                                           const uint16_t* __restrict__ syms, uint32_t maxl) {
  DfLane d;
  d.hi = hi;
  d.lo = lo;
  d.avail = avail;
  bool bad = false;
  const uint32_t a = df_code(d, lut_sh, s_ljl, s_first, s_base, syms, maxl, bad);
  const uint32_t b = df_code(d, lut_sh, s_ljl, s_first, s_base, syms, maxl, bad);
  return make_uint4(d.hi, d.lo, d.avail | (bad ? 0x80000000u : 0u), a | (b << 16));
}

template <int DF_WARPS>
__global__ void __launch_bounds__(DF_WARPS * 32, DF_WARPS == DF_BIG ? 1 : 4) k_huff_decode_full(const uint32_t* __restrict__ payload,
                                                                    const uint64_t* __restrict__ offs, uint64_t nch,
                                                                    uint64_t nfull, const DTab* __restrict__ dt,
                                                                    uint32_t max_len, uint16_t* __restrict__ codes,
                                                                    int32_t* status,
                                                                    const __grid_constant__ CUtensorMap tm_out,
                                                                    int tma_out) {
  extern __shared__ __align__(16) uint32_t dsm[];
  // tma_out: a round's codes leave by one TMA store of a {32 codes, 32 chunks} box per warp, staged in a
  // 2 KB buffer per warp laid out as the map's 64-byte swizzle (1024-byte aligned: the XOR pattern
  // follows the address bits)
  uint4* s_tma = reinterpret_cast<uint4*>(
      (reinterpret_cast<uintptr_t>(dsm) + df_smem_core_bytes(DF_WARPS) + 1023) & ~uintptr_t(1023));
  uint32_t* s_lut = dsm;                                  // 4096
  uint32_t* s_first = s_lut + (1 << HF_LUT_BITS);         // 32
  uint32_t* s_base = s_first + HF_MAXL;
  uint32_t* s_ljl = s_base + HF_MAXL;
  uint32_t* s_rings = s_ljl + HF_MAXL;                    // [DF_WARPS * 32][DF_RING_W]
  uint4* s_out = s_tma;                                   // [DF_WARPS][128] uint4 (staging, both store paths)
  for (int i = threadIdx.x; i < (1 << HF_LUT_BITS); i += blockDim.x) s_lut[i] = dt->lut[i];
  if (threadIdx.x < HF_MAXL) {
    const uint32_t l = threadIdx.x;
    s_first[l] = dt->first[l];
    s_base[l] = dt->base[l];
    s_ljl[l] = (l >= 1 && l <= max_len) ? (uint32_t)(((uint64_t)dt->first[l] + dt->count[l]) << (16 - l))
                                        : (l > max_len ? 0x10000u : 0u);
  }
  SZ3G_SYNCTHREADS();
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  // groups of 32 chunks: persistent for the 32-warp shape, one group per warp for the 8-warp one
  for (uint64_t grp = (uint64_t)blockIdx.x * DF_WARPS + wl; grp * 32 < nfull;
       grp += DF_WARPS == DF_BIG ? (uint64_t)gridDim.x * DF_WARPS : nfull) {
  const uint64_t c0 = grp * 32;
  const uint16_t* syms = reinterpret_cast<const uint16_t*>(dt + 1);
  uint4* so = s_out + wl * 128;
  const uint32_t s_ring = (uint32_t)__cvta_generic_to_shared(s_rings + threadIdx.x * DF_RING_W);
  // &s_lut[idx] = lut_sh + 4 idx; the index is the window's top 12 bits: (hi >> 20) << 2
  const uint32_t lut_sh = (uint32_t)__cvta_generic_to_shared(s_lut);
  // 2^12 and 4 as values the compiler cannot fold (max_len >= 1 for any table that decodes), so that
  // the address is IMAD.HI + IMAD on the FMA pipe (SZ3G_DF_IMAD) rather than shift / mask / add on the
  // ALU pipe, which bounds this kernel
  const uint32_t k_hi = max_len ? (1u << HF_LUT_BITS) : 0u, k4 = max_len ? 4u : 0u;
  const bool live = c0 + lane < nfull;
  const uint64_t c = live ? c0 + lane : nfull - 1;   // a dead lane decodes the last full chunk again, unstored
  const uint64_t lim = offs[nch];
  const uint64_t w0 = offs[c], nwc = offs[c + 1] - w0;
  DfLane d;
  const uint64_t a0 = w0 & ~3ull;
  const uint8_t* pl = reinterpret_cast<const uint8_t*>(payload + a0);
  const uint32_t lim4 = (uint32_t)(lim - a0 < (1ull << 28) ? lim - a0 : (1ull << 28)) * 4u;
  const uint32_t rp4_0 = 4u * (uint32_t)(w0 & 3u);
  d.rp4 = rp4_0;
  d.fp4 = 0;
  d.hi = d.lo = 0;
  d.avail = 0;
  df_topup<DF_RING / 4>(d, s_ring, pl, lim4);   // 16 words
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  d.wn = lds32(s_ring + (d.rp4 & (4 * DF_RING - 1)));
  df_refill(d, s_ring);                      // prime 64 bits
  df_refill(d, s_ring);
  bool bad = false;
  const uint32_t maxl = max_len;
  // one pair step: two codes from the window, then one refill
  auto pair = [&]() -> uint32_t {
    uint32_t o_h;
    // two codes (<= 32 bits, the window holds > 32): LUT entry (len << 16) | sym, 0 = longer than the LUT
    const uint32_t ea = lds32(df_lut_addr(d.hi, k_hi, k4, lut_sh));
    const uint32_t la = ea >> 16;
    const uint32_t hi1 = __funnelshift_l(d.lo, d.hi, la);
    const uint32_t eb = lds32(df_lut_addr(hi1, k_hi, k4, lut_sh));
    if (__any_sync(0xffffffffu, ea == 0u || eb == 0u)) {
      if (SZ3G_DF_SLOW_CALL) {
        const uint4 r = df_slow_pair(d.hi, d.lo, d.avail, lut_sh, s_ljl, s_first, s_base, syms, maxl);
        d.hi = r.x;
        d.lo = r.y;
        d.avail = r.z & 0x7fffffffu;
        bad |= (r.z >> 31) != 0u;
        o_h = r.w;
      } else {
        const uint32_t a = df_code(d, lut_sh, s_ljl, s_first, s_base, syms, maxl, bad);
        const uint32_t b = df_code(d, lut_sh, s_ljl, s_first, s_base, syms, maxl, bad);
        o_h = a | (b << 16);
      }
    } else {
      const uint32_t lb = eb >> 16;
      df_shift(d, la + lb);   // la + lb <= 24
      o_h = __byte_perm(ea, eb, 0x5410);   // (ea & 0xffff) | (eb << 16)
    }
    df_refill(d, s_ring);
    return o_h;
  };
  if (SZ3G_DF_QUARTER && DF_WARPS == DF_BIG && tma_out) {   // c5: 4.36 -> 4.10 ms; the 8-warp shape: +1%, unrolled
    // rounds of 4 quarters, each 4 pair steps (8 codes) written to the staging tile as one 16-byte unit:
    // a quarter's code (not the round's) is unrolled, which keeps the loop in the instruction cache
    for (uint32_t e = 0; e < EW_CHUNK; e += DF_ROUND) {
      uint4* tb = s_tma + wl * 128;   // row r = lane (chunk c0 + r): 64 bytes, 16-byte unit j at j ^ ((r >> 1) & 3)
#pragma unroll 1
      for (uint32_t q = 0; q < 4; q++) {
        if (q || e) df_topup<1>(d, s_ring, pl, lim4);
        uint32_t o4[4];
#pragma unroll
        for (int h = 0; h < 4; h++) o4[h] = pair();
        if (q == 0) {
          if (lane == 0) sz3g::ptx::bulk_wait_read0();   // the previous round's store has read the buffer
          SZ3G_SYNCWARP();
        }
        tb[4 * lane + (q ^ ((lane >> 1) & 3u))] = make_uint4(o4[0], o4[1], o4[2], o4[3]);
      }
      sz3g::ptx::fence_proxy_async_smem();
      SZ3G_SYNCWARP();
      if (lane == 0) {
        sz3g::ptx::tma_store_2d(&tm_out, tb, (int)e, (int)c0);
        sz3g::ptx::bulk_commit();
      }
    }
  } else
  for (uint32_t e = 0; e < EW_CHUNK; e += DF_ROUND) {
    uint32_t o[16];
#pragma unroll
    for (int h = 0; h < 16; h++) {
      if ((h % 4 == 0) && (h || e)) df_topup<1>(d, s_ring, pl, lim4);
      o[h] = pair();
    }
    if (SZ3G_DF_DIRECT) {
      if (live) {
        uint4* dst = reinterpret_cast<uint4*>(codes + c * EW_CHUNK + e);
#pragma unroll
        for (int j = 0; j < 4; j++) dst[j] = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
      }
      continue;
    }
    if (tma_out) {
      uint4* tb = s_tma + wl * 128;   // row r = lane (chunk c0 + r): 64 bytes, 16-byte unit j at j ^ ((r >> 1) & 3)
      if (lane == 0) sz3g::ptx::bulk_wait_read0();   // the previous round's store has read the buffer
      SZ3G_SYNCWARP();
#pragma unroll
      for (int j = 0; j < 4; j++)
        tb[4 * lane + (j ^ ((lane >> 1) & 3))] = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
      sz3g::ptx::fence_proxy_async_smem();
      SZ3G_SYNCWARP();
      if (lane == 0) {
        sz3g::ptx::tma_store_2d(&tm_out, tb, (int)e, (int)c0);
        sz3g::ptx::bulk_commit();
      }
      continue;
    }
    // stage: lane l's 4 uint4 at slots 4 l + j, swizzled (conflict-free both ways)
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const uint32_t i = 4 * lane + j;
      so[i ^ ((i >> 3) & 3u)] = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
    }
    SZ3G_SYNCWARP();
#pragma unroll
    for (int t = 0; t < 4; t++) {
      const uint32_t i = 32 * t + lane, r = i >> 2, j = i & 3u;
      const uint4 v = so[i ^ ((i >> 3) & 3u)];
      if (c0 + r < nfull) reinterpret_cast<uint4*>(codes + (c0 + r) * EW_CHUNK + e)[j] = v;
    }
    SZ3G_SYNCWARP();
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  if (tma_out && lane == 0) sz3g::ptx::bulk_wait0();
  const uint64_t consumed = 8ull * (d.rp4 - rp4_0) - d.avail;   // 32 bits per word taken
  if (live && (bad || consumed > nwc * 32)) atomicOr(status, (int)SZ3G_STATUS_BAD_HUFFMAN);
  }
}

size_t df_smem_bytes(int warps) { return df_smem_core_bytes(warps) + (SZ3G_DF_DIRECT ? 0ull : 16ull * 128 * warps + 1024); }




std::atomic<uint64_t> g_hf_launches{0};

int hf_check(int nl) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return SZ3G_ECUDA;
  g_hf_launches.fetch_add((uint64_t)nl, std::memory_order_relaxed);
  return SZ3G_OK;
}

// the decoder's output as a 2D map: rows = full chunks (2048 codes, 4096 bytes), box {32 codes, 32 chunks},
// 64-byte swizzle (the staging layout of k_huff_decode_full), no L2 promotion (stores)
typedef CUresult (*HfEncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
bool df_out_map(CUtensorMap* m, uint16_t* codes, uint64_t nfull) {
  static HfEncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<HfEncodeTiledFn>(p);
  });
  if (!fn || nfull == 0 || nfull >= (1ull << 31)) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)EW_CHUNK, nfull};
  const cuuint64_t strides[1] = {(cuuint64_t)EW_CHUNK * 2};
  const cuuint32_t box[2] = {32, 32};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, codes, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

int sm_count_hf() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

template <int W>
int df_launch(const uint32_t* payload, const uint64_t* offs, uint64_t nch, uint64_t nfull, const DTab* dt,
              uint32_t max_len, uint16_t* codes, int32_t* status, cudaStream_t st) {
  const size_t smem = df_smem_bytes(W);
  if (cudaFuncSetAttribute(k_huff_decode_full<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return SZ3G_ECUDA;
  if (SZ3G_DF_CARVE >= 0 &&
      cudaFuncSetAttribute(k_huff_decode_full<W>, cudaFuncAttributePreferredSharedMemoryCarveout, SZ3G_DF_CARVE) !=
          cudaSuccess)
    return SZ3G_ECUDA;
  CUtensorMap tm;
  memset(&tm, 0, sizeof(tm));
  const int tma = SZ3G_DF_TMA && !SZ3G_DF_DIRECT && df_out_map(&tm, codes, nfull) ? 1 : 0;
  const uint64_t per_cta = 32ull * W;
  uint64_t nblk = (nfull + per_cta - 1) / per_cta;
  if (W == DF_BIG) nblk = std::min<uint64_t>(nblk, (uint64_t)sm_count_hf());
  k_huff_decode_full<W><<<(unsigned)nblk, W * 32, smem, st>>>(payload, offs, nch, nfull, dt, max_len, codes, status,
                                                             tm, tma);
  return SZ3G_OK;
}

}  // namespace

// encode scratch: the scan's block sums, then (256-byte aligned) the first bit of every 64-code group
// of the full chunks (u16, 32 per chunk)
uint64_t enc_nfull(uint64_t n, uint32_t chunk) { return chunk == EW_CHUNK ? n / EW_CHUNK : 0; }
uint64_t enc_loff_offset(uint64_t n, uint32_t chunk) {
  const uint64_t nch = chunk ? (n + chunk - 1) / chunk : 0;
  return (8 * ((nch + SCAN_TILE - 1) / SCAN_TILE + 2) + 255) / 256 * 256;
}

// launches of this translation unit (folded into sz3g_launch_count)
uint64_t sz3g_huffman_launch_count_internal() { return g_hf_launches.load(); }

extern "C" {

uint64_t sz3g_huffman_scratch_bytes(uint32_t nsym, uint32_t max_len) { return cb_scratch_bytes(nsym, max_len); }
uint64_t sz3g_huffman_dtable_bytes(uint32_t nsym) { return dtable_bytes(nsym); }
uint64_t sz3g_huffman_encode_scratch_bytes(uint64_t n, uint32_t chunk) {
  return enc_loff_offset(n, chunk) + 64 * enc_nfull(n, chunk);
}

int sz3g_huffman_codebook_from_lengths(const uint8_t* lengths, uint32_t nsym, uint32_t max_len,
                                       uint32_t* codewords, void* dtable, int32_t* d_status,
                                       sz3g_stream_t stream) {
  if (!lengths || !codewords || !dtable || !d_status) return SZ3G_EINVAL;
  if (nsym < 1 || nsym > 65536) return SZ3G_ERANGE;
  if (max_len < 1 || max_len > HF_MAX_LEN_LIMIT) return SZ3G_ERANGE;
  if (reinterpret_cast<uintptr_t>(dtable) & 15) return SZ3G_EINVAL;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  k_huff_codebook<<<1, HF_THREADS, 0, st>>>(nullptr, nsym, max_len, const_cast<uint8_t*>(lengths), codewords,
                                            reinterpret_cast<DTab*>(dtable), nullptr, d_status);
  return hf_check(1);
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

int sz3g_huffman_encode(const uint16_t* codes, uint64_t n, uint32_t chunk, const uint32_t* codewords,
                        uint32_t nsym, uint64_t* chunk_offsets, uint32_t* payload, uint64_t payload_cap_words,
                        void* scratch, int32_t* d_status, sz3g_stream_t stream) {
  if ((n > 0 && !codes) || !codewords || !chunk_offsets || !d_status) return SZ3G_EINVAL;
  if (nsym < 1 || nsym > 65536) return SZ3G_ERANGE;
  if (chunk < 1 || chunk > ENC_MAX_CHUNK) return SZ3G_ERANGE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const uint64_t nch = (n + chunk - 1) / chunk;
  if (nch == 0) {
    cudaMemsetAsync(chunk_offsets, 0, 8, st);
    return cudaGetLastError() == cudaSuccess ? SZ3G_OK : SZ3G_ECUDA;
  }
  if (!payload || !scratch) return SZ3G_EINVAL;
  const int sms = sm_count_hf();
  // full 2048-code chunks take the windowed fast path, the rest (a ragged last chunk, another chunk
  // size, unaligned codes) the generic kernels
  const uint64_t nfull = (reinterpret_cast<uintptr_t>(codes) & 15) == 0 ? enc_nfull(n, chunk) : 0;
  uint16_t* loff = reinterpret_cast<uint16_t*>(static_cast<uint8_t*>(scratch) + enc_loff_offset(n, chunk));
  const uint64_t nrest = nch - nfull;
  const unsigned gf = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nfull + EW_WARPS - 1) / EW_WARPS, (uint64_t)sms));
  int nl = 0;
  if (nfull) {
    k_huff_chunk_words_full<<<gf, EW_WARPS * 32, 0, st>>>(codes, nfull, codewords, nsym, chunk_offsets, loff,
                                                          d_status);
    nl++;
  }
  if (nrest) {
    const unsigned gw = (unsigned)std::min<uint64_t>((nrest * 32 + 255) / 256, (uint64_t)sms * 16);
    k_huff_chunk_words<<<gw, 256, 0, st>>>(codes, n, chunk, codewords, nsym, chunk_offsets, nch, d_status, nfull);
    nl++;
  }
  const uint64_t nb = (nch + SCAN_TILE - 1) / SCAN_TILE;
  uint64_t* sums = reinterpret_cast<uint64_t*>(scratch);
  k_scan_sums<<<(unsigned)nb, SCAN_T, 0, st>>>(chunk_offsets, nch, sums);
  k_scan_top<<<1, SCAN_T, 0, st>>>(sums, nb);
  k_scan_apply<<<(unsigned)nb, SCAN_T, 0, st>>>(chunk_offsets, nch, sums, nb);
  if (nfull) {
    const size_t smem = ew_smem_bytes();
    // per launch: the attribute is per device, and a cached flag would skip it on a second GPU
    if (cudaFuncSetAttribute(k_huff_encode_full, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return hf_check(nl + 3);
    k_huff_encode_full<<<gf, EW_WARPS * 32, smem, st>>>(codes, nfull, codewords, nsym, chunk_offsets, loff,
                                                        payload, payload_cap_words, d_status);
    nl++;
  }
  if (nrest) {
    const unsigned ge = (unsigned)std::min<uint64_t>((nrest + ENC_WARPS - 1) / ENC_WARPS, (uint64_t)sms * 8);
    k_huff_encode<<<ge, ENC_WARPS * 32, 0, st>>>(codes, n, chunk, codewords, nsym, chunk_offsets, nch, payload,
                                                 payload_cap_words, d_status, nfull);
    nl++;
  }
  return hf_check(nl + 3);
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
  // full 2048-code chunks of a 16-byte aligned payload: the register-queue decoder; the rest (a
  // ragged last chunk, another chunk size) the ring decoder
  const uint64_t nfull = (chunk == EW_CHUNK && (reinterpret_cast<uintptr_t>(payload) & 15) == 0) ? n / EW_CHUNK : 0;
  int nl = 0;
  if (nfull) {
    // the 32-warp persistent shape once every SM gets at least one group per warp
    const bool big = (nfull + 31) / 32 >= (uint64_t)sm_count_hf() * DF_BIG;
    const DTab* dt = reinterpret_cast<const DTab*>(dtable);
    const int r = big ? df_launch<DF_BIG>(payload, chunk_offsets, nch, nfull, dt, max_len, codes, d_status, st)
                      : df_launch<DF_SMALL>(payload, chunk_offsets, nch, nfull, dt, max_len, codes, d_status, st);
    if (r != SZ3G_OK) return hf_check(nl);
    nl++;
  }
  if (nch > nfull) {
    const size_t smem = dec_smem_bytes();
    if (cudaFuncSetAttribute(k_huff_decode, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return hf_check(nl);
    const uint64_t per_cta = 32ull * DEC_WARPS;
    k_huff_decode<<<(unsigned)((nch - nfull + per_cta - 1) / per_cta), DEC_WARPS * 32, smem, st>>>(
        payload, chunk_offsets, n, chunk, reinterpret_cast<const DTab*>(dtable), max_len, codes, nch, d_status, nfull);
    nl++;
  }
  return hf_check(nl);
}

}  // extern "C"
