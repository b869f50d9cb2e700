// =====================================================================================
//  oracle/huffman_oracle.cpp -- TEST INFRASTRUCTURE ONLY (not part of the product path).
//
//  Plain, slow, single-threaded CPU definition of the encoder stage that follows the
//  quantiser in SZ3's pipeline:
//    * P:156  "The data size will be significantly reduced after conducting Huffman encoding on
//             the quantization codes."
//    * P:418  Huffman encoder: "constructs a Huffman tree based on the frequency of input data
//             using a greedy algorithm, generates codebook according to the tree, and then
//             compress the data using the codebook."
//    * P:413-416, App. A P:948-957  encode / decode / save / load of the encoder module.
//  Readings (G19-G23, oracle/DEFINITION.md H1-H5):
//    H1 symbols are the quantisation codes [0, 2R) with their histogram counts;
//    H2 code lengths = an OPTIMAL prefix code under a maximum length Lmax (minimum sum
//       count*len subject to len <= Lmax), computed by package-merge (Larmore & Hirschberg) with
//       the tie rule below; one active symbol gets length 1;
//    H3 canonical codewords: symbols ordered by (length, symbol), consecutive codes per length;
//    H4 encoding: chunks of C codes, each chunk's codewords concatenated MSB-first and padded to a
//       32-bit word; bit b of a chunk lives in word b/32 at bit 31 - b%32; chunk offsets (in
//       words) are the exclusive prefix sum of the chunk sizes;
//    H5 decoding is the inverse.
//  Package-merge as written here (n >= 2 active symbols, weights w):
//    leaves = active symbols sorted by (count asc, symbol asc);
//    list[Lmax] = leaves;  for l = Lmax-1 .. 1:
//        pk[j]  = list[l+1][2j].w + list[l+1][2j+1].w     (j < |list[l+1]| / 2)
//        list[l] = merge(leaves, pk)  -- ascending weight, a LEAF before a package of equal weight
//    m = 2n - 2;  for l = 1 .. Lmax:  c[l] = #leaves among the first m items of list[l];
//                                    m = 2 * (m - c[l])           (packages taken at level l)
//    len(i-th sorted leaf) = #{ l : i < c[l] }.
//  No code, header, table or constant is shared with paper_2111_02925_b200/.
// =====================================================================================
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

namespace {

struct Item {
  uint64_t w;
  bool leaf;
};

}  // namespace

extern "C" {

// H2: code lengths (lens[nsym], 0 for absent symbols).  Returns 0, or -1 if no symbol is
// active, -2 if 2^max_len < number of active symbols (no prefix code fits).
int orc_huffman_lengths(const int64_t* hist, uint32_t nsym, uint32_t max_len, uint8_t* lens) {
  std::memset(lens, 0, nsym);
  std::vector<uint32_t> sym;
  for (uint32_t s = 0; s < nsym; s++)
    if (hist[s] > 0) sym.push_back(s);
  const uint64_t n = sym.size();
  if (n == 0) return -1;
  if (n == 1) {
    lens[sym[0]] = 1;
    return 0;
  }
  if (max_len < 64 && (1ull << max_len) < n) return -2;
  std::stable_sort(sym.begin(), sym.end(), [&](uint32_t a, uint32_t b) {
    return (uint64_t)hist[a] < (uint64_t)hist[b];   // ties keep symbol order (ascending)
  });
  std::vector<uint64_t> leafw(n);
  for (uint64_t i = 0; i < n; i++) leafw[i] = (uint64_t)hist[sym[i]];
  // lists[l] for l = 1 .. max_len (index l)
  std::vector<std::vector<Item>> lists(max_len + 1);
  for (uint64_t i = 0; i < n; i++) lists[max_len].push_back({leafw[i], true});
  for (uint32_t l = max_len - 1; l >= 1; l--) {
    const std::vector<Item>& below = lists[l + 1];
    std::vector<uint64_t> pk;
    for (size_t j = 0; j + 1 < below.size(); j += 2) pk.push_back(below[j].w + below[j + 1].w);
    std::vector<Item>& cur = lists[l];
    size_t a = 0, b = 0;
    while (a < n || b < pk.size()) {
      if (b == pk.size() || (a < n && leafw[a] <= pk[b])) cur.push_back({leafw[a++], true});
      else cur.push_back({pk[b++], false});
    }
  }
  std::vector<uint64_t> c(max_len + 1, 0);
  uint64_t m = 2 * n - 2;
  for (uint32_t l = 1; l <= max_len; l++) {
    if (m > lists[l].size()) return -3;   // cannot happen when 2^max_len >= n
    uint64_t leaves = 0;
    for (uint64_t t = 0; t < m; t++) leaves += lists[l][t].leaf ? 1 : 0;
    c[l] = leaves;
    m = 2 * (m - leaves);
  }
  for (uint64_t i = 0; i < n; i++) {
    uint32_t len = 0;
    for (uint32_t l = 1; l <= max_len; l++) len += (i < c[l]) ? 1 : 0;
    lens[sym[i]] = (uint8_t)len;
  }
  return 0;
}

// H3: canonical codewords from the lengths (right-aligned in uint32; 0 for absent symbols).
void orc_huffman_canonical(const uint8_t* lens, uint32_t nsym, uint32_t* codes) {
  std::vector<uint32_t> order;
  for (uint32_t s = 0; s < nsym; s++) {
    codes[s] = 0;
    if (lens[s]) order.push_back(s);
  }
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return lens[a] < lens[b]; });
  uint64_t code = 0;
  uint32_t prev = 0;
  for (size_t t = 0; t < order.size(); t++) {
    const uint32_t L = lens[order[t]];
    if (t == 0) {
      code = 0;
    } else {
      code = (code + 1) << (L - prev);
    }
    codes[order[t]] = (uint32_t)code;
    prev = L;
  }
}

// H4: number of 32-bit words of each chunk and the exclusive prefix offsets (offs[nchunks + 1]).
void orc_huffman_chunk_offsets(const uint16_t* q, uint64_t n, uint32_t chunk, const uint8_t* lens,
                               uint64_t* offs) {
  const uint64_t nch = (n + chunk - 1) / chunk;
  uint64_t acc = 0;
  for (uint64_t c = 0; c < nch; c++) {
    offs[c] = acc;
    uint64_t bits = 0;
    for (uint64_t e = c * chunk; e < std::min<uint64_t>(n, (c + 1) * chunk); e++) bits += lens[q[e]];
    acc += (bits + 31) / 32;
  }
  offs[nch] = acc;
}

// H4: encode.  words[offs[nchunks]] must be zeroed by the caller.  Returns -1 if a code has no
// codeword (length 0).
int orc_huffman_encode(const uint16_t* q, uint64_t n, uint32_t chunk, const uint8_t* lens, const uint32_t* codes,
                       const uint64_t* offs, uint32_t* words) {
  const uint64_t nch = (n + chunk - 1) / chunk;
  for (uint64_t c = 0; c < nch; c++) {
    uint64_t bit = 0;   // bit position inside the chunk
    for (uint64_t e = c * chunk; e < std::min<uint64_t>(n, (c + 1) * chunk); e++) {
      const uint32_t L = lens[q[e]];
      if (L == 0) return -1;
      for (int t = (int)L - 1; t >= 0; t--) {   // MSB of the codeword first
        const uint32_t b = (codes[q[e]] >> t) & 1u;
        if (b) words[offs[c] + bit / 32] |= 1u << (31 - bit % 32);
        bit++;
      }
    }
  }
  return 0;
}

// H5: decode by walking the canonical code bit by bit (no tables).  Returns -1 on a bit string
// that matches no codeword, -2 if a chunk runs past its words.
int orc_huffman_decode(const uint32_t* words, const uint64_t* offs, uint64_t n, uint32_t chunk, const uint8_t* lens,
                       const uint32_t* codes, uint32_t nsym, uint16_t* q) {
  // (length, codeword) -> symbol, as a sorted list searched per prefix length
  std::vector<std::pair<uint64_t, uint32_t>> keyed;   // key = (len << 32) | code
  for (uint32_t s = 0; s < nsym; s++)
    if (lens[s]) keyed.push_back({((uint64_t)lens[s] << 32) | codes[s], s});
  std::sort(keyed.begin(), keyed.end());
  const uint64_t nch = (n + chunk - 1) / chunk;
  for (uint64_t c = 0; c < nch; c++) {
    uint64_t bit = 0;
    const uint64_t nbits = (offs[c + 1] - offs[c]) * 32;
    for (uint64_t e = c * chunk; e < std::min<uint64_t>(n, (c + 1) * chunk); e++) {
      uint64_t code = 0;
      bool found = false;
      for (uint32_t L = 1; L <= 32 && !found; L++) {
        if (bit >= nbits) return -2;
        code = (code << 1) | ((words[offs[c] + bit / 32] >> (31 - bit % 32)) & 1u);
        bit++;
        const uint64_t key = ((uint64_t)L << 32) | code;
        auto it = std::lower_bound(keyed.begin(), keyed.end(), std::make_pair(key, 0u));
        if (it != keyed.end() && it->first == key) {
          q[e] = (uint16_t)it->second;
          found = true;
        }
      }
      if (!found) return -1;
    }
  }
  return 0;
}

}  // extern "C"
