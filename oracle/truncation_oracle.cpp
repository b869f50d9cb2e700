// =====================================================================================
//  oracle/truncation_oracle.cpp -- TEST INFRASTRUCTURE ONLY (not part of the product path).
//
//  SZ3-Truncation: "Given the target bytes k as input parameter, it keeps k
//  most-significant bytes of each floating-point data while discarding the rest of the bytes."
//  Readings (G24, DEFINITION.md T1-T2): the stream holds, element after element, the k
//  most-significant bytes of the IEEE-754 representation, most significant first ("big-endian-
//  ordered representation"); decompression zero-fills the discarded bytes.
//  Plain byte loops; no code is shared with paper_2111_02925_b200/.
// =====================================================================================
#include <cstdint>
#include <cstring>

extern "C" {

// T1: out[i*k + j] = byte (s-1-j) of element i (byte 0 = least significant)
int orc_trunc_compress(int dtype, uint64_t n, const void* x, uint32_t k, uint8_t* out) {
  const uint32_t s = dtype == 0 ? 4u : 8u;
  if (dtype != 0 && dtype != 1) return -2;
  if (k < 1 || k > s) return -3;
  const uint8_t* in = static_cast<const uint8_t*>(x);
  for (uint64_t i = 0; i < n; i++) {
    uint64_t bits = 0;
    std::memcpy(&bits, in + i * s, s);   // host is little-endian: bits holds the value's pattern
    for (uint32_t j = 0; j < k; j++) out[i * k + j] = (uint8_t)(bits >> (8 * (s - 1 - j)));
  }
  return 0;
}

// T2: element i = its k stored bytes as the most significant bytes, the rest zero
int orc_trunc_decompress(int dtype, uint64_t n, const uint8_t* in, uint32_t k, void* x) {
  const uint32_t s = dtype == 0 ? 4u : 8u;
  if (dtype != 0 && dtype != 1) return -2;
  if (k < 1 || k > s) return -3;
  uint8_t* out = static_cast<uint8_t*>(x);
  for (uint64_t i = 0; i < n; i++) {
    uint64_t bits = 0;
    for (uint32_t j = 0; j < k; j++) bits |= (uint64_t)in[i * k + j] << (8 * (s - 1 - j));
    std::memcpy(out + i * s, &bits, s);
  }
  return 0;
}

}  // extern "C"

// =====================================================================================
//  Coefficient-code delta coding (NEXT-3; DEFINITION.md C1-C2, reading G25).  The G1 coefficient codes
//  are independent per block; their storage is reduced by integer differencing along the block order
//  (per channel), a zigzag map to unsigned values, and an escape for values >= 65535, so that the
//  symbols fit the Huffman coder of the quantisation codes ("Coefficient Compression" is an
//  empty heading; S:225-233 codes coefficient deltas).  Plain loops.
// =====================================================================================
extern "C" {

// C1: coef[nb][4] (int32) -> sym[4][nb] (uint16, channel-major), escapes in position order.
// Returns the number of escapes (written up to esc_cap).
uint64_t orc_coef_delta_encode(const int32_t* coef, uint64_t nb, uint16_t* sym, uint64_t* esc, uint64_t esc_cap) {
  uint64_t ne = 0;
  for (int ch = 0; ch < 4; ch++) {
    int64_t prev = 0;
    for (uint64_t b = 0; b < nb; b++) {
      const int64_t v = coef[4 * b + ch];
      const int64_t d = v - prev;
      prev = v;
      const uint64_t z = d >= 0 ? (uint64_t)d * 2 : (uint64_t)(-(d + 1)) * 2 + 1;   // zigzag
      if (z >= 65535) {
        sym[ch * nb + b] = 65535;
        if (ne < esc_cap) esc[ne] = z;
        ne++;
      } else {
        sym[ch * nb + b] = (uint16_t)z;
      }
    }
  }
  return ne;
}

// C2: the inverse.  Returns 0, or -1 if the escapes run out.
int orc_coef_delta_decode(const uint16_t* sym, uint64_t nb, const uint64_t* esc, uint64_t nesc, int32_t* coef) {
  uint64_t k = 0;
  for (int ch = 0; ch < 4; ch++) {
    int64_t acc = 0;
    for (uint64_t b = 0; b < nb; b++) {
      uint64_t z = sym[ch * nb + b];
      if (z == 65535) {
        if (k >= nesc) return -1;
        z = esc[k++];
      }
      const int64_t d = (z & 1) ? -(int64_t)(z >> 1) - 1 : (int64_t)(z >> 1);
      acc += d;
      coef[4 * b + ch] = (int32_t)acc;
    }
  }
  return 0;
}

}  // extern "C"
