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
