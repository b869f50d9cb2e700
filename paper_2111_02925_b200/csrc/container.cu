// libsz3g -- self-describing compressed stream (NEXT-3; "Stream format (all integers
// little-endian): magic ..., version u16, dtype u8, ... then ... section bundle; each inner section:
// tag u8, length u64, payload").  Host code only: the sections are the device results copied to the
// host (payloads of the Huffman streams, chunk offsets, coefficient stream, outliers, codebooks); the
// container adds a fixed header and a 64-bit FNV-1a checksum per section so that a damaged stream is
// rejected with the failing section named ("corruption errors with section name").
//
// Layout (little-endian):
//   "SZ3G" | version u16 = 1 | header (sz3g_stream_header, fixed 96-byte encoding below) |
//   nsec u32 | nsec x { tag u8 | length u64 | fnv1a64 u64 | payload[length] }
#include <cstdint>
#include <cstring>

#include "../../include/sz3g.h"

namespace {

constexpr uint16_t kVersion = 1;
constexpr size_t kHeaderBytes = 96;

uint64_t fnv1a(const uint8_t* p, uint64_t n) {
  uint64_t h = 1469598103934665603ull;
  for (uint64_t i = 0; i < n; i++) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}

template <typename V>
void put(uint8_t*& o, V v) {
  std::memcpy(o, &v, sizeof(V));   // the host is little-endian (x86-64 / aarch64)
  o += sizeof(V);
}
template <typename V>
V get(const uint8_t*& i) {
  V v;
  std::memcpy(&v, i, sizeof(V));
  i += sizeof(V);
  return v;
}

void encode_header(const sz3g_stream_header* h, uint8_t* o) {
  uint8_t* p = o;
  put<uint8_t>(p, (uint8_t)h->dtype);
  put<uint8_t>(p, (uint8_t)h->ndim);
  put<uint8_t>(p, (uint8_t)h->eb_mode);
  put<uint8_t>(p, 0);
  put<uint32_t>(p, h->block_size);
  for (int d = 0; d < 3; d++) put<uint64_t>(p, h->dims[d]);
  put<double>(p, h->eb);
  put<double>(p, h->eb_abs);
  put<uint32_t>(p, h->radius);
  put<uint32_t>(p, h->chunk);
  put<uint32_t>(p, h->max_len);
  put<uint32_t>(p, h->flags);
  put<uint64_t>(p, h->n_outliers);
  put<uint64_t>(p, h->nblocks);
  while (p < o + kHeaderBytes) put<uint8_t>(p, 0);
}

void decode_header(const uint8_t* i, sz3g_stream_header* h) {
  const uint8_t* p = i;
  h->dtype = (sz3g_dtype)get<uint8_t>(p);
  h->ndim = get<uint8_t>(p);
  h->eb_mode = (sz3g_eb_mode)get<uint8_t>(p);
  get<uint8_t>(p);
  h->block_size = get<uint32_t>(p);
  for (int d = 0; d < 3; d++) h->dims[d] = get<uint64_t>(p);
  h->eb = get<double>(p);
  h->eb_abs = get<double>(p);
  h->radius = get<uint32_t>(p);
  h->chunk = get<uint32_t>(p);
  h->max_len = get<uint32_t>(p);
  h->flags = get<uint32_t>(p);
  h->n_outliers = get<uint64_t>(p);
  h->nblocks = get<uint64_t>(p);
}

}  // namespace

extern "C" {

uint64_t sz3g_stream_size(const sz3g_section* sections, uint32_t nsec) {
  uint64_t n = 4 + 2 + kHeaderBytes + 4;
  for (uint32_t s = 0; s < nsec; s++) n += 1 + 8 + 8 + sections[s].bytes;
  return n;
}

int sz3g_stream_write(const sz3g_stream_header* hdr, const sz3g_section* sections, uint32_t nsec, void* out,
                      uint64_t cap, uint64_t* written) {
  if (!hdr || (nsec && !sections) || !out || !written) return SZ3G_EINVAL;
  const uint64_t need = sz3g_stream_size(sections, nsec);
  if (need > cap) return SZ3G_ERANGE;
  uint8_t* o = static_cast<uint8_t*>(out);
  std::memcpy(o, "SZ3G", 4);
  o += 4;
  put<uint16_t>(o, kVersion);
  encode_header(hdr, o);
  o += kHeaderBytes;
  put<uint32_t>(o, nsec);
  for (uint32_t s = 0; s < nsec; s++) {
    const sz3g_section& sc = sections[s];
    if (sc.bytes && !sc.data) return SZ3G_EINVAL;
    put<uint8_t>(o, (uint8_t)sc.tag);
    put<uint64_t>(o, sc.bytes);
    put<uint64_t>(o, fnv1a(static_cast<const uint8_t*>(sc.data), sc.bytes));
    if (sc.bytes) std::memcpy(o, sc.data, sc.bytes);
    o += sc.bytes;
  }
  *written = need;
  return SZ3G_OK;
}

int sz3g_stream_read(const void* in, uint64_t len, sz3g_stream_header* hdr, sz3g_section* sections,
                     uint32_t sec_cap, uint32_t* nsec, uint32_t* bad_tag) {
  if (!in || !hdr || !nsec) return SZ3G_EINVAL;
  if (bad_tag) *bad_tag = 0;
  const uint8_t* i = static_cast<const uint8_t*>(in);
  const uint8_t* end = i + len;
  if (len < 4 + 2 + kHeaderBytes + 4 || std::memcmp(i, "SZ3G", 4) != 0) return SZ3G_ECORRUPT;
  i += 4;
  if (get<uint16_t>(i) != kVersion) return SZ3G_ECORRUPT;
  decode_header(i, hdr);
  i += kHeaderBytes;
  const uint32_t n = get<uint32_t>(i);
  if (n > sec_cap || (n && !sections)) return SZ3G_ERANGE;
  for (uint32_t s = 0; s < n; s++) {
    if ((uint64_t)(end - i) < 1 + 8 + 8) return SZ3G_ECORRUPT;
    const uint32_t tag = get<uint8_t>(i);
    const uint64_t bytes = get<uint64_t>(i);
    const uint64_t sum = get<uint64_t>(i);
    if ((uint64_t)(end - i) < bytes || fnv1a(i, bytes) != sum) {
      if (bad_tag) *bad_tag = tag;
      return SZ3G_ECORRUPT;
    }
    sections[s].tag = tag;
    sections[s].data = i;
    sections[s].bytes = bytes;
    i += bytes;
  }
  *nsec = n;
  return i == end ? SZ3G_OK : SZ3G_ECORRUPT;
}

}  // extern "C"
