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
#include <cmath>
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
  put<uint64_t>(p, h->dim0_offset);   // bytes 80..87 (zero in streams written before this field existed)
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
  h->dim0_offset = get<uint64_t>(p);
}

const sz3g_section* find(const sz3g_section* s, uint32_t n, uint32_t tag, int* count) {
  const sz3g_section* f = nullptr;
  *count = 0;
  for (uint32_t i = 0; i < n; i++)
    if (s[i].tag == tag) {
      f = &s[i];
      (*count)++;
    }
  return f;
}

uint64_t cdiv(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// canonical codebook record list: u32 m, m x (u16 symbol, u8 length), symbols increasing
bool book_ok(const sz3g_section* b, uint32_t nsym, uint32_t max_len) {
  if (b->bytes < 4) return false;
  const uint8_t* p = static_cast<const uint8_t*>(b->data);
  uint32_t m;
  std::memcpy(&m, p, 4);
  if (m > nsym || b->bytes != 4 + 3ull * m) return false;
  int64_t prev = -1;
  for (uint32_t r = 0; r < m; r++) {
    uint16_t sym;
    std::memcpy(&sym, p + 4 + 3ull * r, 2);
    const uint8_t len = p[4 + 3ull * r + 2];
    if (sym >= nsym || (int64_t)sym <= prev || len < 1 || len > max_len) return false;
    prev = sym;
  }
  return true;
}

// chunk offsets of a Huffman stream of n symbols against its payload section
bool offsets_ok(const sz3g_section* o, const sz3g_section* d, uint64_t n, uint32_t chunk, uint32_t max_len) {
  const uint64_t nch = cdiv(n, chunk);
  if (o->bytes != 8 * (nch + 1) || d->bytes % 4) return false;
  const uint8_t* p = static_cast<const uint8_t*>(o->data);
  const uint64_t max_words = cdiv((uint64_t)chunk * max_len, 32);
  uint64_t prev;
  std::memcpy(&prev, p, 8);
  if (prev != 0) return false;
  for (uint64_t c = 1; c <= nch; c++) {
    uint64_t v;
    std::memcpy(&v, p + 8 * c, 8);
    if (v < prev || v - prev > max_words) return false;
    prev = v;
  }
  return prev == d->bytes / 4;
}

}  // namespace

extern "C" {

int sz3g_stream_validate(const sz3g_stream_header* h, const sz3g_section* s, uint32_t n, uint32_t* bad_tag) {
  if (!h || (n && !s)) return SZ3G_EINVAL;
  uint32_t dummy;
  uint32_t* bad = bad_tag ? bad_tag : &dummy;
  *bad = 0;
  if ((h->dtype != SZ3G_F32 && h->dtype != SZ3G_F64) || h->ndim < 1 || h->ndim > 3 || h->block_size != 6 ||
      h->radius < 1 || h->radius > 32768 || h->max_len < 1 || h->max_len > 16 || h->chunk < 1 ||
      !std::isfinite(h->eb_abs) || !(h->eb_abs > 0))
    return SZ3G_ECORRUPT;
  uint64_t N = 1;
  for (int d = 0; d < 3; d++) {
    if (h->dims[d] == 0 || (d < 3 - (int)h->ndim && h->dims[d] != 1)) return SZ3G_ECORRUPT;
    if (h->dims[d] > (UINT64_MAX / N)) return SZ3G_ECORRUPT;
    N *= h->dims[d];
  }
  const bool lr = (h->flags & SZ3G_STREAM_LR) != 0, ip = (h->flags & SZ3G_STREAM_INTERP) != 0;
  if ((lr && ip) || (h->flags & ~(SZ3G_STREAM_LR | SZ3G_STREAM_INTERP))) return SZ3G_ECORRUPT;
  // SZ3-Interp has no coefficients: nblocks 0 and no coefficient sections
  const uint64_t nb = ip ? 0 : cdiv(h->dims[0], 6) * cdiv(h->dims[1], 6) * cdiv(h->dims[2], 6);
  if (h->nblocks != nb) return SZ3G_ECORRUPT;
  const sz3g_section* sec[SZ3G_SEC_LR_FLAGS + 1] = {};
  for (uint32_t tag = SZ3G_SEC_CODE_BOOK; tag <= SZ3G_SEC_LR_FLAGS; tag++) {
    int cnt;
    sec[tag] = find(s, n, tag, &cnt);
    const bool coef = tag >= SZ3G_SEC_COEF_BOOK && tag <= SZ3G_SEC_COEF_ESC;
    const bool want = tag == SZ3G_SEC_LR_FLAGS ? lr : !(coef && ip);
    if ((want && cnt != 1) || (!want && cnt != 0)) {
      *bad = tag;
      return SZ3G_ECORRUPT;
    }
  }
  const uint64_t vs = h->dtype == SZ3G_F32 ? 4 : 8;
  if (sec[SZ3G_SEC_OUT_IDX]->bytes != 8 * h->n_outliers) { *bad = SZ3G_SEC_OUT_IDX; return SZ3G_ECORRUPT; }
  if (sec[SZ3G_SEC_OUT_VAL]->bytes != vs * h->n_outliers) { *bad = SZ3G_SEC_OUT_VAL; return SZ3G_ECORRUPT; }
  {
    const uint64_t plane = h->dims[1] * h->dims[2];
    const uint64_t lo = h->dim0_offset * plane, hi = lo + N;
    if (h->dim0_offset > UINT64_MAX / plane || hi < lo) return SZ3G_ECORRUPT;
    const uint8_t* p = static_cast<const uint8_t*>(sec[SZ3G_SEC_OUT_IDX]->data);
    for (uint64_t e = 0; e < h->n_outliers; e++) {
      uint64_t v;
      std::memcpy(&v, p + 8 * e, 8);
      if (v < lo || v >= hi) { *bad = SZ3G_SEC_OUT_IDX; return SZ3G_ECORRUPT; }
    }
  }
  if (!book_ok(sec[SZ3G_SEC_CODE_BOOK], 2 * h->radius, h->max_len)) { *bad = SZ3G_SEC_CODE_BOOK; return SZ3G_ECORRUPT; }
  if (!ip && !book_ok(sec[SZ3G_SEC_COEF_BOOK], 65536, h->max_len)) { *bad = SZ3G_SEC_COEF_BOOK; return SZ3G_ECORRUPT; }
  if (!offsets_ok(sec[SZ3G_SEC_CODE_OFFS], sec[SZ3G_SEC_CODE_DATA], N, h->chunk, h->max_len)) {
    *bad = SZ3G_SEC_CODE_OFFS;
    return SZ3G_ECORRUPT;
  }
  if (!ip && !offsets_ok(sec[SZ3G_SEC_COEF_OFFS], sec[SZ3G_SEC_COEF_DATA], 4 * nb, h->chunk, h->max_len)) {
    *bad = SZ3G_SEC_COEF_OFFS;
    return SZ3G_ECORRUPT;
  }
  if (!ip && sec[SZ3G_SEC_COEF_ESC]->bytes % 8) { *bad = SZ3G_SEC_COEF_ESC; return SZ3G_ECORRUPT; }
  if (lr && sec[SZ3G_SEC_LR_FLAGS]->bytes != cdiv(nb, 8)) { *bad = SZ3G_SEC_LR_FLAGS; return SZ3G_ECORRUPT; }
  return SZ3G_OK;
}


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
