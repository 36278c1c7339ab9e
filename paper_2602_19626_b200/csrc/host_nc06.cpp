// NC06 hybrid binary format, host side ("Hybrid Binary
// Compression (NC06)"; readings D33-D34 in DESIGN.md).
//
//   segment():  rules (1)-(4) of P:516-520, applied once each in order, adjacent same-kind
//               regions merged after every rule (D33)
//   blob codec: every binary region concatenated, LZMA (.xz, preset 6, CRC64) if >= 4 KB
//               else DEFLATE (zlib stream, level 9), raw unless strictly smaller;
//               liblzma is dlopen'ed (the image ships liblzma.so.5 without its headers)
//   container:  "NC06" | ver u8 = 1 | flags u8 | tau u16 | n u16 | n x {kind u8, len u32}
//               | method u8 | blob_len u32 | blob | NC05 text section from its chunk count on
// The text regions, concatenated, go through the unchanged NC05 text path (api.cpp).
#include <dlfcn.h>
#include <zlib.h>

#include <cstring>
#include <mutex>

#include "nc06.hpp"

namespace nc {

static inline bool text_byte(uint8_t b) { return (b >= 32 && b <= 126) || b == 9 || b == 10 || b == 13; }

static void merge(std::vector<Region> &r) {
  std::vector<Region> o;
  for (const Region &x : r) {
    if (x.len == 0) continue;
    if (!o.empty() && o.back().kind == x.kind) o.back().len += x.len;
    else o.push_back(x);
  }
  r.swap(o);
}

std::vector<Region> segment(const uint8_t *in, size_t n) {
  std::vector<Region> r;
  for (size_t i = 0; i < n;) {   // rule 1: runs of the byte class
    const uint8_t k = text_byte(in[i]) ? kText : kBinary;
    size_t j = i + 1;
    while (j < n && (text_byte(in[j]) ? kText : kBinary) == k) ++j;
    r.push_back(Region{k, j - i});
    i = j;
  }
  for (Region &x : r)   // rule 2: text runs < 64 bytes demoted
    if (x.kind == kText && x.len < 64) x.kind = kBinary;
  merge(r);
  {                     // rule 3: binary gaps <= 8 bytes between text runs bridged
    std::vector<uint8_t> k(r.size());
    for (size_t i = 0; i < r.size(); ++i)
      k[i] = (r[i].kind == kBinary && r[i].len <= 8 && i > 0 && i + 1 < r.size() && r[i - 1].kind == kText &&
              r[i + 1].kind == kText) ? kText : r[i].kind;
    for (size_t i = 0; i < r.size(); ++i) r[i].kind = k[i];
    merge(r);
  }
  {                     // rule 4: binary chunks < 64 bytes adjacent to text absorbed
    std::vector<uint8_t> k(r.size());
    for (size_t i = 0; i < r.size(); ++i)
      k[i] = (r[i].kind == kBinary && r[i].len < 64 &&
              ((i > 0 && r[i - 1].kind == kText) || (i + 1 < r.size() && r[i + 1].kind == kText))) ? kText
                                                                                                   : r[i].kind;
    for (size_t i = 0; i < r.size(); ++i) r[i].kind = k[i];
    merge(r);
  }
  return r;
}

// ------------------------------------------------------------------ liblzma ---
namespace {
typedef int (*lzma_easy_buffer_encode_t)(uint32_t, int, const void *, const uint8_t *, size_t, uint8_t *, size_t *,
                                         size_t);
typedef int (*lzma_stream_buffer_decode_t)(uint64_t *, uint32_t, const void *, const uint8_t *, size_t *, size_t,
                                           uint8_t *, size_t *, size_t);
typedef size_t (*lzma_stream_buffer_bound_t)(size_t);
struct Lzma {
  lzma_easy_buffer_encode_t enc = nullptr;
  lzma_stream_buffer_decode_t dec = nullptr;
  lzma_stream_buffer_bound_t bound = nullptr;
};
const Lzma &lzma() {
  static Lzma L;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = dlopen("liblzma.so.5", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    L.enc = (lzma_easy_buffer_encode_t)dlsym(h, "lzma_easy_buffer_encode");
    L.dec = (lzma_stream_buffer_decode_t)dlsym(h, "lzma_stream_buffer_decode");
    L.bound = (lzma_stream_buffer_bound_t)dlsym(h, "lzma_stream_buffer_bound");
  });
  if (!L.enc || !L.dec || !L.bound) fail(NC_ERR_BACKEND, "liblzma.so.5 not available");
  return L;
}
constexpr int kLzmaCheckCrc64 = 4, kLzmaOk = 0, kLzmaStreamEnd = 1;
}  // namespace

uint8_t blob_encode(const uint8_t *in, size_t n, std::vector<uint8_t> &out) {
  out.clear();
  if (n == 0) return kRaw;
  std::vector<uint8_t> c;
  uint8_t m;
  if (n >= 4096) {
    const Lzma &L = lzma();
    c.resize(L.bound(n));
    size_t pos = 0;
    if (L.enc(6, kLzmaCheckCrc64, nullptr, in, n, c.data(), &pos, c.size()) != kLzmaOk)
      fail(NC_ERR_BACKEND, "lzma encode failed");
    c.resize(pos);
    m = kLzma;
  } else {
    uLongf len = compressBound((uLong)n);
    c.resize(len);
    if (compress2(c.data(), &len, in, (uLong)n, 9) != Z_OK) fail(NC_ERR_BACKEND, "deflate failed");
    c.resize(len);
    m = kDeflate;
  }
  if (c.size() < n) {
    out.swap(c);
    return m;
  }
  out.assign(in, in + n);
  return kRaw;
}

void blob_decode(uint8_t method, const uint8_t *in, size_t n, size_t expect, std::vector<uint8_t> &out) {
  out.assign(expect, 0);
  if (method == kRaw) {
    if (n != expect) fail(NC_ERR_INTEGRITY, "raw binary section length mismatch");
    if (n) std::memcpy(out.data(), in, n);
  } else if (method == kDeflate) {
    uLongf len = (uLongf)expect;
    const int r = uncompress(out.data(), &len, in, (uLong)n);
    if (r != Z_OK || len != expect) fail(NC_ERR_INTEGRITY, "DEFLATE binary section does not decode to its length");
  } else if (method == kLzma) {
    const Lzma &L = lzma();
    uint64_t memlimit = UINT64_MAX;
    size_t ip = 0, op = 0;
    const int r = L.dec(&memlimit, 0, nullptr, in, &ip, n, out.data(), &op, out.size());
    if (r != kLzmaOk && r != kLzmaStreamEnd) fail(NC_ERR_INTEGRITY, "LZMA binary section does not decode");
    if (op != expect || ip != n) fail(NC_ERR_INTEGRITY, "LZMA binary section length mismatch");
  } else {
    fail(NC_ERR_FORMAT, "unknown binary method");
  }
}

static void put16(std::vector<uint8_t> &o, uint16_t v) { o.push_back(v & 255); o.push_back(v >> 8); }
static void put32(std::vector<uint8_t> &o, uint32_t v) {
  for (int i = 0; i < 4; ++i) o.push_back((v >> (8 * i)) & 255);
}
static uint32_t get32(const uint8_t *p) { return p[0] | (p[1] << 8) | (p[2] << 16) | ((uint32_t)p[3] << 24); }

void write_nc06(uint8_t flags, uint16_t tau_milli, const std::vector<Region> &regs, uint8_t method,
                const std::vector<uint8_t> &payload, const uint8_t *nc05, size_t nc05_n, std::vector<uint8_t> &out) {
  if (regs.size() > 0xFFFF) fail(NC_ERR_INVALID, "too many NC06 entries");
  if (payload.size() > 0xFFFFFFFFull) fail(NC_ERR_INVALID, "binary section exceeds 4 GB");
  if (nc05_n < 9 || std::memcmp(nc05, "NC05", 4) != 0) fail(NC_ERR_FORMAT, "text section is not NC05");
  out.clear();
  out.insert(out.end(), {'N', 'C', '0', '6', 1, flags});
  put16(out, tau_milli);
  put16(out, (uint16_t)regs.size());
  for (const Region &r : regs) {
    if (r.len > 0xFFFFFFFFull) fail(NC_ERR_INVALID, "NC06 region exceeds 4 GB");
    out.push_back(r.kind);
    put32(out, (uint32_t)r.len);
  }
  out.push_back(method);
  put32(out, (uint32_t)payload.size());
  out.insert(out.end(), payload.begin(), payload.end());
  out.insert(out.end(), nc05 + 7, nc05 + nc05_n);   // chunk count, chunk table, streams
}

Nc06View read_nc06(const uint8_t *in, size_t n) {
  Nc06View v;
  if (n < 10) fail(NC_ERR_TRUNCATED, "NC06 header truncated");
  if (std::memcmp(in, "NC06", 4) != 0) fail(NC_ERR_FORMAT, "bad magic");
  if (in[4] != 1) fail(NC_ERR_FORMAT, "unsupported NC06 version");
  v.flags = in[5];
  v.tau_milli = (uint16_t)(in[6] | (in[7] << 8));
  const uint32_t ne = in[8] | (in[9] << 8);
  if (v.flags & ~0x07u) fail(NC_ERR_FORMAT, "reserved flag bits set");
  size_t off = 10;
  if (n < off + 5ull * ne + 5) fail(NC_ERR_TRUNCATED, "NC06 entry table truncated");
  for (uint32_t i = 0; i < ne; ++i) {
    const uint8_t k = in[off];
    if (k != kText && k != kBinary) fail(NC_ERR_FORMAT, "bad NC06 entry kind");
    v.regs.push_back(Region{k, get32(in + off + 1)});
    (k == kText ? v.text_len : v.bin_len) += get32(in + off + 1);
    off += 5;
  }
  v.method = in[off];
  const uint32_t bl = get32(in + off + 1);
  off += 5;
  if (off + bl + 2 > n) fail(NC_ERR_TRUNCATED, "NC06 binary section truncated");
  v.payload_off = off;
  v.payload_len = bl;
  off += bl;
  v.text_off = off;   // chunk count u16 + table + streams (validated by read_nc05 on the rebuilt NC05)
  return v;
}

}  // namespace nc
