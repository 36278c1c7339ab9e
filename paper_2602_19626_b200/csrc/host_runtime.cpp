// Host runtime: NCW1 reader, tokenizer, chunker, WNC encoder, NC05 container,
// parameter validation.  Pure C++ (no CUDA); exercised on CPU by the tests.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>

#include "nc_internal.hpp"

namespace nc {

// ------------------------------------------------------------------ NCW1 ---
NcwFile read_ncw(const std::string &path) {
  NcwFile f;
  std::ifstream is(path, std::ios::binary | std::ios::ate);
  if (!is) fail(NC_ERR_INVALID, "cannot open weight file " + path);
  size_t n = (size_t)is.tellg();
  is.seekg(0);
  f.raw.resize(n);
  if (!is.read(f.raw.data(), (std::streamsize)n)) fail(NC_ERR_FORMAT, "read failed: " + path);
  if (n < 64 || std::memcmp(f.raw.data(), "NCW1", 4) != 0) fail(NC_ERR_FORMAT, "not an NCW1 file");
  uint32_t h[10];
  std::memcpy(h, f.raw.data() + 4, sizeof(h));
  if (h[0] != 1) fail(NC_ERR_FORMAT, "unsupported NCW1 version");
  Shape &s = f.s;
  s.n_layers = h[1]; s.d = h[2]; s.H = h[3]; s.KV = h[4]; s.dh = h[5]; s.d_ff = h[6];
  s.V = h[7]; s.bos = h[8]; s.n_special = h[9];
  std::memcpy(&s.rope_theta, f.raw.data() + 44, 8);
  std::memcpy(&s.eps, f.raw.data() + 52, 8);
  uint64_t per_layer = 2ull * s.d + (uint64_t)(s.H * s.dh + 2 * s.KV * s.dh) * s.d +
                       (uint64_t)s.d * s.H * s.dh + 3ull * s.d * s.d_ff;
  uint64_t nf = (uint64_t)s.V * s.d + s.n_layers * per_layer + s.d;
  size_t off = 64 + nf * 4;
  if (off + 4 > n) fail(NC_ERR_FORMAT, "NCW1 truncated (tensors)");
  uint32_t nv;
  std::memcpy(&nv, f.raw.data() + off, 4);
  off += 4;
  if (nv != s.V) fail(NC_ERR_FORMAT, "NCW1 vocab count mismatch");
  f.vocab.resize(nv);
  for (uint32_t i = 0; i < nv; ++i) {
    if (off + 2 > n) fail(NC_ERR_FORMAT, "NCW1 truncated (vocab)");
    uint16_t ln;
    std::memcpy(&ln, f.raw.data() + off, 2);
    off += 2;
    if (off + ln > n) fail(NC_ERR_FORMAT, "NCW1 truncated (vocab)");
    f.vocab[i].assign(f.raw.data() + off, ln);
    off += ln;
  }
  if (off != n) fail(NC_ERR_FORMAT, "NCW1 trailing bytes");
  return f;
}

// ------------------------------------------------------------- tokenizer ---
// Trie with sorted child edges; greedy longest match (D30).
void Tokenizer::build(const std::vector<std::string> &vocab, uint32_t n_special) {
  vocab_ = vocab;
  // build with temporary maps, then flatten
  struct TNode {
    int32_t tok = -1;
    std::vector<std::pair<uint8_t, uint32_t>> kids;
  };
  std::vector<TNode> t(1);
  for (uint32_t id = n_special; id < vocab.size(); ++id) {
    const std::string &s = vocab[id];
    if (s.empty()) continue;
    uint32_t cur = 0;
    for (unsigned char c : s) {
      uint32_t nxt = UINT32_MAX;
      for (auto &kv : t[cur].kids)
        if (kv.first == c) { nxt = kv.second; break; }
      if (nxt == UINT32_MAX) {
        nxt = (uint32_t)t.size();
        t[cur].kids.push_back({c, nxt});
        t.emplace_back();
      }
      cur = nxt;
    }
    if (t[cur].tok < 0) t[cur].tok = (int32_t)id;  // first id wins for duplicate strings
  }
  nodes_.assign(t.size(), Node());
  edges_.clear();
  for (size_t i = 0; i < t.size(); ++i) {
    std::sort(t[i].kids.begin(), t[i].kids.end());
    nodes_[i].tok = t[i].tok;
    nodes_[i].first = (uint32_t)edges_.size();
    nodes_[i].count = (uint32_t)t[i].kids.size();
    for (auto &kv : t[i].kids) edges_.push_back({kv.first, kv.second});
  }
  for (int b = 0; b < 256; ++b) root_children_[b] = UINT32_MAX;
  for (uint32_t e = nodes_[0].first; e < nodes_[0].first + nodes_[0].count; ++e)
    root_children_[edges_[e].byte] = edges_[e].child;
}

void Tokenizer::encode(const uint8_t *data, size_t n, std::vector<uint32_t> &out) const {
  size_t i = 0;
  while (i < n) {
    int32_t best = -1;
    size_t best_len = 0;
    uint32_t cur = root_children_[data[i]];
    size_t j = i + 1;
    while (cur != UINT32_MAX) {
      if (nodes_[cur].tok >= 0) { best = nodes_[cur].tok; best_len = j - i; }
      if (j >= n) break;
      const Node &nd = nodes_[cur];
      uint8_t c = data[j];
      uint32_t lo = nd.first, hi = nd.first + nd.count, nxt = UINT32_MAX;
      while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (edges_[mid].byte < c) lo = mid + 1;
        else hi = mid;
      }
      if (lo < nd.first + nd.count && edges_[lo].byte == c) nxt = edges_[lo].child;
      cur = nxt;
      ++j;
    }
    if (best < 0) fail(NC_ERR_INVALID, "byte not in vocabulary");
    out.push_back((uint32_t)best);
    i += best_len;
  }
}

void Tokenizer::decode(const uint32_t *ids, size_t n, std::string &out) const {
  for (size_t i = 0; i < n; ++i) {
    if (ids[i] >= vocab_.size()) fail(NC_ERR_INTEGRITY, "decoded token id out of range");
    out += vocab_[ids[i]];
  }
}

// ---------------------------------------------------------------- chunks ---
std::vector<uint64_t> split_chunks(const uint8_t *in, size_t n, uint32_t n_chunks) {
  std::vector<uint64_t> cuts{0};
  if (n_chunks > 1 && n > 0) {
    uint64_t step = (n + n_chunks - 1) / n_chunks;
    for (uint32_t i = 1; i < n_chunks; ++i) {
      uint64_t target = std::max<uint64_t>((uint64_t)i * step, cuts.back());
      if (target >= n) break;
      const void *p = std::memchr(in + target, '\n', n - target);
      uint64_t cut = p ? (uint64_t)((const uint8_t *)p - in) + 1 : target;
      if (cut >= n) break;
      if (cut > cuts.back()) cuts.push_back(cut);
    }
  }
  cuts.push_back(n);
  return cuts;
}

// ------------------------------------------------------------------- WNC ---
static constexpr uint64_t kHalf = 1ull << 31, kQuarter = 1ull << 30, kThreeQ = 3ull << 30;

void WncEncoder::put(uint32_t bit) {
  acc_ = (acc_ << 1) | bit;
  if (++nacc_ == 8) { bytes_.push_back((uint8_t)acc_); acc_ = 0; nacc_ = 0; }
  ++nbits_;
}
void WncEncoder::emit(uint32_t bit) {
  put(bit);
  for (; pending_ > 0; --pending_) put(bit ^ 1u);
}
void WncEncoder::encode(uint32_t cum_lo, uint32_t freq, uint32_t cdf_bits) {
  if (freq == 0) fail(NC_ERR_INTEGRITY, "zero-width symbol interval");
  uint64_t R = high_ - low_ + 1;
  high_ = low_ + ((R * (uint64_t)(cum_lo + (uint64_t)freq)) >> cdf_bits) - 1;
  low_ = low_ + ((R * (uint64_t)cum_lo) >> cdf_bits);
  for (;;) {
    if (high_ < kHalf) {
      emit(0);
    } else if (low_ >= kHalf) {
      emit(1);
      low_ -= kHalf; high_ -= kHalf;
    } else if (low_ >= kQuarter && high_ < kThreeQ) {
      ++pending_;
      low_ -= kQuarter; high_ -= kQuarter;
    } else {
      break;
    }
    low_ = 2 * low_;
    high_ = 2 * high_ + 1;
  }
}
void WncEncoder::finish(std::vector<uint8_t> &out, uint64_t &bit_count) {
  ++pending_;
  emit(low_ < kQuarter ? 0u : 1u);
  bit_count = nbits_;
  if (nacc_) { bytes_.push_back((uint8_t)(acc_ << (8 - nacc_))); acc_ = 0; nacc_ = 0; }
  out.swap(bytes_);
}

// ------------------------------------------------------------------ rANS ---
void ans_encode(const uint32_t *cum, const uint32_t *freq, size_t n, uint32_t cdf_bits,
                std::vector<uint8_t> &out, uint64_t &bit_count) {
  constexpr uint64_t L = 1ull << 31;
  uint64_t x = L;
  std::vector<uint32_t> words;                       // in emission order (reversed below)
  for (size_t k = n; k-- > 0;) {                     // rANS codes the symbols in reverse
    const uint64_t f = freq[k];
    if (f == 0) fail(NC_ERR_INTEGRITY, "zero-width symbol interval");
    const uint64_t x_max = ((L >> cdf_bits) << 32) * f;
    if (x >= x_max) {
      words.push_back((uint32_t)x);
      x >>= 32;
    }
    x = ((x / f) << cdf_bits) + x % f + cum[k];
  }
  words.push_back((uint32_t)x);                      // flush: low, then high (reversed: high first)
  words.push_back((uint32_t)(x >> 32));
  out.clear();
  out.reserve(4 * words.size());
  for (size_t k = words.size(); k-- > 0;)
    for (int by = 3; by >= 0; --by) out.push_back((uint8_t)(words[k] >> (8 * by)));
  bit_count = 32ull * words.size();
}

// ------------------------------------------------------------------ NC05 ---
static void put_u16(std::vector<uint8_t> &o, uint16_t v) { o.push_back(v & 255); o.push_back(v >> 8); }
static void put_u32(std::vector<uint8_t> &o, uint32_t v) {
  for (int i = 0; i < 4; ++i) o.push_back((v >> (8 * i)) & 255);
}
static uint32_t get_u32(const uint8_t *p) { return p[0] | (p[1] << 8) | (p[2] << 16) | ((uint32_t)p[3] << 24); }

void write_nc05(uint8_t flags, uint16_t tau_milli, const std::vector<Nc05Chunk> &chunks,
                std::vector<uint8_t> &out) {
  if (chunks.size() > 0xFFFF) fail(NC_ERR_INVALID, "too many chunks for NC05");
  size_t total = 9 + 12 * chunks.size();
  for (auto &c : chunks) total += c.stream.size();
  out.clear();
  out.reserve(total);
  out.insert(out.end(), {'N', 'C', '0', '5'});
  out.push_back(flags);
  put_u16(out, tau_milli);
  put_u16(out, (uint16_t)chunks.size());
  for (auto &c : chunks) {
    if (c.stream.size() != (c.bits + 7ull) / 8) fail(NC_ERR_INTEGRITY, "stream_len != ceil(bits/8)");
    put_u32(out, c.tokens);
    put_u32(out, c.bits);
    put_u32(out, (uint32_t)c.stream.size());
  }
  for (auto &c : chunks) out.insert(out.end(), c.stream.begin(), c.stream.end());
}

Nc05View read_nc05(const uint8_t *in, size_t n) {
  Nc05View v;
  if (n < 9) fail(NC_ERR_TRUNCATED, "NC05 header truncated");
  if (std::memcmp(in, "NC05", 4) != 0) fail(NC_ERR_FORMAT, "bad magic");
  v.flags = in[4];
  v.tau_milli = (uint16_t)(in[5] | (in[6] << 8));
  uint32_t nch = in[7] | (in[8] << 8);
  if (v.flags & ~0x07u) fail(NC_ERR_FORMAT, "reserved flag bits set");
  if (v.tau_milli == 0) fail(NC_ERR_FORMAT, "temperature 0");
  if (n < 9 + 12ull * nch) fail(NC_ERR_TRUNCATED, "NC05 chunk table truncated");
  uint64_t off = 9 + 12ull * nch;
  for (uint32_t i = 0; i < nch; ++i) {
    const uint8_t *e = in + 9 + 12 * i;
    Nc05View::Ent ent{get_u32(e), get_u32(e + 4), get_u32(e + 8), off};
    if (ent.len != (ent.bits + 7ull) / 8) fail(NC_ERR_FORMAT, "stream_len != ceil(bit_count/8)");
    if (ent.tokens > (uint32_t)INT32_MAX) fail(NC_ERR_FORMAT, "token_count out of range");
    off += ent.len;
    if (off > n) fail(NC_ERR_TRUNCATED, "NC05 stream truncated");
    v.ents.push_back(ent);
  }
  if (off != n) fail(NC_ERR_FORMAT, "NC05 trailing bytes");
  return v;
}

// ---------------------------------------------------------------- params ---
Params validate(const nc_params *p) {
  nc_params d;
  nc_params_default(&d);
  if (!p) p = &d;
  Params q;
  q.cdf_bits = p->cdf_bits;
  q.flags = p->flags;
  if (!(q.cdf_bits == 16 || q.cdf_bits == 24)) fail(NC_ERR_INVALID, "cdf_bits must be 16 or 24");
  if (q.flags & ~7u) fail(NC_ERR_INVALID, "flags: only NGRAM | HEAD | SKIP (bits 0-2) are defined");
  if (!(p->temperature > 0.f)) fail(NC_ERR_INVALID, "temperature must be > 0");
  double tm = std::nearbyint((double)p->temperature * 1000.0);
  if (tm < 1 || tm > 65535) fail(NC_ERR_INVALID, "temperature out of the u16 milli range");
  q.tau_milli = (uint32_t)tm;
  q.inv_tau = 1000.0 / tm;
  q.window = p->window;
  q.slide = p->slide;
  if (q.window == 0 || q.window % 128 || q.slide == 0 || q.slide % 128 || q.slide >= q.window)
    fail(NC_ERR_INVALID, "window/slide must be multiples of 128 with slide < window");
  q.warmup = p->warmup;
  q.eta = p->eta;
  q.alpha = p->alpha;
  q.orders = p->ngram_orders;
  if (q.orders < 1 || q.orders > 4) fail(NC_ERR_INVALID, "ngram_orders must be 1..4");
  q.cap = p->ngram_cap;
  if (q.cap == 0) fail(NC_ERR_INVALID, "ngram_cap must be > 0");
  q.n_chunks = p->n_chunks;
  q.chunks_per_gpu = p->chunks_per_gpu ? p->chunks_per_gpu : 64;
  q.max_slab_rows = p->max_slab_rows ? p->max_slab_rows : 32768;
  q.debug_dump = p->debug_dump;
  if (p->window_variant & ~3u) fail(NC_ERR_INVALID, "window_variant: only bits 0-1 are defined");
  q.refresh = (p->window_variant & NC_WINDOW_REFRESH) != 0;
  if (p->coder > NC_CODER_ANS) fail(NC_ERR_INVALID, "coder must be NC_CODER_WNC or NC_CODER_ANS");
  q.coder = p->coder;
  q.lmax = (p->window_variant & NC_WINDOW_LMAX_M1) ? q.window - 1 : q.window;
  return q;
}

}  // namespace nc
