// HF-format SmolLM2 checkpoints and their byte-level BPE tokenizer (
// P:269-282 the SmolLM2-135M model, P:305-311 its HF tokenizer; readings D35-D36).
//
//   read_hf(dir): config.json + model.safetensors (F32 / F16 / BF16 tensors, HF Llama
//     names) -> the NCW1 tensor order in memory (fp32), vocabulary bytes from tokenizer.json
//   BpeTokenizer: tokenizer.json's BPE (vocab + ranked merges) behind SmolLM2's
//     pre-tokenizer -- Digits(individual_digits) then ByteLevel(use_regex) with the GPT-2
//     pattern  's|'t|'re|'ve|'m|'ll|'d| ?\p{L}+| ?\p{N}+| ?[^\s\p{L}\p{N}]+|\s+(?!\S)|\s+
//     scanned by hand over code points (Unicode L / N tables generated from unicodedata);
//     bytes map to the GPT-2 byte-level alphabet; the lowest-ranked adjacent pair merges
//     first, leftmost on ties.  Invalid UTF-8 bytes are single "other" characters (D35), so
//     any byte string tokenizes and decode(encode(x)) == x.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <unordered_map>

#include "hf.hpp"
#include "json.hpp"

namespace nc {

namespace {
#include "unicode_tables.inc"

bool in_ranges(const uint32_t (*r)[2], size_t n, uint32_t cp) {
  size_t lo = 0, hi = n;
  while (lo < hi) {
    const size_t mid = (lo + hi) / 2;
    if (cp < r[mid][0]) hi = mid;
    else if (cp > r[mid][1]) lo = mid + 1;
    else return true;
  }
  return false;
}
bool is_L(uint32_t cp) { return in_ranges(kUniL, sizeof(kUniL) / sizeof(kUniL[0]), cp); }
bool is_N(uint32_t cp) { return in_ranges(kUniN, sizeof(kUniN) / sizeof(kUniN[0]), cp); }
bool is_WS(uint32_t cp) {   // Unicode White_Space
  return (cp >= 9 && cp <= 13) || cp == 0x20 || cp == 0x85 || cp == 0xA0 || cp == 0x1680 ||
         (cp >= 0x2000 && cp <= 0x200A) || cp == 0x2028 || cp == 0x2029 || cp == 0x202F || cp == 0x205F ||
         cp == 0x3000;
}

std::string read_file(const std::string &path) {
  std::ifstream is(path, std::ios::binary | std::ios::ate);
  if (!is) fail(NC_ERR_INVALID, "cannot open " + path);
  const size_t n = (size_t)is.tellg();
  is.seekg(0);
  std::string s(n, '\0');
  if (!is.read(&s[0], (std::streamsize)n)) fail(NC_ERR_FORMAT, "read failed: " + path);
  return s;
}

// GPT-2 byte-level alphabet: byte -> code point
uint32_t byte_cp(uint8_t b) {
  static uint32_t map[256];
  static bool init = false;
  if (!init) {
    bool direct[256] = {};
    for (int c = '!'; c <= '~'; ++c) direct[c] = true;
    for (int c = 0xA1; c <= 0xAC; ++c) direct[c] = true;
    for (int c = 0xAE; c <= 0xFF; ++c) direct[c] = true;
    uint32_t n = 0;
    for (int c = 0; c < 256; ++c) map[c] = direct[c] ? (uint32_t)c : 256 + n++;
    init = true;
  }
  return map[b];
}

// decode one UTF-8 code point at p (invalid -> the byte itself, length 1, valid = false)
uint32_t utf8_next(const uint8_t *p, size_t n, size_t &len, bool &valid) {
  const uint8_t c = p[0];
  valid = true;
  if (c < 0x80) { len = 1; return c; }
  int k = 0;
  uint32_t cp = 0, minv = 0;
  if ((c & 0xE0) == 0xC0) { k = 1; cp = c & 0x1F; minv = 0x80; }
  else if ((c & 0xF0) == 0xE0) { k = 2; cp = c & 0x0F; minv = 0x800; }
  else if ((c & 0xF8) == 0xF0) { k = 3; cp = c & 0x07; minv = 0x10000; }
  else { len = 1; valid = false; return c; }
  if ((size_t)k + 1 > n) { len = 1; valid = false; return c; }
  for (int i = 1; i <= k; ++i) {
    if ((p[i] & 0xC0) != 0x80) { len = 1; valid = false; return c; }
    cp = (cp << 6) | (p[i] & 0x3F);
  }
  if (cp < minv || cp > 0x10FFFF || (cp >= 0xD800 && cp < 0xE000)) { len = 1; valid = false; return c; }
  len = (size_t)k + 1;
  return cp;
}

void append_utf8(std::string &o, uint32_t cp) {
  if (cp < 0x80) o += (char)cp;
  else if (cp < 0x800) { o += (char)(0xC0 | (cp >> 6)); o += (char)(0x80 | (cp & 63)); }
  else { o += (char)(0xE0 | (cp >> 12)); o += (char)(0x80 | ((cp >> 6) & 63)); o += (char)(0x80 | (cp & 63)); }
}
}  // namespace

// ------------------------------------------------------------------ BPE ---
void BpeTokenizer::build(const std::string &tokenizer_json, uint32_t V, std::vector<std::string> &vocab_bytes,
                         uint32_t &n_special) {
  const Json tj = Json::parse(tokenizer_json.data(), tokenizer_json.size());
  const Json &model = tj.at("model");
  if (model.at("type").string() != "BPE") fail(NC_ERR_INVALID, "tokenizer.json: only BPE models are supported");
  if (const Json *bf = model.get("byte_fallback"); bf && bf->kind == Json::Bool && bf->b)
    fail(NC_ERR_INVALID, "tokenizer.json: byte_fallback BPE is not supported");
  // pre-tokenizer: ByteLevel, optionally after Digits(individual_digits = true)
  digits_ = false;
  const Json &pt = tj.at("pre_tokenizer");
  auto check_bl = [&](const Json &j) {
    if (j.at("type").string() != "ByteLevel") fail(NC_ERR_INVALID, "tokenizer.json: unsupported pre-tokenizer");
    if (const Json *a = j.get("add_prefix_space"); a && a->b) fail(NC_ERR_INVALID, "add_prefix_space unsupported");
    if (const Json *u = j.get("use_regex"); u && u->kind == Json::Bool && !u->b) fail(NC_ERR_INVALID, "use_regex=false unsupported");
  };
  if (pt.at("type").string() == "Sequence") {
    const Json &seq = pt.at("pretokenizers");
    if (seq.arr.size() == 2 && seq.arr[0].at("type").string() == "Digits") {
      if (!seq.arr[0].at("individual_digits").b) fail(NC_ERR_INVALID, "Digits(individual_digits=false) unsupported");
      digits_ = true;
      check_bl(seq.arr[1]);
    } else if (seq.arr.size() == 1) {
      check_bl(seq.arr[0]);
    } else {
      fail(NC_ERR_INVALID, "tokenizer.json: unsupported pre-tokenizer sequence");
    }
  } else {
    check_bl(pt);
  }
  // vocabulary: token string (byte-level alphabet) -> id
  uint32_t inv[0x200] = {};
  for (int b = 0; b < 256; ++b) inv[byte_cp((uint8_t)b)] = (uint32_t)b + 1;
  vocab_bytes.assign(V, std::string());
  std::unordered_map<std::string, uint32_t> ids;
  for (const auto &kv : model.at("vocab").obj) {
    const uint32_t id = (uint32_t)kv.second.number();
    if (id >= V) fail(NC_ERR_INVALID, "tokenizer id beyond the model's vocabulary");
    ids[kv.first] = id;
    std::string bytes;
    const uint8_t *p = reinterpret_cast<const uint8_t *>(kv.first.data());
    for (size_t i = 0, len = 0; i < kv.first.size(); i += len) {
      bool ok;
      const uint32_t cp = utf8_next(p + i, kv.first.size() - i, len, ok);
      if (!ok || cp >= 0x200 || !inv[cp]) { bytes.clear(); break; }   // not a byte-level token
      bytes += (char)(inv[cp] - 1);
    }
    vocab_bytes[id] = bytes;
  }
  n_special = 0;
  if (const Json *at = tj.get("added_tokens"))
    for (const Json &t : at->arr) {
      const uint32_t id = (uint32_t)t.at("id").number();
      if (id >= V) fail(NC_ERR_INVALID, "added token beyond the vocabulary");
      vocab_bytes[id] = t.at("content").string();   // specials are never produced from input (D35)
      if (t.get("special") && t.at("special").b) ++n_special;
    }
  for (int b = 0; b < 256; ++b) {
    std::string s;
    append_utf8(s, byte_cp((uint8_t)b));
    auto it = ids.find(s);
    if (it == ids.end()) fail(NC_ERR_INVALID, "tokenizer.json: byte-level alphabet incomplete");
    byte_id_[b] = it->second;
  }
  // merges: "a b" strings or [a, b] pairs, rank = position
  merges_.clear();
  const Json &mg = model.at("merges");
  for (size_t r = 0; r < mg.arr.size(); ++r) {
    std::string a, b;
    if (mg.arr[r].kind == Json::Str) {
      const std::string &s = mg.arr[r].str;
      const size_t sp = s.find(' ');
      if (sp == std::string::npos) fail(NC_ERR_FORMAT, "tokenizer.json: bad merge");
      a = s.substr(0, sp);
      b = s.substr(sp + 1);
    } else {
      a = mg.arr[r].arr.at(0).string();
      b = mg.arr[r].arr.at(1).string();
    }
    auto ia = ids.find(a), ib = ids.find(b), im = ids.find(a + b);
    if (ia == ids.end() || ib == ids.end() || im == ids.end()) fail(NC_ERR_FORMAT, "tokenizer.json: merge of unknown tokens");
    const uint64_t key = ((uint64_t)ia->second << 32) | ib->second;
    if (!merges_.count(key)) merges_[key] = Merge{(uint32_t)r, im->second};
  }
}

// BPE of one pre-token (bytes): start from the byte symbols, merge the lowest-ranked
// adjacent pair (leftmost on ties) until no pair has a merge
void BpeTokenizer::bpe_word(const uint8_t *w, size_t n, std::vector<uint32_t> &out) const {
  std::vector<uint32_t> sym(n);
  for (size_t i = 0; i < n; ++i) sym[i] = byte_id_[w[i]];
  while (sym.size() > 1) {
    uint32_t best = UINT32_MAX, best_id = 0;
    size_t at = 0;
    for (size_t i = 0; i + 1 < sym.size(); ++i) {
      auto it = merges_.find(((uint64_t)sym[i] << 32) | sym[i + 1]);
      if (it != merges_.end() && it->second.rank < best) { best = it->second.rank; best_id = it->second.id; at = i; }
    }
    if (best == UINT32_MAX) break;
    sym[at] = best_id;
    sym.erase(sym.begin() + at + 1);
  }
  out.insert(out.end(), sym.begin(), sym.end());
}

void BpeTokenizer::encode(const uint8_t *data, size_t n, std::vector<uint32_t> &out) const {
  enum Cls : uint8_t { L_, N_, WS_, O_ };
  struct U { uint32_t off, len, cp; Cls c; };
  std::vector<U> u;
  u.reserve(n);
  for (size_t i = 0, len = 0; i < n; i += len) {
    bool ok;
    const uint32_t cp = utf8_next(data + i, n - i, len, ok);
    const Cls c = !ok ? O_ : is_WS(cp) ? WS_ : is_L(cp) ? L_ : is_N(cp) ? N_ : O_;
    u.push_back(U{(uint32_t)i, (uint32_t)len, ok ? cp : 0xFFFFFFFFu, c});
  }
  auto emit = [&](size_t a, size_t b) {   // units [a, b)
    if (a >= b) return;
    bpe_word(data + u[a].off, (size_t)(u[b - 1].off + u[b - 1].len - u[a].off), out);
  };
  auto regex_split = [&](size_t a, size_t b) {   // the GPT-2 pattern over units [a, b)
    static const char *kContr[] = {"s", "t", "re", "ve", "m", "ll", "d"};
    size_t i = a;
    while (i < b) {
      if (u[i].cp == '\'') {   // 's|'t|'re|'ve|'m|'ll|'d (in this order, case-sensitive)
        bool hit = false;
        for (const char *sfx : kContr) {
          const size_t L = std::strlen(sfx);
          bool m = i + L < b;
          for (size_t k = 0; m && k < L; ++k) m = u[i + 1 + k].cp == (uint32_t)sfx[k];
          if (m) { emit(i, i + 1 + L); i += 1 + L; hit = true; break; }
        }
        if (hit) continue;
      }
      bool sp = u[i].cp == ' ' && i + 1 < b;
      for (Cls want : {L_, N_, O_}) {
        size_t j = (sp && u[i + 1].c == want) ? i + 1 : i;
        if (u[j].c == want) {
          size_t k = j;
          while (k < b && u[k].c == want) ++k;
          emit(i, k);
          i = k;
          goto next;
        }
      }
      {   // whitespace: \s+(?!\S) | \s+
        size_t k = i;
        while (k < b && u[k].c == WS_) ++k;
        const size_t e = (k == b || k - i < 2) ? k : k - 1;
        emit(i, e);
        i = e;
      }
    next:;
    }
  };
  if (!digits_) {
    regex_split(0, u.size());
    return;
  }
  // Digits(individual_digits): every numeric character is its own piece
  size_t s = 0;
  for (size_t i = 0; i < u.size(); ++i)
    if (u[i].c == N_) {
      regex_split(s, i);
      regex_split(i, i + 1);
      s = i + 1;
    }
  regex_split(s, u.size());
}

// ----------------------------------------------------------- safetensors ---
NcwFile read_hf(const std::string &dir, std::unique_ptr<BpeTokenizer> &bpe) {
  NcwFile f;
  const std::string cfg_s = read_file(dir + "/config.json");
  const Json cfg = Json::parse(cfg_s.data(), cfg_s.size());
  auto num = [&](const char *k, double dflt) {
    const Json *j = cfg.get(k);
    return (j && j->kind == Json::Num) ? j->num : dflt;
  };
  Shape &s = f.s;
  s.d = (uint32_t)cfg.at("hidden_size").number();
  s.n_layers = (uint32_t)cfg.at("num_hidden_layers").number();
  s.H = (uint32_t)cfg.at("num_attention_heads").number();
  s.KV = (uint32_t)num("num_key_value_heads", s.H);
  s.dh = (uint32_t)num("head_dim", s.d / s.H);
  s.d_ff = (uint32_t)cfg.at("intermediate_size").number();
  s.V = (uint32_t)cfg.at("vocab_size").number();
  s.bos = (uint32_t)num("bos_token_id", 0);
  s.eps = num("rms_norm_eps", 1e-6);
  s.rope_theta = num("rope_theta", 10000.0);
  if (const Json *rp = cfg.get("rope_parameters"); rp && rp->kind == Json::Obj) {
    if (const Json *t = rp->get("rope_theta")) s.rope_theta = t->number();
    if (const Json *ty = rp->get("rope_type"); ty && ty->kind == Json::Str && ty->str != "default")
      fail(NC_ERR_INVALID, "config.json: only default RoPE is supported");
  }
  if (const Json *rs = cfg.get("rope_scaling"); rs && rs->kind != Json::Null)
    fail(NC_ERR_INVALID, "config.json: rope_scaling is not supported");
  if (const Json *t = cfg.get("tie_word_embeddings"); !t || t->kind != Json::Bool || !t->b)
    fail(NC_ERR_INVALID, "config.json: the head must be tied to the embedding (SmolLM2, D16)");
  if (const Json *a = cfg.get("hidden_act"); a && a->kind == Json::Str && a->str != "silu")
    fail(NC_ERR_INVALID, "config.json: only SiLU MLPs are supported");

  const std::string st = read_file(dir + "/model.safetensors");
  if (st.size() < 8) fail(NC_ERR_FORMAT, "safetensors truncated");
  uint64_t hn;
  std::memcpy(&hn, st.data(), 8);
  if (8 + hn > st.size()) fail(NC_ERR_FORMAT, "safetensors header truncated");
  const Json hdr = Json::parse(st.data() + 8, hn);
  const size_t base = 8 + hn;
  const size_t d = s.d, qd = (size_t)s.H * s.dh, kvd = (size_t)s.KV * s.dh, ff = s.d_ff, V = s.V;
  const uint64_t per_layer = 2ull * d + (qd + 2 * kvd) * d + d * qd + 3ull * d * ff;
  const uint64_t nf = V * d + s.n_layers * per_layer + d;
  f.raw.assign(f.tensor_off + nf * 4, 0);
  float *dst = reinterpret_cast<float *>(f.raw.data() + f.tensor_off);
  auto take = [&](const std::string &name, std::vector<uint64_t> shape) {
    const Json *t = hdr.get(name);
    if (!t) fail(NC_ERR_FORMAT, "safetensors: missing tensor " + name);
    const std::string &dt = t->at("dtype").string();
    const Json &sh = t->at("shape");
    uint64_t cnt = 1;
    if (sh.arr.size() != shape.size()) fail(NC_ERR_FORMAT, "safetensors: rank mismatch for " + name);
    for (size_t i = 0; i < shape.size(); ++i) {
      if ((uint64_t)sh.arr[i].number() != shape[i]) fail(NC_ERR_FORMAT, "safetensors: shape mismatch for " + name);
      cnt *= shape[i];
    }
    const uint64_t b0 = (uint64_t)t->at("data_offsets").arr.at(0).number();
    const uint64_t b1 = (uint64_t)t->at("data_offsets").arr.at(1).number();
    const size_t es = dt == "F32" ? 4 : (dt == "F16" || dt == "BF16") ? 2 : 0;
    if (!es) fail(NC_ERR_INVALID, "safetensors: unsupported dtype " + dt);
    if (b1 - b0 != cnt * es || base + b1 > st.size()) fail(NC_ERR_FORMAT, "safetensors: bad offsets for " + name);
    const uint8_t *src = reinterpret_cast<const uint8_t *>(st.data() + base + b0);
    for (uint64_t i = 0; i < cnt; ++i) {
      float v;
      if (es == 4) {
        std::memcpy(&v, src + 4 * i, 4);
      } else {
        uint16_t h;
        std::memcpy(&h, src + 2 * i, 2);
        if (dt == "BF16") {
          const uint32_t w = (uint32_t)h << 16;
          std::memcpy(&v, &w, 4);
        } else {   // IEEE half
          const uint32_t sgn = (h >> 15) & 1, ex = (h >> 10) & 31, man = h & 1023;
          float m = ex == 0 ? std::ldexp((float)man, -24) : ex == 31 ? (man ? NAN : INFINITY)
                                                                     : std::ldexp((float)(man | 1024), (int)ex - 25);
          v = sgn ? -m : m;
        }
      }
      *dst++ = v;
    }
  };
  take("model.embed_tokens.weight", {V, d});
  for (uint32_t l = 0; l < s.n_layers; ++l) {
    const std::string p = "model.layers." + std::to_string(l) + ".";
    take(p + "input_layernorm.weight", {d});
    take(p + "self_attn.q_proj.weight", {qd, d});
    take(p + "self_attn.k_proj.weight", {kvd, d});
    take(p + "self_attn.v_proj.weight", {kvd, d});
    take(p + "self_attn.o_proj.weight", {d, qd});
    take(p + "post_attention_layernorm.weight", {d});
    take(p + "mlp.gate_proj.weight", {ff, d});
    take(p + "mlp.up_proj.weight", {ff, d});
    take(p + "mlp.down_proj.weight", {d, ff});
  }
  take("model.norm.weight", {d});

  bpe.reset(new BpeTokenizer());
  const std::string tj = read_file(dir + "/tokenizer.json");
  bpe->build(tj, s.V, f.vocab, s.n_special);
  return f;
}

}  // namespace nc
