// extern "C" boundary of libnc.so (include/nc.h).  Argument marshalling,
// error capture and container plumbing only; all compute is in the engine.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <thread>
#include <vector>

#include "engine.hpp"
#include "nc06.hpp"

namespace {
thread_local std::string g_err;
}  // namespace
void nc::set_last_error(const std::string &m) { g_err = m; }
namespace {

nc_status set_err(nc_status c, const std::string &m) {
  g_err = m;
  return c;
}

template <class F>
nc_status guard(F &&f) {
  try {
    f();
    return NC_OK;
  } catch (nc::Error &e) {
    return set_err(e.code, e.what());
  } catch (std::bad_alloc &) {
    return set_err(NC_ERR_NOMEM, "host allocation failed");
  } catch (std::exception &e) {
    return set_err(NC_ERR_BACKEND, e.what());
  }
}

template <class T>
T *dup_out(const std::vector<T> &v) {
  T *p = static_cast<T *>(std::malloc(v.empty() ? 1 : v.size() * sizeof(T)));
  if (!p) throw std::bad_alloc();
  if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
  return p;
}

void require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    nc::fail(NC_ERR_BACKEND, "no CUDA device available (libnc has no CPU fallback)");
}

uint32_t effective_chunks(const nc::Params &p, int world) {
  return p.n_chunks ? p.n_chunks : (uint32_t)world * p.chunks_per_gpu;
}
}  // namespace

extern "C" {

void nc_params_default(nc_params *p) {
  if (!p) return;
  std::memset(p, 0, sizeof(*p));
  p->cdf_bits = 24;
  p->flags = NC_FLAG_NGRAM | NC_FLAG_HEAD;
  p->temperature = 1.0f;
  p->window = 2048;
  p->slide = 512;
  p->warmup = 100;
  p->eta = 1.0;
  p->alpha = 1e-3;
  p->ngram_orders = 4;
  p->ngram_cap = 500000;
  p->n_chunks = 0;
  p->chunks_per_gpu = 64;
  p->max_slab_rows = 32768;
  p->debug_dump = 0;
  p->window_variant = 0;
  p->coder = NC_CODER_WNC;
}

nc_status nc_set_allocator(void *(*alloc)(size_t, void *), void (*free_fn)(void *, void *), void *ctx) {
  if ((alloc == nullptr) != (free_fn == nullptr)) return set_err(NC_ERR_INVALID, "alloc and free must both be set");
  nc::set_allocator(alloc, free_fn, ctx);
  return NC_OK;
}

nc_status nc_model_load(const char *path, int device, nc_model **out) {
  if (!path || !out) return set_err(NC_ERR_INVALID, "null argument");
  *out = nullptr;
  nc_model *m = new nc_model();
  nc_status st = guard([&] {
    require_device();
    nc::model_load(m, path, device);
  });
  if (st != NC_OK) {
    nc::model_free(m);
    delete m;
    return st;
  }
  *out = m;
  return NC_OK;
}

void nc_model_free(nc_model *m) {
  if (!m) return;
  nc::model_free(m);
  delete m;
}

nc_status nc_model_load_hf(const char *model_dir, int device, nc_model **out) {
  if (!model_dir || !out) return set_err(NC_ERR_INVALID, "null argument");
  *out = nullptr;
  nc_model *m = new nc_model();
  nc_status st = guard([&] {
    require_device();
    nc::model_load_hf(m, model_dir, device);
  });
  if (st != NC_OK) {
    nc::model_free(m);
    delete m;
    return st;
  }
  *out = m;
  return NC_OK;
}

nc_status nc_host_bpe_encode(const char *tokenizer_json_path, uint32_t vocab, const uint8_t *in, size_t n,
                             uint32_t **tokens, size_t *n_tokens) {
  if (!tokenizer_json_path || (!in && n) || !tokens || !n_tokens) return set_err(NC_ERR_INVALID, "null argument");
  *tokens = nullptr; *n_tokens = 0;
  return guard([&] {
    std::ifstream is(tokenizer_json_path, std::ios::binary);
    if (!is) nc::fail(NC_ERR_INVALID, std::string("cannot open ") + tokenizer_json_path);
    std::string js((std::istreambuf_iterator<char>(is)), std::istreambuf_iterator<char>());
    nc::BpeTokenizer t;
    std::vector<std::string> vb;
    uint32_t ns = 0;
    t.build(js, vocab, vb, ns);
    std::vector<uint32_t> o;
    t.encode(in, n, o);
    *tokens = dup_out(o);
    *n_tokens = o.size();
  });
}

nc_status nc_model_info(const nc_model *m, uint32_t *vocab, uint32_t *n_layers, uint32_t *d_model) {
  if (!m) return set_err(NC_ERR_INVALID, "null model");
  if (vocab) *vocab = m->s.V;
  if (n_layers) *n_layers = m->s.n_layers;
  if (d_model) *d_model = m->s.d;
  return NC_OK;
}

static void tokenize_all(const nc_model *m, const uint8_t *in, size_t n, uint32_t n_chunks,
                         std::vector<uint32_t> &tokens, std::vector<uint32_t> &ntok) {
  std::vector<uint64_t> cuts = nc::split_chunks(in, n, n_chunks ? n_chunks : 1);
  const size_t nc_ = cuts.size() - 1;
  // chunks are independent: tokenize them on host threads (the trie is read-only)
  std::vector<std::vector<uint32_t>> per(nc_);
  const unsigned nt = std::max(1u, std::min<unsigned>((unsigned)nc_, std::thread::hardware_concurrency()));
  auto work = [&](unsigned t) {
    for (size_t c = t; c < nc_; c += nt) m->encode(in + cuts[c], cuts[c + 1] - cuts[c], per[c]);
  };
  if (nt <= 1 || n < (1u << 16)) {
    work(0);
    if (nt > 1)
      for (unsigned t = 1; t < nt; ++t) work(t);
  } else {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) th.emplace_back(work, t);
    for (auto &x : th) x.join();
  }
  tokens.clear();
  ntok.clear();
  size_t total = 0;
  for (auto &v : per) total += v.size();
  tokens.reserve(total);
  for (auto &v : per) {
    if (v.size() > 0xFFFFFFFFull) nc::fail(NC_ERR_INVALID, "chunk too long");
    ntok.push_back((uint32_t)v.size());
    tokens.insert(tokens.end(), v.begin(), v.end());
  }
}

nc_status nc_tokenize(const nc_model *m, const uint8_t *in, size_t n, uint32_t n_chunks, uint32_t **tokens,
                      size_t *n_tokens, uint32_t **chunk_ntok, uint32_t *n_chunks_out) {
  if (!m || (!in && n) || !tokens || !n_tokens || !chunk_ntok || !n_chunks_out)
    return set_err(NC_ERR_INVALID, "null argument");
  *tokens = nullptr; *chunk_ntok = nullptr; *n_tokens = 0; *n_chunks_out = 0;
  return guard([&] {
    std::vector<uint32_t> t, nt;
    tokenize_all(m, in, n, n_chunks, t, nt);
    *tokens = dup_out(t);
    *chunk_ntok = dup_out(nt);
    *n_tokens = t.size();
    *n_chunks_out = (uint32_t)nt.size();
  });
}

nc_status nc_compress_tokens(nc_model *m, const uint32_t *tokens_dev, const uint32_t *chunk_ntok, uint32_t n_chunks,
                             const nc_params *p, void *cuda_stream, uint8_t **out, size_t *out_n) {
  if (!m || !out || !out_n || (n_chunks && !chunk_ntok)) return set_err(NC_ERR_INVALID, "null argument");
  *out = nullptr; *out_n = 0;
  nc::stats() = nc::Stats{};
  return guard([&] {
    require_device();
    nc::Params q = nc::validate(p);
    std::vector<uint32_t> ntok(chunk_ntok, chunk_ntok + n_chunks);
    size_t total = 0;
    for (uint32_t c : ntok) total += c;
    nc::check_tokens_device(m, tokens_dev, total, (cudaStream_t)cuda_stream);
    nc::CompressOut co;
    const auto t0 = std::chrono::steady_clock::now();
    nc::compress_device(m, tokens_dev, ntok, q, (cudaStream_t)cuda_stream, co);
    const auto t1 = std::chrono::steady_clock::now();
    std::vector<uint8_t> blob;
    nc::encode_container(q, ntok, co, blob);
    *out = dup_out(blob);
    *out_n = blob.size();
    if (std::getenv("NC_TIMELINE")) {
      const auto t2 = std::chrono::steady_clock::now();
      fprintf(stderr, "host: compress_device %.2f ms, range coder + container %.2f ms\n",
              std::chrono::duration<double, std::milli>(t1 - t0).count(),
              std::chrono::duration<double, std::milli>(t2 - t1).count());
    }
  });
}

}  // extern "C"

namespace {
// the NC05 text path shared by nc_compress and the NC06 text section
void compress_nc05(nc_model *m, const uint8_t *in, size_t n, const nc::Params &q, cudaStream_t s,
                   std::vector<uint8_t> &blob) {
  std::vector<uint32_t> tokens, ntok;
  tokenize_all(m, in, n, effective_chunks(q, 1), tokens, ntok);
  NC_CUDA(cudaSetDevice(m->device));
  uint32_t *tok_d = static_cast<uint32_t *>(nc::dev_alloc(tokens.size() * 4 + 4, s));
  try {
    if (!tokens.empty()) NC_CUDA(cudaMemcpyAsync(tok_d, tokens.data(), tokens.size() * 4, cudaMemcpyHostToDevice, s));
    nc::CompressOut co;
    nc::compress_device(m, tok_d, ntok, q, s, co);
    nc::dev_free(tok_d, s);
    tok_d = nullptr;
    nc::encode_container(q, ntok, co, blob);
  } catch (...) {
    if (tok_d) nc::dev_free(tok_d, s);
    throw;
  }
}
void decompress_nc05(nc_model *m, const uint8_t *in, size_t n, nc::Params q, cudaStream_t s, std::string &text) {
  nc::Nc05View view = nc::read_nc05(in, n);
  q.flags = view.flags;
  q.tau_milli = view.tau_milli;
  q.inv_tau = 1000.0 / view.tau_milli;
  std::vector<std::vector<uint32_t>> toks;
  nc::decompress_device(m, in, view, q, s, toks);
  for (auto &t : toks) m->tok.decode(t.data(), t.size(), text);
}
}  // namespace

extern "C" {

nc_status nc_compress(nc_model *m, const uint8_t *in, size_t n, const nc_params *p, void *cuda_stream,
                      uint8_t **out, size_t *out_n) {
  if (!m || (!in && n) || !out || !out_n) return set_err(NC_ERR_INVALID, "null argument");
  *out = nullptr; *out_n = 0;
  nc::stats() = nc::Stats{};
  return guard([&] {
    require_device();
    nc::Params q = nc::validate(p);
    std::vector<uint8_t> blob;
    compress_nc05(m, in, n, q, (cudaStream_t)cuda_stream, blob);
    *out = dup_out(blob);
    *out_n = blob.size();
  });
}

nc_status nc_decompress(nc_model *m, const uint8_t *in, size_t n, const nc_params *p, void *cuda_stream,
                        uint8_t **out, size_t *out_n) {
  if (!m || (!in && n) || !out || !out_n) return set_err(NC_ERR_INVALID, "null argument");
  *out = nullptr; *out_n = 0;
  nc::stats() = nc::Stats{};
  return guard([&] {
    require_device();
    nc::Params q = nc::validate(p);
    std::string text;
    decompress_nc05(m, in, n, q, (cudaStream_t)cuda_stream, text);
    std::vector<uint8_t> o(text.begin(), text.end());
    *out = dup_out(o);
    *out_n = o.size();
  });
}

nc_status nc_compress_file(nc_model *m, const uint8_t *in, size_t n, const nc_params *p, void *cuda_stream,
                           uint8_t **out, size_t *out_n) {
  if (!m || (!in && n) || !out || !out_n) return set_err(NC_ERR_INVALID, "null argument");
  *out = nullptr; *out_n = 0;
  nc::stats() = nc::Stats{};
  return guard([&] {
    require_device();
    nc::Params q = nc::validate(p);
    std::vector<nc::Region> regs = nc::segment(in, n);
    if (regs.size() > 0xFFFF) regs.assign(1, nc::Region{nc::kBinary, (uint64_t)n});   // D34
    std::vector<uint8_t> text, binary;
    size_t off = 0;
    for (const nc::Region &r : regs) {
      (r.kind == nc::kText ? text : binary).insert((r.kind == nc::kText ? text : binary).end(), in + off,
                                                   in + off + r.len);
      off += r.len;
    }
    // the binary blob codec (host) runs beside the GPU text path
    std::vector<uint8_t> payload;
    uint8_t method = nc::kRaw;
    std::string err;
    std::thread codec([&] {
      try {
        method = nc::blob_encode(binary.data(), binary.size(), payload);
      } catch (std::exception &e) { err = e.what(); }
    });
    std::vector<uint8_t> t05;
    try {
      compress_nc05(m, text.data(), text.size(), q, (cudaStream_t)cuda_stream, t05);
    } catch (...) {
      codec.join();
      throw;
    }
    codec.join();
    if (!err.empty()) nc::fail(NC_ERR_BACKEND, err);
    std::vector<uint8_t> blob;
    nc::write_nc06((uint8_t)q.flags, (uint16_t)q.tau_milli, regs, method, payload, t05.data(), t05.size(), blob);
    *out = dup_out(blob);
    *out_n = blob.size();
  });
}

nc_status nc_decompress_file(nc_model *m, const uint8_t *in, size_t n, const nc_params *p, void *cuda_stream,
                             uint8_t **out, size_t *out_n) {
  if (!m || (!in && n) || !out || !out_n) return set_err(NC_ERR_INVALID, "null argument");
  *out = nullptr; *out_n = 0;
  nc::stats() = nc::Stats{};
  return guard([&] {
    require_device();
    nc::Params q = nc::validate(p);
    if (n >= 4 && std::memcmp(in, "NC05", 4) == 0) {   // a plain text container
      std::string text;
      decompress_nc05(m, in, n, q, (cudaStream_t)cuda_stream, text);
      std::vector<uint8_t> o(text.begin(), text.end());
      *out = dup_out(o);
      *out_n = o.size();
      return;
    }
    nc::Nc06View v = nc::read_nc06(in, n);
    std::vector<uint8_t> t05{'N', 'C', '0', '5', v.flags, (uint8_t)(v.tau_milli & 255), (uint8_t)(v.tau_milli >> 8)};
    t05.insert(t05.end(), in + v.text_off, in + n);
    std::vector<uint8_t> binary;
    std::string err;
    std::thread codec([&] {
      try {
        nc::blob_decode(v.method, in + v.payload_off, v.payload_len, v.bin_len, binary);
      } catch (nc::Error &e) { err = e.what(); }
        catch (std::exception &e) { err = e.what(); }
    });
    std::string text;
    try {
      decompress_nc05(m, t05.data(), t05.size(), q, (cudaStream_t)cuda_stream, text);
    } catch (...) {
      codec.join();
      throw;
    }
    codec.join();
    if (!err.empty()) nc::fail(NC_ERR_INTEGRITY, err);
    if (text.size() != v.text_len) nc::fail(NC_ERR_INTEGRITY, "NC06 text entries do not match the decoded text");
    std::vector<uint8_t> o;
    o.reserve(v.text_len + v.bin_len);
    size_t ti = 0, bi = 0;
    for (const nc::Region &r : v.regs) {
      if (r.kind == nc::kText) {
        o.insert(o.end(), text.begin() + ti, text.begin() + ti + r.len);
        ti += r.len;
      } else {
        o.insert(o.end(), binary.begin() + bi, binary.begin() + bi + r.len);
        bi += r.len;
      }
    }
    *out = dup_out(o);
    *out_n = o.size();
  });
}

nc_status nc_host_segment(const uint8_t *in, size_t n, uint8_t **kinds, uint64_t **lens, size_t *n_regions) {
  if ((!in && n) || !kinds || !lens || !n_regions) return set_err(NC_ERR_INVALID, "null argument");
  *kinds = nullptr; *lens = nullptr; *n_regions = 0;
  return guard([&] {
    std::vector<nc::Region> r = nc::segment(in, n);
    std::vector<uint8_t> k;
    std::vector<uint64_t> l;
    for (auto &x : r) { k.push_back(x.kind); l.push_back(x.len); }
    *kinds = dup_out(k);
    *lens = dup_out(l);
    *n_regions = r.size();
  });
}

nc_status nc_host_blob_encode(const uint8_t *in, size_t n, uint8_t *method, uint8_t **out, size_t *out_n) {
  if ((!in && n) || !method || !out || !out_n) return set_err(NC_ERR_INVALID, "null argument");
  *out = nullptr; *out_n = 0;
  return guard([&] {
    std::vector<uint8_t> o;
    *method = nc::blob_encode(in, n, o);
    *out = dup_out(o);
    *out_n = o.size();
  });
}

nc_status nc_host_blob_decode(uint8_t method, const uint8_t *in, size_t n, size_t expect_n, uint8_t **out,
                              size_t *out_n) {
  if ((!in && n) || !out || !out_n) return set_err(NC_ERR_INVALID, "null argument");
  *out = nullptr; *out_n = 0;
  return guard([&] {
    std::vector<uint8_t> o;
    nc::blob_decode(method, in, n, expect_n, o);
    *out = dup_out(o);
    *out_n = o.size();
  });
}

nc_status nc_last_stats(uint64_t *kernel_launches, double *walk_ms, double *forward_ms, double *head_ms) {
  const nc::Stats &s = nc::stats();
  if (kernel_launches) *kernel_launches = s.launches;
  if (walk_ms) *walk_ms = s.walk_ms;
  if (forward_ms) *forward_ms = s.forward_ms;
  if (head_ms) *head_ms = s.head_ms;
  return NC_OK;
}

nc_status nc_debug_set_splitk(int mode) {
  return guard([&] { nc::set_splitk_mode(mode); });
}

nc_status nc_set_profiling(int on) {
  return guard([&] {
    nc::prof().reset();
    nc::prof().on = on != 0;
  });
}

nc_status nc_profile(int cls, uint64_t *launches, double *ms, double *work, const char **name) {
  static const char *names[nc::K_NCLASS] = {"embed", "rms", "gemm_qkv", "attention", "gemm_o",
                                            "gemm_gateup", "gemm_down", "gemm_head", "walk", "misc"};
  if (cls < 0 || cls >= nc::K_NCLASS) return set_err(NC_ERR_INVALID, "bad class");
  if (launches) *launches = nc::prof().n[cls];
  if (ms) *ms = nc::prof().ms[cls];
  if (work) *work = nc::prof().work[cls];
  if (name) *name = names[cls];
  return NC_OK;
}

void nc_free(void *p) { std::free(p); }
const char *nc_last_error(void) { return g_err.c_str(); }

// ---------------------------------------------------------------- debug ---
nc_status nc_debug_quantize(const float *p, uint32_t V, uint32_t cdf_bits, uint32_t *counts_out) {
  if (!p || !counts_out || V == 0) return set_err(NC_ERR_INVALID, "null argument");
  return guard([&] {
    require_device();
    if (!(cdf_bits == 16 || cdf_bits == 24) || V >= (1u << cdf_bits)) nc::fail(NC_ERR_INVALID, "bad cdf_bits / V");
    float *pd;
    uint32_t *cd;
    NC_CUDA(cudaMalloc(&pd, V * 4));
    NC_CUDA(cudaMalloc(&cd, V * 4));
    NC_CUDA(cudaMemcpy(pd, p, V * 4, cudaMemcpyHostToDevice));
    nc::launch_quantize_debug(pd, V, cdf_bits, cd, nullptr);
    cudaError_t e = cudaMemcpy(counts_out, cd, V * 4, cudaMemcpyDeviceToHost);
    cudaFree(pd);
    cudaFree(cd);
    NC_CUDA(e);
    for (uint32_t v = 0; v < V; ++v)
      if (counts_out[v] == 0) nc::fail(NC_ERR_INTEGRITY, "negative residual exceeds the argmax count (D6)");
  });
}

nc_status nc_debug_walk(int device, const float *logits, const uint32_t *tok, uint32_t n_tok, uint32_t V,
                        const nc_params *p, uint32_t *cum, uint32_t *freq, float *p_true) {
  if ((!logits || !tok || !cum || !freq || !p_true) && n_tok) return set_err(NC_ERR_INVALID, "null argument");
  return guard([&] {
    require_device();
    nc::Params q = nc::validate(p);
    nc::debug_walk(device, logits, 0, tok, n_tok, V, q, cum, freq, p_true);
  });
}

nc_status nc_debug_walk_dump(int device, const float *logits, uint32_t n_logit_rows, const uint32_t *tok,
                             uint32_t n_tok, uint32_t V,
                             const nc_params *p, uint32_t *cum, uint32_t *freq, float *p_true, float *pt_true,
                             const uint32_t *rows, uint32_t n_rows, float *pt_rows, float *p_rows,
                             uint32_t *counts_rows) {
  if ((!logits || !tok || !cum || !freq || !p_true || !pt_true) && n_tok) return set_err(NC_ERR_INVALID, "null argument");
  if (n_rows && (!rows || !pt_rows || !p_rows || !counts_rows)) return set_err(NC_ERR_INVALID, "null dump argument");
  return guard([&] {
    require_device();
    nc::Params q = nc::validate(p);
    nc::debug_walk(device, logits, n_logit_rows, tok, n_tok, V, q, cum, freq, p_true, pt_true, rows, n_rows, pt_rows,
                   p_rows,
                   counts_rows);
  });
}

nc_status nc_debug_forward(nc_model *m, const uint32_t *x, uint32_t rows, const nc_params *p, int mode,
                           float *logits_out) {
  if (!m || (!x && rows) || (!logits_out && rows)) return set_err(NC_ERR_INVALID, "null argument");
  return guard([&] {
    require_device();
    nc::Params q = nc::validate(p);
    nc::debug_forward(m, x, rows, q, mode, logits_out);
  });
}

nc_status nc_debug_gemm(int device, const float *A, const float *B, uint32_t M, uint32_t N, uint32_t K, int mode,
                        float *out) {
  if (!A || !B || !out || !M || !N || !K) return set_err(NC_ERR_INVALID, "null argument");
  return guard([&] {
    require_device();
    nc::debug_gemm(device, A, B, M, N, K, mode, out);
  });
}

nc_status nc_debug_attention(int device, const float *q, const float *k, const float *v, uint32_t n, uint32_t H,
                             uint32_t KV, uint32_t window, uint32_t slide, int mode, float *o) {
  if (!q || !k || !v || !o || !H || !KV || H % KV) return set_err(NC_ERR_INVALID, "bad argument");
  return guard([&] {
    require_device();
    if (window % 128 || slide % 128 || slide >= window) nc::fail(NC_ERR_INVALID, "window/slide");
    nc::debug_attention(device, q, k, v, n, H, KV, window, slide, mode, o);
  });
}

// ----------------------------------------------------------- host pieces ---
nc_status nc_host_split(const uint8_t *in, size_t n, uint32_t n_chunks, uint64_t *cuts, uint32_t *n_cuts) {
  if ((!in && n) || !cuts || !n_cuts) return set_err(NC_ERR_INVALID, "null argument");
  return guard([&] {
    auto c = nc::split_chunks(in, n, n_chunks ? n_chunks : 1);
    std::memcpy(cuts, c.data(), c.size() * 8);
    *n_cuts = (uint32_t)c.size();
  });
}

nc_status nc_host_wnc_encode(const uint32_t *cum, const uint32_t *freq, size_t n, uint32_t cdf_bits, uint8_t **stream,
                             size_t *stream_n, uint64_t *bit_count) {
  if ((!cum || !freq) && n) return set_err(NC_ERR_INVALID, "null argument");
  if (!stream || !stream_n || !bit_count) return set_err(NC_ERR_INVALID, "null argument");
  *stream = nullptr; *stream_n = 0;
  return guard([&] {
    nc::WncEncoder enc;
    for (size_t i = 0; i < n; ++i) {
      if ((uint64_t)cum[i] + freq[i] > (1ull << cdf_bits)) nc::fail(NC_ERR_INVALID, "interval beyond T");
      enc.encode(cum[i], freq[i], cdf_bits);
    }
    std::vector<uint8_t> s;
    enc.finish(s, *bit_count);
    *stream = dup_out(s);
    *stream_n = s.size();
  });
}

nc_status nc_host_ans_encode(const uint32_t *cum, const uint32_t *freq, size_t n, uint32_t cdf_bits, uint8_t **stream,
                             size_t *stream_n, uint64_t *bit_count) {
  if ((!cum || !freq) && n) return set_err(NC_ERR_INVALID, "null argument");
  if (!stream || !stream_n || !bit_count) return set_err(NC_ERR_INVALID, "null argument");
  *stream = nullptr; *stream_n = 0;
  return guard([&] {
    if (cdf_bits < 1 || cdf_bits > 31) nc::fail(NC_ERR_INVALID, "cdf_bits");
    for (size_t i = 0; i < n; ++i)
      if ((uint64_t)cum[i] + freq[i] > (1ull << cdf_bits)) nc::fail(NC_ERR_INVALID, "interval beyond T");
    std::vector<uint8_t> s;
    nc::ans_encode(cum, freq, n, cdf_bits, s, *bit_count);
    *stream = dup_out(s);
    *stream_n = s.size();
  });
}

nc_status nc_host_tokenize_vocab(const uint8_t *vocab_blob, const uint32_t *vocab_len, uint32_t V, uint32_t n_special,
                                 const uint8_t *in, size_t n, uint32_t **tokens, size_t *n_tokens) {
  if (!vocab_blob || !vocab_len || !tokens || !n_tokens || (!in && n)) return set_err(NC_ERR_INVALID, "null argument");
  *tokens = nullptr; *n_tokens = 0;
  return guard([&] {
    std::vector<std::string> vocab(V);
    size_t off = 0;
    for (uint32_t i = 0; i < V; ++i) {
      vocab[i].assign(reinterpret_cast<const char *>(vocab_blob) + off, vocab_len[i]);
      off += vocab_len[i];
    }
    nc::Tokenizer tk;
    tk.build(vocab, n_special);
    std::vector<uint32_t> t;
    tk.encode(in, n, t);
    *tokens = dup_out(t);
    *n_tokens = t.size();
  });
}

}  // extern "C"
