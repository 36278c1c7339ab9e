// Engine: device model, forward orchestration, compress / decompress drivers.
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "hf.hpp"
#include "kernels.cuh"
#include "nc_internal.hpp"
#include "walk.cuh"

struct nc_model {
  int device = 0;
  nc::Shape s{};
  nc::Tokenizer tok;                                     // greedy longest match over the vocabulary (D30)
  std::unique_ptr<nc::BpeTokenizer> bpe;                 // HF byte-level BPE (nc_model_load_hf, NEXT-2)
  // token ids of a byte string with the model's tokenizer (decode is the vocabulary bytes for both)
  void encode(const uint8_t *in, size_t n, std::vector<uint32_t> &out) const {
    if (bpe) bpe->encode(in, n, out);
    else tok.encode(in, n, out);
  }
  std::vector<std::string> vocab;
  float *E = nullptr;                                    // [V, d] fp32 (embedding gather)
  // tf32 hi/lo planes of every projection for the tcgen05 3xTF32 GEMM (D14); the fp32
  // staging copies (gains folded) are freed once the planes exist
  float *E_head_hi = nullptr, *E_head_lo = nullptr;
  std::vector<float *> wqkv_hi, wqkv_lo, wo_hi, wo_lo, wgu_hi, wgu_lo, wd_hi, wd_lo;
  static constexpr int attn_tile_rows() { return 128; }
  float *rope_cos = nullptr, *rope_sin = nullptr;        // [rope_len, 32]
  int rope_len = 0;
  std::vector<void *> owned;                             // model_free releases them (allocator hook / cudaFree)
  std::vector<bool> owned_hook;                          // owned[i] came from the allocator hook
  cudaStream_t walk_stream = nullptr;                    // the walk runs beside the next slab's forward
  cudaStream_t ng_stream = nullptr;                      // the N-gram precompute runs ahead of the walk
};

namespace nc {

void check_cuda(cudaError_t e, const char *what);
#define NC_CUDA(x) ::nc::check_cuda((x), #x)

// device allocation through the hook
void *dev_alloc(size_t bytes, cudaStream_t s);
void dev_free(void *p, cudaStream_t s);
void set_allocator(void *(*a)(size_t, void *), void (*f)(void *, void *), void *ctx);
// tcgen05 GEMM split-K policy (k_gemm_tc.cu): 1 automatic, 0 never
void set_splitk_mode(int mode);

struct Stats {
  uint64_t launches = 0;
  double walk_ms = 0, forward_ms = 0, head_ms = 0;
};
Stats &stats();  // thread-local

// Optional per-kernel-class CUDA-event profiling (bench.py's live roofline).
enum KClass { K_EMBED = 0, K_RMS, K_QKV, K_ATTN, K_OPROJ, K_GATEUP, K_DOWN, K_HEAD, K_WALK, K_MISC, K_NCLASS };
struct Prof {
  bool on = false;
  struct Rec { int cls; cudaEvent_t a, b; double work; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  uint64_t n[K_NCLASS] = {};
  double ms[K_NCLASS] = {}, work[K_NCLASS] = {};
  cudaEvent_t ev();
  void begin(int cls, double work, cudaStream_t s);   // records start
  void end(cudaStream_t s);                           // records end of the last begin
  void collect();                                     // after a stream sync
  void reset();
};
Prof &prof();

void model_load(nc_model *m, const std::string &path, int device);
void model_load_hf(nc_model *m, const std::string &dir, int device);   // config.json + safetensors + tokenizer.json
void model_setup(nc_model *m, const NcwFile &f, int device);
void model_free(nc_model *m);
void ensure_rope(nc_model *m, int64_t max_pos);

// NC_ERR_INVALID unless every device token id is < V (caller-supplied ids index E, b, cu)
void check_tokens_device(nc_model *m, const uint32_t *tokens_dev, size_t n, cudaStream_t s);
// Compress pre-tokenized chunks whose tokens live in device memory.
struct CompressOut {
  std::vector<uint32_t> cum, freq;   // per token, all chunks concatenated
  std::vector<float> p_true;         // debug_dump only
  std::vector<uint32_t> err;         // per chunk
};
// container_chunks: chunks of the whole container (a shard's are a subset; the walk's cluster
// size depends on it, so compression and decompression must agree), -1 = ntok.size()
void compress_device(nc_model *m, const uint32_t *tokens_dev, const std::vector<uint32_t> &ntok,
                     const Params &p, cudaStream_t s, CompressOut &out, int container_chunks = -1);
// Decode all chunks of a parsed container; returns token ids per chunk.
void decompress_device(nc_model *m, const uint8_t *blob, const Nc05View &view, const Params &p,
                       cudaStream_t s, std::vector<std::vector<uint32_t>> &toks, int container_chunks = -1);
// host encode + container
void encode_container(const Params &p, const std::vector<uint32_t> &ntok, const CompressOut &co,
                      std::vector<uint8_t> &out);
// debug
void debug_gemm(int device, const float *A, const float *B, uint32_t M, uint32_t N, uint32_t K, int mode,
                float *out);
void debug_attention(int device, const float *q, const float *k, const float *v, uint32_t n, uint32_t H, uint32_t KV,
                     uint32_t window, uint32_t slide, int mode, float *o);
void debug_forward(nc_model *m, const uint32_t *x, uint32_t rows, const Params &p, int mode, float *out);
void debug_walk(int device, const float *logits, uint32_t n_logit_rows, const uint32_t *tok, uint32_t n, uint32_t V,
                const Params &p, uint32_t *cum, uint32_t *freq, float *p_true, float *pt_true = nullptr,
                const uint32_t *rows = nullptr, uint32_t n_rows = 0, float *pt_rows = nullptr,
                float *p_rows = nullptr, uint32_t *c_rows = nullptr);

}  // namespace nc
