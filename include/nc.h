/*
 * nc.h -- C ABI of libnc.so, the B200-native hot path of the Nacrith
 * LLM + arithmetic-coding text compressor (arXiv 2602.19626, PAPER.md).
 *
 * The boundary follows the paper's problem statement: "REQUIRE text string s
 * ... RETURN ArithEncoder.finish()" (alg:compress) and its mirror,
 * decompression, packaged in the NC05 container.
 * SURVEY.md §8(b) lists these entry points.  P:<n> = PAPER.md line n,
 * S:<n> = SPEC.md line n, Dn = SURVEY.md §8(c) reading n.
 *
 * Conventions (all entry points):
 *   - Every pointer argument is a HOST pointer unless its name ends in _dev.
 *   - Inputs are borrowed for the duration of the call; nothing is retained.
 *   - Buffers returned through uint8_t** / uint32_t** are malloc'ed by the
 *     library; release them with nc_free().  On any non-OK status no output
 *     buffer is returned (the out pointers are set to NULL / 0).
 *   - Errors: every call returns nc_status; nc_last_error() returns a
 *     thread-local message describing the last non-OK status of this thread.
 *   - Device memory comes from the allocator hook (nc_set_allocator) when one
 *     is set.  The default is the library's own pool over cudaMalloc: blocks are
 *     cached per (device, size) after a call returns and reused by later calls
 *     (a block may be up to twice the requested size); the pool grows and never
 *     returns memory to the driver while the process runs.
 *   - A model is bound to one CUDA device and is not safe for concurrent calls;
 *     use one model per GPU and one process per GPU for multi-GPU runs.
 *   - There is no CPU fallback: without a usable CUDA device every compute
 *     entry point returns NC_ERR_BACKEND.
 */
#ifndef NC_H_
#define NC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nc_model nc_model; /* device weights + vocabulary for ONE device */
typedef struct nc_comm nc_comm;   /* NCCL communicator (NULL = single GPU)      */

typedef enum {
  NC_OK = 0,
  NC_ERR_FORMAT = 1,    /* malformed container / weight file     */
  NC_ERR_BACKEND = 2,   /* CUDA / NCCL failure, no device (S:577 exit 2)      */
  NC_ERR_INVALID = 3,   /* bad argument or parameter                          */
  NC_ERR_NOMEM = 4,     /* host or device allocation failed                   */
  NC_ERR_TRUNCATED = 5, /* container shorter than its tables say              */
  NC_ERR_INTEGRITY = 6  /* decoded bit_count / token_count mismatch, or a
                           quantizer residual that would drop a count below 1 */
} nc_status;

/* Feature flags (NC05 flags byte). */
#define NC_FLAG_NGRAM 1u /* bit0: N-gram + mixer            */
#define NC_FLAG_HEAD 2u  /* bit1: adaptive log-space bias head */
#define NC_FLAG_SKIP 4u  /* bit2: confidence-based LLM skip (P:452-469,
                            alg:compress lines 5-6): after the warmup, a
                            token with H(p_ng) < 1.5 bits is coded with
                            p = p_ng.  Needs NC_FLAG_NGRAM (ignored
                            without it).  The forward still runs (its K/V
                            are retained) and every model updates on
                            every token (alg:compress line 12; DESIGN D32) */

typedef struct {
  uint32_t cdf_bits;     /* 24 (default) or 16; T = 2^cdf_bits */
  uint32_t flags;        /* NC_FLAG_* ; default NGRAM|HEAD                    */
  float temperature;     /* tau > 0; stored as u16 round(tau*1000);
                            the effective value is tau_milli/1000 (D29)      */
  uint32_t window;       /* L, default 2048; multiple of 128          */
  uint32_t slide;        /* C, default 512; multiple of 128, C < L    */
  uint32_t warmup;       /* W, default 100                            */
  double eta;            /* mixer learning rate, default 1.0 (D24)            */
  double alpha;          /* bias-head learning rate, default 1e-3     */
  uint32_t ngram_orders; /* context tables k=1..ngram_orders, default 4 (D18) */
  uint32_t ngram_cap;    /* contexts per order before freezing, 500000 (D22) */
  uint32_t n_chunks;     /* total chunks; 0 = world*chunks_per_gpu    */
  uint32_t chunks_per_gpu; /* used when n_chunks == 0, default 64             */
  uint32_t max_slab_rows;  /* forward slab size in rows over all chunks
                              (default 32768); 0 = default                    */
  uint32_t debug_dump;   /* test only: nonzero -> keep per-token p(t) values  */
  uint32_t window_variant; /* NC_WINDOW_* bits, default 0 = retained KV with
                              L_max = L (D9-D10, what the paper ran) */
  uint32_t coder;        /* NC_CODER_WNC (default) or NC_CODER_ANS; like L and C it is not
                            stored in the container: the decoder must pass the same value */
} nc_params;

/* Entropy coder of the chunk streams.  NC_CODER_WNC: the paper's 32-bit arithmetic coder
 * (D7-D8).  NC_CODER_ANS: rANS, the paper's future-work replacement (
 * reading D39): 64-bit state in [2^31, 2^64), 32-bit renormalisation words, symbols coded in
 * reverse on the host, decoded forward on the device; bit_count = 32 x words; a stream whose
 * decoder does not end in the start state 2^31 with every word consumed is NC_ERR_INTEGRITY. */
#define NC_CODER_WNC 0u
#define NC_CODER_ANS 1u

/* Window variants, nc_params.window_variant.  Not stored in the
 * container: the decoder must pass the same value (a mismatch fails the integrity checks). */
#define NC_WINDOW_REFRESH 1u /* refresh semantics: on every slide the surviving window is
                                re-evaluated from scratch (the naive re-evaluation of
                                P:489-492), so row j's logits are those of a fresh
                                evaluation of x[w(j) .. j] (S:361's window equivalence);
                                ~L/C times the prefill FLOPs of retained KV */
#define NC_WINDOW_LMAX_M1 2u /* L_max = L - 1 (D10's other reading: the cache slides when
                                full, so the context is at most L - 1 tokens):
                                w(j) = C ceil(max(0, j + 1 - L_max) / C) */

void nc_params_default(nc_params *p);

/* Device allocator hook (e.g. the torch caching allocator).  alloc(bytes, ctx)
 * returns device memory on the current device or NULL; free(ptr, ctx).  Pass
 * NULLs to restore the default.  Not thread-safe against running calls. */
nc_status nc_set_allocator(void *(*alloc)(size_t bytes, void *ctx),
                           void (*free_fn)(void *ptr, void *ctx), void *ctx);

/* Load an NCW1 weight file (format: synth/weights.py) onto CUDA device
 * `device`: config, fp32 tensors (tied head, D16) and the vocabulary used by
 * the tokenizer (D30).  Weights are re-laid out for the kernels on load
 * (RMSNorm gains folded into the following projection). */
nc_status nc_model_load(const char *path, int device, nc_model **out);
void nc_model_free(nc_model *m);

/* Load an HF-format SmolLM2 checkpoint directory:
 * model_dir/config.json (LlamaConfig: hidden_size, num_hidden_layers, num_attention_heads,
 * num_key_value_heads, head_dim, intermediate_size, vocab_size, rms_norm_eps, rope_theta /
 * rope_parameters, bos_token_id; tie_word_embeddings must be true, default RoPE only),
 * model_dir/model.safetensors (HF Llama tensor names, F32 / F16 / BF16, converted to fp32)
 * and model_dir/tokenizer.json (byte-level BPE behind ByteLevel or Digits + ByteLevel
 * pre-tokenization; the model then tokenizes with it instead of the greedy synthetic-vocab
 * matcher, D35-D36).  Errors: NC_ERR_INVALID for unsupported configurations, NC_ERR_FORMAT
 * for malformed files. */
nc_status nc_model_load_hf(const char *model_dir, int device, nc_model **out);
/* vocab size, n_layers, d_model of a loaded model (any may be NULL). */
nc_status nc_model_info(const nc_model *m, uint32_t *vocab, uint32_t *n_layers,
                        uint32_t *d_model);

/* Compress `n` bytes at `in` (host) into a full NC05 container:
 * split into params->n_chunks chunks at newlines (D28), tokenize
 * each (D30), then for every chunk run the teacher-forced windowed forward
 * (eq:lm, P:482-502 retained-KV window, D9-D10) and the per-token
 * bias-head -> softmax -> N-gram mix -> floors -> CDF quantize walk
 * (P:316-450), and arithmetic-code the true tokens.
 * cuda_stream: a cudaStream_t (NULL = the legacy default stream). */
nc_status nc_compress(nc_model *m, const uint8_t *in, size_t n, const nc_params *p,
                      void *cuda_stream, uint8_t **out, size_t *out_n);

/* Inverse of nc_compress.  The flags byte and temperature come from
 * the container; cdf_bits, window, slide, warmup, eta, alpha, ngram_orders and
 * ngram_cap must equal the compress-time params (they are not stored, §8(b)).
 * A mismatch shows up as NC_ERR_INTEGRITY (bit_count check).  Decoding runs on
 * the device one token per chunk per step with the same kernels as compression
 * (bit-identical logits, D15) and a device-side WNC decoder (D27). */
nc_status nc_decompress(nc_model *m, const uint8_t *in, size_t n, const nc_params *p,
                        void *cuda_stream, uint8_t **out, size_t *out_n);

/* NC06 hybrid binary format.
 * nc_compress_file: any bytes -> NC06.  The input is segmented into alternating text and
 * binary regions by the paper's four rules (printable ASCII + tab/LF/CR is text-like;
 * text runs < 64 B demoted; binary gaps <= 8 B between text bridged; binary chunks < 64 B
 * next to text absorbed; DESIGN D33); the binary regions, concatenated, are compressed
 * with LZMA (>= 4 KB) or DEFLATE, or stored raw if neither is smaller (D34);
 * the text regions, concatenated, take the nc_compress path (params->n_chunks chunks).
 * Layout (little-endian): "NC06" | version u8 = 1 | flags u8 | tau_milli u16 |
 * entry_count u16 | entry_count x {kind u8 (0 binary, 1 text), length u32} |
 * method u8 (0 raw, 1 DEFLATE, 2 LZMA) | blob_length u32 | blob | the NC05 text section
 * from its chunk_count field on.  Regions larger than 4 GB are NC_ERR_INVALID.
 * nc_decompress_file: NC06 (or a plain NC05 container) -> the original bytes; the same
 * params rules as nc_decompress.  Errors: NC_ERR_FORMAT / NC_ERR_TRUNCATED for a malformed
 * container, NC_ERR_INTEGRITY if a section does not decode to its entry lengths. */
nc_status nc_compress_file(nc_model *m, const uint8_t *in, size_t n, const nc_params *p,
                           void *cuda_stream, uint8_t **out, size_t *out_n);
nc_status nc_decompress_file(nc_model *m, const uint8_t *in, size_t n, const nc_params *p,
                             void *cuda_stream, uint8_t **out, size_t *out_n);

/* Split + tokenize only (host; D28 + D30).  tokens: all chunks' token ids
 * concatenated; chunk_ntok[i]: token count of chunk i (n_chunks_out entries). */
nc_status nc_tokenize(const nc_model *m, const uint8_t *in, size_t n, uint32_t n_chunks,
                      uint32_t **tokens, size_t *n_tokens, uint32_t **chunk_ntok,
                      uint32_t *n_chunks_out);

/* The compress hot path on pre-tokenized input.  tokens_dev: DEVICE pointer to
 * the concatenated token ids of n_chunks chunks, chunk_ntok (host) their
 * counts.  Produces the NC05 container (host).  This is what bench.py times as
 * the device-resident "value" (the tokens are already in HBM). */
nc_status nc_compress_tokens(nc_model *m, const uint32_t *tokens_dev, const uint32_t *chunk_ntok,
                             uint32_t n_chunks, const nc_params *p, void *cuda_stream,
                             uint8_t **out, size_t *out_n);

/* Multi-GPU: every rank passes the FULL input and the same
 * params; rank r compresses chunks [r*k, (r+1)*k) (k = ceil(chunks/world)) and
 * returns its byte range [part_offset, part_offset + part_n) of the final
 * container of total_n bytes.  One NCCL allgather of the chunk table.
 * Concatenating the parts in rank order == nc_compress with the same n_chunks. */
nc_status nc_comm_unique_id(uint8_t id[128]);
nc_status nc_comm_init(int rank, int world, const uint8_t id[128], int device, nc_comm **out);
void nc_comm_free(nc_comm *c);
nc_status nc_compress_shard(nc_model *m, nc_comm *c, const uint8_t *in, size_t n,
                            const nc_params *p, void *cuda_stream, uint8_t **part,
                            size_t *part_n, uint64_t *part_offset, uint64_t *total_n);
nc_status nc_decompress_shard(nc_model *m, nc_comm *c, const uint8_t *in, size_t n,
                              const nc_params *p, void *cuda_stream, uint8_t **part,
                              size_t *part_n, uint64_t *part_offset, uint64_t *total_n);

void nc_free(void *p);             /* frees any library-returned buffer */
const char *nc_last_error(void);   /* thread-local; never NULL           */

/* Number of kernels the library launched during the last compute call on this
 * thread, and the device time (ms, CUDA events) of its dominant kernel class. */
nc_status nc_last_stats(uint64_t *kernel_launches, double *walk_ms, double *forward_ms,
                        double *head_ms);

/* Per-kernel-class device timing (CUDA events around every launch, on the
 * launching stream).  nc_set_profiling(1) enables it and clears the totals;
 * classes: 0 embed, 1 rms, 2 gemm_qkv, 3 attention, 4 gemm_o, 5 gemm_gateup,
 * 6 gemm_down, 7 gemm_head, 8 walk, 9 misc.  work = algorithmic FLOPs (GEMMs,
 * attention) or bytes (embed, rms, walk: 4*V logits bytes per token, §8(d))
 * summed over the launches since the last reset. */
nc_status nc_set_profiling(int on);
nc_status nc_profile(int cls, uint64_t *launches, double *ms, double *work, const char **name);

/* ---- test-only entry points (no side effects on models) ------------------ */

/* Split-K policy of the tcgen05 GEMM (process-wide): 1 = automatic (default:
 * split the k loop across CTAs when the tile grid would leave most SMs idle,
 * e.g. decode steps), 0 = never.  Both give bit-identical results (the span
 * partials are summed in the same order, D15); tests compare the two. */
nc_status nc_debug_set_splitk(int mode);

/* GPU quantizer on caller floats (host array p[V]): counts_out[V] (host) per
 * c_i = max(1, floor(p_i (T-V))) + residual to argmax (D4-D6).
 * "Integer CDFs bit-exact given identical float inputs" is checked with it. */
nc_status nc_debug_quantize(const float *p, uint32_t V, uint32_t cdf_bits, uint32_t *counts_out);

/* Run the per-token walk kernel (bias head, softmax, N-gram mix, quantize,
 * updates) on caller logits (host, n_tok x V fp32, row j predicts tok[j]) for
 * ONE chunk, on `device`.  Outputs (host, n_tok entries each): cum, freq,
 * p_true = p(t_j) in fp32.  Used to test the walker in isolation. */
nc_status nc_debug_walk(int device, const float *logits, const uint32_t *tok, uint32_t n_tok,
                        uint32_t V, const nc_params *p, uint32_t *cum, uint32_t *freq,
                        float *p_true);

/* nc_debug_walk plus the walk's internals, for the parity tests of SURVEY §8(d)
 * ("probability-parity sampling"):
 *   pt_true[n_tok] (host): p~(t_j), the bias-head softmax of the true token BEFORE the
 *     N-gram mix, for every row;
 *   rows[n_rows] (host, strictly ascending, each < n_tok): rows whose full vectors are
 *     dumped; for the k-th of them, at offset k*V of each (host) array:
 *       pt_rows = p~ (fp32), p_rows = the quantized distribution p (fp32, mixed after the
 *       warmup), counts_rows = the walk's integer counts c (after the
 *       residual is added to the argmax, D4-D6) -- what the coder used for that row.
 * n_rows = 0 dumps nothing (rows / pt_rows / p_rows / counts_rows may then be NULL).
 * n_logit_rows: logits holds n_logit_rows x V floats and token j uses row j % n_logit_rows
 *   (long sequential walks without an n_tok x V array); 0 = n_tok rows.
 * Errors: NC_ERR_INVALID on null or unsorted arguments; NC_ERR_INTEGRITY as nc_debug_walk. */
nc_status nc_debug_walk_dump(int device, const float *logits, uint32_t n_logit_rows, const uint32_t *tok,
                             uint32_t n_tok, uint32_t V,
                             const nc_params *p, uint32_t *cum, uint32_t *freq, float *p_true, float *pt_true,
                             const uint32_t *rows, uint32_t n_rows, float *pt_rows, float *p_rows,
                             uint32_t *counts_rows);

/* Forward only: logits (host, rows x V fp32) of ONE chunk for LM input ids x
 * (host, x[0] = BOS), window from params.  mode 0 = prefill kernels (slabbed),
 * mode 1 = the decode-step path (one row per step through the KV ring). */
nc_status nc_debug_forward(nc_model *m, const uint32_t *x, uint32_t rows, const nc_params *p,
                           int mode, float *logits_out);

/* One GEMM out[M,N] = A[M,K] B[N,K]^T (host fp32 arrays) through the forward's
 * GEMM kernel: mode 0 = tcgen05 3xTF32 (TMA + TMEM), 1 = SIMT fp32.  K % 32 == 0. */
nc_status nc_debug_gemm(int device, const float *A, const float *B, uint32_t M, uint32_t N, uint32_t K, int mode,
                        float *out);

/* One attention layer for ONE chunk: o[n, H*64] from q[n, H*64] (RoPE already
 * applied), k, v [n, KV*64] (host fp32, positions 0..n-1), block-window mask
 * (window, slide).  mode 0 = tensor-core kernel (3xTF32), 1 = SIMT fp32. */
nc_status nc_debug_attention(int device, const float *q, const float *k, const float *v, uint32_t n, uint32_t H,
                             uint32_t KV, uint32_t window, uint32_t slide, int mode, float *o);

/* Host-side pieces exported for CPU tests of the host logic (no GPU needed). */
nc_status nc_host_split(const uint8_t *in, size_t n, uint32_t n_chunks, uint64_t *cuts,
                        uint32_t *n_cuts); /* cuts: n_chunks+1 capacity, chunk i = [cuts[i], cuts[i+1]) */
nc_status nc_host_wnc_encode(const uint32_t *cum, const uint32_t *freq, size_t n, uint32_t cdf_bits,
                             uint8_t **stream, size_t *stream_n, uint64_t *bit_count);
/* rANS encoding of (cum, freq) pairs in coding order (NC_CODER_ANS's stream of one chunk). */
nc_status nc_host_ans_encode(const uint32_t *cum, const uint32_t *freq, size_t n, uint32_t cdf_bits,
                             uint8_t **stream, size_t *stream_n, uint64_t *bit_count);
nc_status nc_host_tokenize_vocab(const uint8_t *vocab_blob, const uint32_t *vocab_len, uint32_t V,
                                 uint32_t n_special, const uint8_t *in, size_t n,
                                 uint32_t **tokens, size_t *n_tokens);

/* NC06 host pieces (no device needed): the segmentation (kinds[i] 0 binary / 1 text,
 * lens[i] bytes, in input order), and the binary blob codec (method as in NC06;
 * decode checks that the payload decodes to exactly expect_n bytes). */
nc_status nc_host_segment(const uint8_t *in, size_t n, uint8_t **kinds, uint64_t **lens, size_t *n_regions);
nc_status nc_host_blob_encode(const uint8_t *in, size_t n, uint8_t *method, uint8_t **out, size_t *out_n);
nc_status nc_host_blob_decode(uint8_t method, const uint8_t *in, size_t n, size_t expect_n, uint8_t **out,
                              size_t *out_n);

/* The byte-level BPE of a tokenizer.json on host bytes (no device; tests compare it with the
 * HF tokenizers library).  vocab: the model's vocabulary size (ids must be below it). */
nc_status nc_host_bpe_encode(const char *tokenizer_json_path, uint32_t vocab, const uint8_t *in, size_t n,
                             uint32_t **tokens, size_t *n_tokens);

/* SMs (CTAs of one thread-block cluster) the per-token walk holds per chunk at
 * vocabulary size V with n_chunks chunks in the container or shard (host query, no
 * device needed).  bench.py uses it to rank kernels by their share of
 * the GPU's SM-time. */
nc_status nc_host_walk_ctas(uint32_t V, uint32_t n_chunks, uint32_t *ctas);

/* Shard plan pieces of nc_compress_shard (host only; tested with gloo on CPU):
 * the chunk range of a rank, and its part of the final container given the
 * gathered chunk table (3 x u32 per chunk: token_count, bit_count, stream_len). */
nc_status nc_host_shard_range(uint32_t n_chunks, int world, int rank, uint32_t *c0, uint32_t *c1);
nc_status nc_host_shard_part(const uint32_t *table, uint32_t n_chunks, uint8_t flags, uint16_t tau_milli,
                             int world, int rank, const uint8_t *my_streams, size_t my_len, uint8_t **part,
                             size_t *part_n, uint64_t *part_offset, uint64_t *total_n);

#ifdef __cplusplus
}
#endif
#endif /* NC_H_ */
