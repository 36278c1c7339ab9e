// Per-chunk walk state and launchers for the vocab-row CDF kernel and the
// N-gram precompute kernel.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace nc {

constexpr int kSlots = 64;            // N-gram continuation cap
constexpr int kMaxOrders = 4;         // context tables k = 1..4 (D18)
constexpr int kMaxSparse = kMaxOrders * kSlots;

struct NgRecord {                     // one context's continuation table
  uint32_t n;                         // context occurrences (never decremented, D19)
  uint32_t nslot;                     // used slots (<= 64)
  uint32_t tok[kSlots];
  uint32_t cnt[kSlots];
};

// N-gram prediction of one token in closed form:
//   p_ng(v) = a0f * (c(v) + 1) + add[v]  (add = sum_k a_k cnt_k(v), merged in order k = 1..4)
struct __align__(16) NgTok {
  uint32_t n;                         // number of distinct sparse ids
  float a0f;                          // a0 / (N + V) as f32, N = tokens seen = i
  uint32_t pad[2];
  uint32_t tok[kMaxSparse];
  float add[kMaxSparse];
};

struct WalkState {                    // per chunk, device resident
  double lw[2];                       // mixer: lw[0] = log-odds d = lw_llm - lw_ng (f64), lw[1] = 0
  uint32_t i;                         // tokens walked so far (walk kernel)
  uint32_t ng_i;                      // tokens seen by the N-gram (precompute / inline)
  uint32_t hist[4];                   // last 4 tokens (oldest first), N-gram side
  uint32_t nrec[kMaxOrders];          // records in use per order
  uint32_t err;                       // nonzero = integrity failure
  float wl, wn;                       // current mixer weights (softmax of lw) as f32
  uint32_t pend;                      // decoder: pending E3 (underflow) steps, as the encoder counts them
  // device decoder: WNC (D27) uses low, high, value, bitpos; rANS (D39) keeps its state x in
  // value and its read position (bits, a multiple of 32) in bitpos
  unsigned long long low, high, value, bitpos;
};

struct WalkArgs {
  // per launch: entry e handles chunk chunk_of[e], rows [row0[e], row0[e]+count[e]) of logits,
  // i.e. tokens st.i .. st.i + count - 1 of that chunk
  const int32_t *chunk_of, *row0, *count;
  int n_entries;
  const float *logits; int64_t ldl;
  // encode inputs / outputs, indexed by tok_off[c] + i
  const uint32_t *tokens; const int64_t *tok_off;
  uint32_t *out_cum, *out_freq; float *out_p;
  float *out_pt;                      // test only (may be NULL): p~(t) of every token, before mixing
  // test only: full vectors of chunk dump_chunk at the sorted token indices dump_rows[0, n_dump):
  // dump_pt / dump_p = p~ and the quantized p (fp32), dump_c = the walk's final counts (after the
  // residual), each [n_dump][V]
  const uint32_t *dump_rows; uint32_t n_dump; int dump_chunk;
  float *dump_pt, *dump_p; uint32_t *dump_c;
  NgTok *ng_pre;                      // encode: precomputed N-gram predictions, ring of ng_ring per chunk:
  uint32_t ng_ring;                   //   token i of chunk c at ng_pre[c * ng_ring + i % ng_ring]
  float *ng_spadd;                    // precompute scratch (separate from the walk's spadd)
  // decode
  const uint8_t *streams; const int64_t *stream_off; const uint64_t *stream_bits;
  uint32_t *out_tok; uint32_t *next_x;
  // state
  WalkState *st; double *b; uint32_t *cu; float *spadd;
  unsigned long long *ng_keys; uint32_t *ng_vals; NgRecord *ng_recs;
  uint32_t hcap, rcap;                // per (chunk, order) hash slots (pow2) / record pool
  // params
  uint32_t V, cdf_bits, warmup, flags, orders, cap;
  float inv_tau; double alpha, eta;
  int mode;                           // 0 encode, 1 decode
  uint32_t coder;                     // decode: NC_CODER_WNC (0) or NC_CODER_ANS (1)
  int n_chunks_total;                 // chunks of the container (or shard): with V, fixes the cluster size
};

void launch_walk(const WalkArgs &a, cudaStream_t s);
int walk_ctas_per_chunk(uint32_t V, int n_chunks);   // CTAs (one cluster) per chunk in the walk
void walk_timing_report();            // diagnostics build (-DNC_WALK_TIMING): phase cycles -> stderr
// encode only: N-gram predictions for the entries' tokens (one warp per chunk)
void launch_ngram_precompute(const WalkArgs &a, cudaStream_t s);
void launch_walk_init(WalkState *st, int n_chunks, cudaStream_t s);
void launch_quantize_debug(const float *p, uint32_t V, uint32_t cdf_bits, uint32_t *counts, cudaStream_t s);

}  // namespace nc
