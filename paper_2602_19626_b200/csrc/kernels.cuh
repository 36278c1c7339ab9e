// Device-side declarations of the hot-path kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace nc {

constexpr int kHeadDim = 64;  // d_h of SmolLM2 (BASELINE.json); kernels are specialised to it

// Per-slab row metadata: LM input id, chunk, absolute position of row (x-space, BOS = 0).
struct RowMeta {
  const uint32_t *x;    // [M]
  const int32_t *chunk; // [M]
  const int32_t *pos;   // [M]  (-1 = padding row)
};

// K/V ring of one layer set: [chunk][layer][ring][KV][64] fp32.
struct KvRing {
  float *k, *v;                 // fp32 (SIMT attention)
  float *k_hi, *k_lo, *v_hi, *v_lo;  // tf32 planes (tensor-core attention); null when unused
  int n_layers, ring, kv;
  __host__ __device__ size_t off(int c, int layer, int pos) const {
    return (((size_t)c * n_layers + layer) * ring + (size_t)(pos % ring)) * kv * kHeadDim;
  }
};

// ---------------------------------------------------------------- launchers
void launch_embed(const uint32_t *x, int M, const float *E, int d, float *h, float *h_hi, float *h_lo, cudaStream_t s);
void launch_rms(const float *h, int M, int d, float eps, float *rinv, cudaStream_t s);

enum GemmEpi { EPI_QKV = 0, EPI_RESID = 1, EPI_SWIGLU = 2, EPI_HEAD = 3 };
struct GemmArgs {
  const float *A; int lda;      // [M, K] row-major
  const float *B; int ldb;      // [N, K] row-major (weights)
  int M, N, K;
  const float *rinv;            // per-row scale (QKV, SWIGLU, HEAD) or null
  float *C; int ldc;            // output (RESID: in/out residual; HEAD: logits; SWIGLU: act)
  // QKV epilogue
  int layer, n_q_cols, n_kv_cols; // 576, 192
  RowMeta rows; KvRing ring;
  const float *rope_cos, *rope_sin;  // [max_pos, 32]
};
void launch_gemm(GemmEpi epi, const GemmArgs &a, cudaStream_t s);

struct AttnTile { int chunk, p0, nrows, qrow0; };
struct AttnArgs {
  const AttnTile *tiles; int n_tiles;
  const float *q; float *o; int ldq;   // [rows, H*64]
  float *o_hi, *o_lo;                  // optional tf32 planes of o for the tensor-core O projection
  KvRing ring; int layer;
  int H, KV, window, slide;
};
void launch_attention(const AttnArgs &a, cudaStream_t s);

}  // namespace nc
