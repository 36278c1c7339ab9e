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

// K/V ring of one layer set: [chunk][layer][ring][KV][64], stored as tf32 hi/lo planes.
struct KvRing {
  float *k_hi, *k_lo, *v_hi, *v_lo;  // tf32 planes read by the tensor-core attention
  int n_layers, ring, kv;
  __host__ __device__ size_t off(int c, int layer, int pos) const {
    return (((size_t)c * n_layers + layer) * ring + (size_t)(pos % ring)) * kv * kHeadDim;
  }
};

// ---------------------------------------------------------------- launchers
void launch_embed(const uint32_t *x, int M, const float *E, int d, float *h, float *h_hi, float *h_lo, float *ssq,
                  float *rinv, float eps, cudaStream_t s);

enum GemmEpi { EPI_QKV = 0, EPI_RESID = 1, EPI_SWIGLU = 2, EPI_HEAD = 3 };

// <= 128 consecutive rows [p0, p0 + nrows) of one chunk at slab rows qrow0..; w0 >= 0: the
// window start of every row of the tile (refresh slabs, NEXT-4), -1: w(j) of the formula (D10)
struct AttnTile { int chunk, p0, nrows, qrow0, w0; };

}  // namespace nc
