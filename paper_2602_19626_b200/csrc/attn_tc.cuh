// Host interface of the tensor-core window attention.
#pragma once
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace nc {

struct AttnTcArgs {
  const AttnTile *tiles; int n_tiles;        // tiles of <= 128 consecutive rows of one chunk
  const float *q_hi, *q_lo; int ldq; int q_rows;
  const float *k_hi, *k_lo, *v_hi, *v_lo;    // ring planes [chunk][layer][ring][KV][64]
  int ring, n_chunks, n_layers, layer;
  float *o_hi, *o_lo; int ldo;               // output tf32 planes [rows, H*64]
  int H, KV, window, slide;                  // window = L_max of the w(j) formula (D10)
  // decode steps (every tile one row of one chunk): the tile's rows are the H/KV q heads of one
  // KV group at that single position (q / o planes viewed as [rows * H, 64]); one item per
  // (tile, KV group) instead of per (tile, q head) -- each row's arithmetic is unchanged (D15)
  int heads_as_rows;
  int debug;                                 // unused
  int *item_ctr;                             // set by the launcher (persistent item scheduler)
};

void launch_attention_tc(const AttnTcArgs &a, cudaStream_t s);

// diagnostics build (-DNC_ATT_TIMING): print per-phase cycle sums to stderr
void attn_timing_report();

}  // namespace nc
