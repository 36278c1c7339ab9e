// Host interface of the tcgen05 3xTF32 GEMM.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace nc {

struct TcGemmArgs {
  int M, N, K;
  const float *rinv;          // per-row RMSNorm scale (QKV, SWIGLU, HEAD)
  // RESID: the RMSNorm statistics of the new h, for the next projection.  Every epilogue warp
  // writes its rows' sums of squares per 32-column slice (ssq_out [N / 32][ssq_ld >= M rounded
  // up to 32]) and counts in
  // rms_ctr (one counter per 32 rows); the last of the N / 64 warps covering those rows forms
  // rinv_out = 1/sqrt(sum_s ssq[s] / rms_d + rms_eps) (slices in order) and resets the counter
  float *ssq_out, *rinv_out; int *rms_ctr; float rms_d, rms_eps; int ssq_ld;
  float *C; int ldc;          // fp32 output: logits (HEAD), residual h in/out (RESID), q (QKV)
  float *C_hi, *C_lo;         // tf32 planes written for the next GEMM (RESID: h, SWIGLU: act; QKV: q planes)
  int layer, n_q_cols, n_kv_cols;
  RowMeta rows; KvRing ring;
  const float *rope_cos, *rope_sin;
  int *tile_ctr;               // set by the launcher
  // split-K (set by the launcher when the tile grid is much smaller than the SM count,
  // e.g. decode steps of one row per chunk): sps = 64-wide k spans per work item (0 = off),
  // ws = raw span partials [span][M][N] fp32, fix_ctr = per (tile, epilogue warp) arrival counters
  int sps;
  int a_box;                   // set by the launcher: rows of the A TMA box when M <= 128 (else 0)
  float *ws;
  int *fix_ctr;
  int no_store;                // diagnostics only (debug_gemm timing): skip the epilogue's global writes
};

struct TcOperands {
  const float *A_hi, *A_lo;   // [a_rows >= M, K]
  uint64_t a_rows;
  const float *B_hi, *B_lo;   // [N, K]
};

void launch_gemm_tc(GemmEpi epi, const TcGemmArgs &a, const TcOperands &op, cudaStream_t s);
// SMs left out of persistent grids (occupied by a concurrently running walk)
void set_reserved_sms(int n);
// split-K policy: 1 automatic (default), 0 never (tests: bit identity of the two)
void set_splitk_mode(int mode);
// programmatic dependent launch for the persistent grids (on unless NC_PDL=0)
bool pdl_enabled();
// diagnostics build (-DNC_GEMM_TIMING): epilogue phase cycles -> stderr
void gemm_timing_report();
void launch_split_planes(const float *x, float *hi, float *lo, size_t n, cudaStream_t s);

}  // namespace nc
