// fp32-accurate GEMM on the 5th-gen tensor cores: 3xTF32 with tcgen05.mma
// kind::tf32 (SURVEY.md D14 / hard part H2), operands staged by TMA, the
// accumulator in TMEM, and the layer's epilogue fused on the TMEM read-out.
//
//   C[m, n] = epi( sum_k A[m,k] B[n,k] ),  A = A_hi + A_lo, B = B_hi + B_lo (tf32 planes)
//   per 32-wide k block: D = sum_k (A_hi B_lo + A_lo B_hi), then D += sum_k A_hi B_hi (fixed order)
//
// Precision: every tcgen05.mma that accumulates into D rounds the sum toward
// zero (measured: relative bias -1.6e-5 at K = 1536 on positive data, i.e.
// ~0.5 ulp per MMA; tools/gemm_precision.py).  So each 32-wide k block is
// accumulated in a FRESH TMEM partial (12 MMAs) and the epilogue warps add the
// partials in fp32 round-to-nearest registers ("promotion"), which restores
// ~fp32 accuracy (D14).
//
// Tile shape.  A tcgen05.mma costs the same ~153 cycles for every N up to 256
// (tools/micro/mma_bench.cu: M=128 tf32 N=64/128/256 all 153 cycles), and the
// chip's TMA/L2 service rate (~6.3 KB/cycle, B300_MICROARCH) cannot feed 148
// SMs streaming four fp32 planes for 128 x 256 tiles.  So a CTA PAIR
// (cluster of 2, cta_group::2) computes a 256 x 256 tile: each CTA stages its
// 128 rows of A and 128 of the 256 rows of B (64 KB per 32-wide k block), the
// leader issues M=256 N=256 MMAs that read both CTAs' shared memory, and each
// CTA's TMEM holds its 128 x 256 accumulator rows.
//
// Warp roles (320 threads = 10 warps per CTA, 1 CTA / SM):
//   warps 0-7 promotion + epilogue (both CTAs): warp w reads TMEM lanes 32(w%4).. and
//           column half w/4; tcgen05.ld partials -> fp32 RN sums (128 registers)
//           -> fused epilogue -> global
//   warp 8  TMA producer (one thread; both CTAs load their halves, bytes land on the
//           leader's barrier) and TMEM allocator (2 x 256 fp32 columns, pair alloc)
//   warp 9  MMA issuer (leader only): 12 pair MMAs per 32-wide k block into a partial buffer
// Tiles are claimed dynamically by the leader's producer (atomic counter; the
// last CTA to exit resets it) and broadcast to the peer through DSMEM, so CTAs
// that start late -- e.g. on SMs a concurrently running walk held -- find no
// work instead of stalling the GEMM.  Claim order: see tile_mn.
//
// Row results do not depend on which other rows share the tile (each output
// element is one fixed sequence of MMAs), so prefill and decode agree bit for
// bit (D15).
//
// Split-K (decode: a few rows, a handful of tiles on 148 SMs).  A work item is
// (tile, run of sps 64-wide k spans).  Every span still gets its own fresh TMEM
// partial from the same MMA sequence; the epilogue warps write the raw partials
// to a workspace instead of summing them, and the last warp to arrive for its
// (tile, warp) region re-reads all partials and sums them in span order --
// exactly the promotion sum of the unsplit kernel -- before running the same
// epilogue code.  So split and unsplit launches give identical bits.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>

#include "gemm_tc.cuh"
#include "tc_common.cuh"

namespace nc {

constexpr int TBM = 128;              // rows per CTA (pair tile: 256)
// tile width of the few-row GEMMs of decode steps (M <= 128): their k loop is bound by the
// N-proportional MMA cost (12 pair MMAs per 32-wide k block), not by rows
#ifndef NC_DECODE_BN
#define NC_DECODE_BN 64
#endif
// BN = pair tile columns (MMA N; each CTA stages BN / 2 rows of B): 256, or 192 for
// the N = 576 residual GEMMs (576 = 3 x 192: no padded MMA work, smaller output bursts)
constexpr int TBK = 32, NPART = 2, NSCHED = 4;
// k blocks per TMEM partial.  Promotion reads the whole 128 x 256 fp32 partial
// (128 KB) per CTA; tcgen05.ld moves ~64 B/cycle/SM (B300_MICROARCH), i.e.
// 2048 cycles, against 12 * 128 = 1536 MMA cycles per 32-wide k block -- so a
// partial spans 2 k blocks (3072 MMA cycles) to keep the tensor pipe the bound.
#ifndef NC_KPP
#define NC_KPP 2
#endif
constexpr int KPP = NC_KPP;
// split-K fixup: rows folded at once (all spans in flight) and the largest span count
constexpr int SK_ROWS = 2, SK_MIN_SPANS = 16, SK_MAX_SPANS = 24, SK_MAX_ROWS = 16;
constexpr int TILE_A_BYTES = TBM * TBK * 4;          // 16 KB
constexpr int TMEM_COLS = 512;                              // NPART x BN <= 512, power of two
template <int BN>
struct TileCfg {
  // epilogue warps: 4 TMEM lane quarters x column groups; 192-wide tiles take three groups
  // of 64 (one attention head / two 32-column residual slices per warp) so their output
  // phase -- which the MMA of the next tile can only run two partials ahead of -- is short
  static constexpr int EPI_COLS = (BN == 192 || BN == 64) ? 64 : BN / 2;  // columns per epilogue warp
  static constexpr int EPI_WARPS = 4 * (BN / EPI_COLS);                  // 8, or 12 at BN = 192
  static constexpr int THREADS = 32 * (EPI_WARPS + 2);                   // + TMA/allocator + MMA warps
  static constexpr int W_TMA = EPI_WARPS, W_MMA = EPI_WARPS + 1;
  static constexpr int OUT_STAGE_BYTES = EPI_WARPS * 32 * 32 * 4;        // per-warp 32 x 32 transpose tiles
  // sch_empty arrivals per tile claim: leader MMA + the epilogue warps of both CTAs + the peer's producer
  static constexpr int SCHED_CONSUMERS = 1 + 2 * EPI_WARPS + 1;
  static constexpr int TILE_B_BYTES = (BN / 2) * TBK * 4;                // 16 / 12 KB
  static constexpr int STAGE_BYTES = 2 * TILE_A_BYTES + 2 * TILE_B_BYTES;   // 64 / 56 KB per CTA
  // pipeline depth: 3 stages of 64 / 56 KB; the 128-wide tiles (decode steps, whose k loop
  // is bound by TMA round trips rather than MMAs) fit a fourth 48 KB stage
  static constexpr int STAGES = BN == 64 ? 5 : (BN == 128 ? 4 : 3);
  static constexpr int SMEM = STAGES * STAGE_BYTES + OUT_STAGE_BYTES + 1024 /*align*/ + 512 /*barriers*/;
  static_assert(NPART * BN <= TMEM_COLS && BN % 32 == 0 && EPI_COLS % 32 == 0, "tile");
};

// This lane's 32 row values -> the warp's swizzled staging tile -> one TMA bulk tensor
// store of the warp's 32 x 32 box at (c0, r0) (the tile layout is exactly the
// SWIZZLE_128B box layout; rows past the tensor's extent are clipped).  The warp waits
// only until the previous store has READ the tile, never for global writes.
__device__ __forceinline__ void tma_store32(float *stg, const CUtensorMap *map, int c0, int r0, const float *v,
                                            int lane) {
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 8; ++k)
    *reinterpret_cast<float4 *>(stg + lane * 32 + 4 * (k ^ (lane & 7))) =
        make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(r0), "r"(tc::smem_u32(stg))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
}
// tf32 hi/lo planes of 32 values through two TMA stores
__device__ __forceinline__ void tma_store32_planes(float *stg, const CUtensorMap *mh, const CUtensorMap *ml, int c0,
                                                   int r0, const float *v, int lane) {
  float hi[32], lo[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) tc::split_tf32(v[k], hi[k], lo[k]);
  tma_store32(stg, mh, c0, r0, hi, lane);
  tma_store32(stg, ml, c0, r0, lo, lane);
}

// Row-contiguous output through a per-warp 32 x 32 shared tile.  Lane l holds
// 32 consecutive outputs v[0..31] of row l (its TMEM lane); written to the
// tile as 8 float4 chunks swizzled by (l & 7), read back 4 rows per
// instruction (lanes 8i..8i+7 -> row 4i'+i, chunk lane&7), so each global
// access covers 128 contiguous bytes of one row.  d0 (d1, d2) are the row's
// destinations (this lane's row); d0 == nullptr skips the row.
//   ST_PLAIN  d0 = v
//   ST_SPLIT  d0 = tf32 hi(v), d1 = lo(v)
//   ST_RESID  h = d0 + v (fp32 RN); d0 = h, d1 = hi(h), d2 = lo(h); and, if ssq != nullptr, the
//             slice's sum of squares of h for each row r of the warp at ssq[r] (one coalesced
//             128 B store; rows past M hold garbage): per lane ((x^2 + y^2) + z^2) + w^2 (fma)
//             over its 4 columns, then an xor tree over the row's 8 lanes (1, 2, 4) -- the same
//             arithmetic as embed_kernel's
enum { ST_PLAIN = 0, ST_SPLIT = 1, ST_RESID = 2 };
template <int MODE>
__device__ __forceinline__ void store_rows32(float *stg, const float *v, float *d0, float *d1, float *d2, int lane,
                                             float *ssq = nullptr) {
#pragma unroll
  for (int k = 0; k < 8; ++k)
    *reinterpret_cast<float4 *>(stg + lane * 32 + 4 * (k ^ (lane & 7))) =
        make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
  __syncwarp();
  const int c4 = lane & 7;
  float4 hin[MODE == ST_RESID ? 8 : 1];
  if (MODE == ST_RESID) {   // residual rows (L2-resident: prefetched at tile start); all loads before any store
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = 4 * i + (lane >> 3);
      const float *p0 =
          reinterpret_cast<const float *>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(d0), r));
      hin[i] = p0 ? *reinterpret_cast<const float4 *>(p0 + 4 * c4) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  float mine = 0.f;   // ST_RESID: row `lane`'s slice sum (row 4 i + j sits in lanes 8 j .. 8 j + 7 at step i)
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = 4 * i + (lane >> 3);
    float sq = 0.f;
    float *p0 = reinterpret_cast<float *>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(d0), r));
    float *p1 = MODE != ST_PLAIN
                    ? reinterpret_cast<float *>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(d1), r))
                    : nullptr;
    float *p2 = MODE == ST_RESID
                    ? reinterpret_cast<float *>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(d2), r))
                    : nullptr;
    if (p0) {
      float4 y = *reinterpret_cast<const float4 *>(stg + r * 32 + 4 * (c4 ^ (r & 7)));
      if (MODE == ST_PLAIN) {
        *reinterpret_cast<float4 *>(p0 + 4 * c4) = y;
      } else {
        if (MODE == ST_RESID) {
          y.x = __fadd_rn(hin[i].x, y.x); y.y = __fadd_rn(hin[i].y, y.y);
          y.z = __fadd_rn(hin[i].z, y.z); y.w = __fadd_rn(hin[i].w, y.w);
          *reinterpret_cast<float4 *>(p0 + 4 * c4) = y;
          sq = __fmaf_rn(y.w, y.w, __fmaf_rn(y.z, y.z, __fmaf_rn(y.y, y.y, __fmul_rn(y.x, y.x))));
        }
        float4 hi, lo;
        tc::split_tf32(y.x, hi.x, lo.x); tc::split_tf32(y.y, hi.y, lo.y);
        tc::split_tf32(y.z, hi.z, lo.z); tc::split_tf32(y.w, hi.w, lo.w);
        float *ph = MODE == ST_RESID ? p1 : p0, *pl = MODE == ST_RESID ? p2 : p1;
        *reinterpret_cast<float4 *>(ph + 4 * c4) = hi;
        *reinterpret_cast<float4 *>(pl + 4 * c4) = lo;
      }
    }
    if (MODE == ST_RESID && ssq) {   // the row's 8 lanes reduce (all lanes shuffle)
      float t = sq;
      t = __fadd_rn(t, __shfl_xor_sync(0xffffffffu, t, 1));
      t = __fadd_rn(t, __shfl_xor_sync(0xffffffffu, t, 2));
      t = __fadd_rn(t, __shfl_xor_sync(0xffffffffu, t, 4));
      const float u = __shfl_sync(0xffffffffu, t, 8 * (lane & 3));
      if ((lane >> 2) == i) mine = u;
    }
  }
  if (MODE == ST_RESID && ssq) ssq[lane] = mine;
  __syncwarp();
}

// One 64-column head (q, k or v) of this warp's 32 rows: both 32-column halves
// go through the swizzled tile so every lane holds the rotate-half pairs
// (d, d + 32) of 4 rows x 4 columns; RoPE then reads each row's cos/sin as
// row-contiguous float4s (per-lane scalar table reads were 64 uncoalesced loads
// per head and dominated the QKV GEMM).  Same per-element arithmetic as before:
//   y1 = fma(x1, c, -x2 s),  y2 = fma(x2, c, x1 s).
// PLANES: d0/d1 = tf32 hi/lo destinations of the row; else d0 = fp32 destination.
template <bool PLANES>
__device__ __forceinline__ void store_head64(float *stg, const float *x, int pos, bool rope, const float *cos_t,
                                             const float *sin_t, float *d0, float *d1, int lane) {
  const int c4 = lane & 7;
  float4 t[2][8];
#pragma unroll
  for (int hf = 0; hf < 2; ++hf) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      *reinterpret_cast<float4 *>(stg + lane * 32 + 4 * (k ^ (lane & 7))) =
          make_float4(x[32 * hf + 4 * k], x[32 * hf + 4 * k + 1], x[32 * hf + 4 * k + 2], x[32 * hf + 4 * k + 3]);
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = 4 * i + (lane >> 3);
      t[hf][i] = *reinterpret_cast<const float4 *>(stg + r * 32 + 4 * (c4 ^ (r & 7)));
    }
    __syncwarp();
  }
  // the rows' cos/sin in two batches of four (read-only path, a batch's loads in flight
  // together): loaded inside the store loop they sat behind the previous row's stores
  // (possible aliasing), one L2 round trip per row -- the QKV output phase was ~12k cycles
  // per tile.  (All eight at once spills at the 128-register cap of the 448-thread CTA.)
#pragma unroll
  for (int ib = 0; ib < 2; ++ib) {
    float4 cs[4], sn4[4];
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      const int pr = __shfl_sync(0xffffffffu, pos, 4 * (4 * ib + ii) + (lane >> 3));
      if (rope && pr >= 0) {
        cs[ii] = __ldg(reinterpret_cast<const float4 *>(cos_t + (size_t)pr * 32 + 4 * c4));
        sn4[ii] = __ldg(reinterpret_cast<const float4 *>(sin_t + (size_t)pr * 32 + 4 * c4));
      } else {
        cs[ii] = sn4[ii] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
  for (int ii = 0; ii < 4; ++ii) {
    const int i = 4 * ib + ii;
    const int r = 4 * i + (lane >> 3);
    const int pr = __shfl_sync(0xffffffffu, pos, r);
    float *p0 = reinterpret_cast<float *>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(d0), r));
    float *p1 = PLANES ? reinterpret_cast<float *>(
                             __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(d1), r))
                       : nullptr;
    if (pr < 0 || !p0) continue;
    float4 y1 = t[0][i], y2 = t[1][i];
    if (rope) {
      const float4 c = cs[ii], sn = sn4[ii];
      const float4 x1 = y1, x2 = y2;
      y1.x = __fmaf_rn(x1.x, c.x, __fmul_rn(-x2.x, sn.x)); y2.x = __fmaf_rn(x2.x, c.x, __fmul_rn(x1.x, sn.x));
      y1.y = __fmaf_rn(x1.y, c.y, __fmul_rn(-x2.y, sn.y)); y2.y = __fmaf_rn(x2.y, c.y, __fmul_rn(x1.y, sn.y));
      y1.z = __fmaf_rn(x1.z, c.z, __fmul_rn(-x2.z, sn.z)); y2.z = __fmaf_rn(x2.z, c.z, __fmul_rn(x1.z, sn.z));
      y1.w = __fmaf_rn(x1.w, c.w, __fmul_rn(-x2.w, sn.w)); y2.w = __fmaf_rn(x2.w, c.w, __fmul_rn(x1.w, sn.w));
    }
    if (PLANES) {
      float4 h1, l1, h2, l2;
      tc::split_tf32(y1.x, h1.x, l1.x); tc::split_tf32(y1.y, h1.y, l1.y);
      tc::split_tf32(y1.z, h1.z, l1.z); tc::split_tf32(y1.w, h1.w, l1.w);
      tc::split_tf32(y2.x, h2.x, l2.x); tc::split_tf32(y2.y, h2.y, l2.y);
      tc::split_tf32(y2.z, h2.z, l2.z); tc::split_tf32(y2.w, h2.w, l2.w);
      *reinterpret_cast<float4 *>(p0 + 4 * c4) = h1;
      *reinterpret_cast<float4 *>(p1 + 4 * c4) = l1;
      *reinterpret_cast<float4 *>(p0 + 32 + 4 * c4) = h2;
      *reinterpret_cast<float4 *>(p1 + 32 + 4 * c4) = l2;
    } else {
      *reinterpret_cast<float4 *>(p0 + 4 * c4) = y1;
      *reinterpret_cast<float4 *>(p0 + 32 + 4 * c4) = y2;
    }
  }
  }
}

#ifdef NC_GEMM_TIMING
// diagnostics build only: epilogue phase cycle sums of warp 0 lane 0 (per tile)
__device__ unsigned long long g_gemm_clk[4 * 8];   // [EPI][phase]
#define GEMM_MARK(k)                                                                        \
  do {                                                                                      \
    if (threadIdx.x == 0) {                                                                 \
      const long long _n = clock64();                                                       \
      atomicAdd(&g_gemm_clk[EPI * 8 + (k)], (unsigned long long)(_n - _gt));                 \
      _gt = _n;                                                                             \
    }                                                                                       \
  } while (0)
#else
#define GEMM_MARK(k) do {} while (0)
#endif

template <int EPI, int BN, bool SPLIT>
__global__ __launch_bounds__(TileCfg<BN>::THREADS, 1) void gemm_tc_kernel(const __grid_constant__ CUtensorMap tmAh,
                                                                const __grid_constant__ CUtensorMap tmAl,
                                                                const __grid_constant__ CUtensorMap tmBh,
                                                                const __grid_constant__ CUtensorMap tmBl,
                                                                const __grid_constant__ CUtensorMap tmC0,
                                                                const __grid_constant__ CUtensorMap tmC1,
                                                                const __grid_constant__ CUtensorMap tmC2,
                                                                TcGemmArgs a) {
  using C_ = TileCfg<BN>;
  constexpr int TBN = BN, EPI_COLS = C_::EPI_COLS, TILE_B_BYTES = C_::TILE_B_BYTES, STAGE_BYTES = C_::STAGE_BYTES;
  constexpr int TSTAGES = C_::STAGES;
  constexpr int EPI_WARPS = C_::EPI_WARPS, W_TMA = C_::W_TMA, W_MMA = C_::W_MMA;
  constexpr int OUT_STAGE_BYTES = C_::OUT_STAGE_BYTES, SCHED_CONSUMERS = C_::SCHED_CONSUMERS;
  static_assert(KPP <= TSTAGES, "a partial's k blocks must fit the pipeline (corrections-first MMA order)");
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float *stage_out = reinterpret_cast<float *>(smem + TSTAGES * STAGE_BYTES);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + TSTAGES * STAGE_BYTES + OUT_STAGE_BYTES);
  uint64_t *empty = full + TSTAGES;
  uint64_t *tfull = empty + TSTAGES;
  uint64_t *tempty = tfull + NPART;
  uint64_t *sch_full = tempty + NPART, *sch_empty = sch_full + NSCHED;
  int *sch_tile = reinterpret_cast<int *>(sch_empty + NSCHED);
  uint32_t *tmem_base_smem = reinterpret_cast<uint32_t *>(sch_tile + NSCHED);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc::cluster_ctarank();      // 0 = leader of the pair
  const int num_m = (a.M + 2 * TBM - 1) / (2 * TBM), num_n = (a.N + TBN - 1) / TBN;
  const int n_tiles = num_m * num_n;
  const int nk = a.K / TBK;
  const int nspan = (nk + KPP - 1) / KPP;
  const int sps = (SPLIT && a.sps > 0) ? a.sps : nspan;      // spans per work item
  const int nsplit = (nspan + sps - 1) / sps;
  const int n_items = n_tiles * nsplit;
  // work item -> tile, k-block range [kb_lo, kb_hi)
  auto item_k = [&](int t, int &tile, int &kb_lo, int &kb_hi) {
    tile = t / nsplit;
    const int sp = t - tile * nsplit;
    kb_lo = sp * sps * KPP;
    kb_hi = min(nk, (sp + 1) * sps * KPP);
  };
  // Claim order.  Many N tiles (vocab head, gate/up): bands of RB M tiles, M-fastest
  // inside a band, sweeping every N tile -- the band's A rows (RB x 256 rows, ~37 MB of
  // tf32 planes at K = 576) stay in L2 while B streams once per band.  (Plain
  // M-fastest re-read all of A from DRAM for every N tile on the head: 25.8 GB per
  // launch.)  Few N tiles: N-fastest, the A tile is reused across them from L2.
  constexpr int RB = 32;
  const bool m_fast = num_n >= num_m;
  auto tile_mn = [&](int t, int &mb, int &nb) {
    if (m_fast) {
      const int band = t / (RB * num_n), r = t - band * RB * num_n;
      const int rows = min(RB, num_m - band * RB);
      mb = band * RB + r % rows;
      nb = r / rows;
    } else {
      nb = t % num_n;
      mb = t / num_n;
    }
  };

  if (warp == W_TMA && lane == 0) {
    tc::tma_prefetch(&tmAh); tc::tma_prefetch(&tmAl); tc::tma_prefetch(&tmBh); tc::tma_prefetch(&tmBl);
    for (int s = 0; s < TSTAGES; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
    for (int s = 0; s < NPART; ++s) { tc::mbar_init(&tfull[s], 1); tc::mbar_init(&tempty[s], 2 * EPI_WARPS); }
    for (int s = 0; s < NSCHED; ++s) { tc::mbar_init(&sch_full[s], 1); tc::mbar_init(&sch_empty[s], SCHED_CONSUMERS); }
    tc::fence_barrier_init();
  }
  if (warp == W_TMA) tc::tmem_alloc_pair(tmem_base_smem, TMEM_COLS);
  tc::fence_before();
  tc::cluster_sync();
  tc::fence_after();
  const uint32_t tmem_base = *tmem_base_smem;
  tc::pdl_launch_dependents();
  tc::pdl_wait();   // everything below reads what earlier kernels wrote (or claims tiles)

  if (warp == W_TMA) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      // few rows (decode, M <= 128): A comes as an a_box-row box into the first rows of the
      // leader's A tile and the peer loads no A at all (its rows 128.. are all >= M); the
      // MMA still reads 128 rows, the extra rows only feed output rows that are never stored
      const bool load_a = a.a_box == 0 || rank == 0;
      const uint32_t stage_tx = a.a_box == 0 ? 2 * STAGE_BYTES : 2 * 2 * TILE_B_BYTES + 2 * a.a_box * TBK * 4;
      for (int jt = 0;; ++jt) {
        const int slot = jt % NSCHED;
        int t;
        if (rank == 0) {
          tc::mbar_wait(&sch_empty[slot], ((jt / NSCHED) & 1) ^ 1);
          const int claimed = atomicAdd(a.tile_ctr, 1);
          t = claimed < n_items ? claimed : -1;
          sch_tile[slot] = t;
          tc::st_cluster_s32(tc::mapa(&sch_tile[slot], 1), t);
          tc::mbar_arrive(&sch_full[slot]);
          tc::mbar_arrive_cluster(tc::mapa(&sch_full[slot], 1));
        } else {
          tc::mbar_wait_cluster(&sch_full[slot], (jt / NSCHED) & 1);
          t = sch_tile[slot];
          tc::mbar_arrive_remote(tc::mapa(&sch_empty[slot], 0));
        }
        if (t < 0) break;
        int mb, nb, tile, kb_lo, kb_hi;
        item_k(t, tile, kb_lo, kb_hi);
        tile_mn(tile, mb, nb);
        const int row_a = mb * 2 * TBM + (int)rank * TBM, row_b = nb * TBN + (int)rank * (TBN / 2);
        for (int kb = kb_lo; kb < kb_hi; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t *st = smem + stage * STAGE_BYTES;
          if (rank == 0) tc::mbar_expect_tx(&full[stage], stage_tx);   // both CTAs' bytes
          if (load_a) {
            tc::tma_load_2d_pair(st, &tmAh, kb * TBK, row_a, &full[stage]);
            tc::tma_load_2d_pair(st + TILE_A_BYTES, &tmAl, kb * TBK, row_a, &full[stage]);
          }
          tc::tma_load_2d_pair(st + 2 * TILE_A_BYTES, &tmBh, kb * TBK, row_b, &full[stage]);
          tc::tma_load_2d_pair(st + 2 * TILE_A_BYTES + TILE_B_BYTES, &tmBl, kb * TBK, row_b, &full[stage]);
          if (++stage == TSTAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == W_MMA) {
    // ------------------------------------------------------ MMA issuer (leader)
    if (rank == 0 && lane == 0) {
      constexpr uint32_t idesc = tc::idesc_tf32(2 * TBM, TBN);
      int stage = 0;
      uint32_t phase = 0;
      int buf = 0;
      uint32_t buf_phase = 0;
      for (int jt = 0;; ++jt) {
        const int slot = jt % NSCHED;
        tc::mbar_wait(&sch_full[slot], (jt / NSCHED) & 1);
        const int t = sch_tile[slot];
        tc::mbar_arrive(&sch_empty[slot]);
        if (t < 0) break;
        int tile, kb_lo, kb_hi;
        item_k(t, tile, kb_lo, kb_hi);
        // one TMEM partial per KPP k blocks (a fresh accumulator, promoted in fp32 RN by
        // the epilogue); within it see the two orders below
        for (int kb0 = kb_lo; kb0 < kb_hi; kb0 += KPP) {
          const int nkp = min(KPP, kb_hi - kb0);
          tc::mbar_wait(&tempty[buf], buf_phase ^ 1);   // partial drained by both CTAs' epilogues
          const uint32_t d = tmem_base + buf * BN;
          int st = stage;
          uint32_t ph = phase;
#ifndef NC_MMA_CORR_FIRST
          // per k block its corrections then its hi*hi, the stage released right after: the
          // producer runs a k block further ahead than with all of a span's corrections first
          // (measured: QKV/O/down GEMMs -4 to -5 %, step -1 ms), at 12 instead of 8 large-
          // magnitude truncations per partial (GEMM max rel. error 4.3e-7 -> 5.9e-7 at K = 576,
          // tools/gemm_precision.py).  -DNC_MMA_CORR_FIRST restores the corrections-first order.
          for (int i = 0; i < nkp; ++i) {
            tc::mbar_wait(&full[st], ph);
            tc::fence_after();
            const uint32_t s0 = tc::smem_u32(smem + st * STAGE_BYTES);
            const uint64_t dah = tc::desc_k_sw128(s0), dal = tc::desc_k_sw128(s0 + TILE_A_BYTES);
            const uint64_t dbh = tc::desc_k_sw128(s0 + 2 * TILE_A_BYTES);
            const uint64_t dbl = tc::desc_k_sw128(s0 + 2 * TILE_A_BYTES + TILE_B_BYTES);
#pragma unroll
            for (int j = 0; j < TBK / 8; ++j) {
              const uint64_t adv = (uint64_t)(j * 32) >> 4;
              tc::mma_tf32_pair(d, dah + adv, dbl + adv, idesc, (i | j) != 0);
              tc::mma_tf32_pair(d, dal + adv, dbh + adv, idesc, 1);
            }
#pragma unroll
            for (int j = 0; j < TBK / 8; ++j) {
              const uint64_t adv = (uint64_t)(j * 32) >> 4;
              tc::mma_tf32_pair(d, dah + adv, dbh + adv, idesc, 1);
            }
            tc::mma_commit_pair(&empty[st]);
            if (++st == TSTAGES) { st = 0; ph ^= 1; }
          }
          stage = st;
          phase = ph;
#else
          for (int i = 0; i < nkp; ++i) {
            tc::mbar_wait(&full[st], ph);
            tc::fence_after();
            const uint32_t s0 = tc::smem_u32(smem + st * STAGE_BYTES);
            const uint64_t dah = tc::desc_k_sw128(s0), dal = tc::desc_k_sw128(s0 + TILE_A_BYTES);
            const uint64_t dbh = tc::desc_k_sw128(s0 + 2 * TILE_A_BYTES);
            const uint64_t dbl = tc::desc_k_sw128(s0 + 2 * TILE_A_BYTES + TILE_B_BYTES);
#pragma unroll
            for (int j = 0; j < TBK / 8; ++j) {
              const uint64_t adv = (uint64_t)(j * 32) >> 4;   // 8 tf32 = 32 bytes along K
              tc::mma_tf32_pair(d, dah + adv, dbl + adv, idesc, (i | j) != 0);
              tc::mma_tf32_pair(d, dal + adv, dbh + adv, idesc, 1);
            }
            if (++st == TSTAGES) { st = 0; ph ^= 1; }
          }
          for (int i = 0; i < nkp; ++i) {
            const uint32_t s0 = tc::smem_u32(smem + stage * STAGE_BYTES);
            const uint64_t dah = tc::desc_k_sw128(s0), dbh = tc::desc_k_sw128(s0 + 2 * TILE_A_BYTES);
#pragma unroll
            for (int j = 0; j < TBK / 8; ++j) {
              const uint64_t adv = (uint64_t)(j * 32) >> 4;
              tc::mma_tf32_pair(d, dah + adv, dbh + adv, idesc, 1);
            }
            tc::mma_commit_pair(&empty[stage]);
            if (++stage == TSTAGES) { stage = 0; phase ^= 1; }
          }
#endif
          tc::mma_commit_pair(&tfull[buf]);
          if (++buf == NPART) { buf = 0; buf_phase ^= 1; }
        }
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    const int q = warp & 3;     // TMEM lanes 32q .. 32q+31
    const int hc = warp >> 2;   // column group of the tile (EPI_COLS wide)
    const uint32_t sch_empty_leader = tc::mapa(&sch_empty[0], 0);
    const uint32_t tempty_leader = tc::mapa(&tempty[0], 0);
    int buf = 0;
    uint32_t buf_phase = 0;
    // RESID: RMSNorm statistics of the rows this warp stored (first row rms_pend, -1 = none),
    // counted after the next tile's k loop -- by then the stores have drained and the fence is
    // cheap (a fence right after them stalled the store-bound epilogue).  The last of the N / EPI_COLS warps
    // covering these 32 rows sums their slice sums in order into rinv_out.
    int rms_pend = -1;
    auto rms_flush = [&]() {
      if (EPI != EPI_RESID || rms_pend < 0) return;
      __threadfence();
      __syncwarp();
      int last = 0;
      if (lane == 0) {
        int *ctr = a.rms_ctr + rms_pend / 32;
        last = atomicAdd(ctr, 1) == (a.N + EPI_COLS - 1) / EPI_COLS - 1;
        if (last) *ctr = 0;   // every warp of these rows is in: reset for the next launch
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      const int mr = rms_pend + lane;
      if (last && mr < a.M) {
        __threadfence();
        const int ns = a.N / 32;
        const float *q = a.ssq_out + mr;
        float ss = 0.f;
        for (int k = 0; k < ns; ++k) ss = __fadd_rn(ss, __ldcg(q + (size_t)k * a.ssq_ld));
        a.rinv_out[mr] = __frsqrt_rn(__fadd_rn(__fdiv_rn(ss, a.rms_d), a.rms_eps));
      }
      rms_pend = -1;
    };
    for (int jt = 0;; ++jt) {
      const int slot = jt % NSCHED;
#ifdef NC_GEMM_TIMING
      long long _gt = clock64();
#endif
      tc::mbar_wait_cluster(&sch_full[slot], (jt / NSCHED) & 1);
      GEMM_MARK(0);   // wait for the tile
      const int t = sch_tile[slot];
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_remote(sch_empty_leader + slot * 8);
      if (t < 0) {
        rms_flush();
        break;
      }
#ifdef NC_GEMM_TIMING
      if (threadIdx.x == 0) atomicAdd(&g_gemm_clk[EPI * 8 + 7], 1ull);
#endif
      int mb, nb, tile, kb_lo, kb_hi;
      item_k(t, tile, kb_lo, kb_hi);
      tile_mn(tile, mb, nb);
      const int m = mb * (2 * TBM) + (int)rank * TBM + q * 32 + lane;
      const int row0 = mb * (2 * TBM) + (int)rank * TBM + q * 32;   // this warp's first row (TMA stores)
      const bool row_ok = m < a.M;
      const float rs = (EPI != EPI_RESID && row_ok && a.rinv) ? a.rinv[m] : 1.f;   // loaded under the k loop
      constexpr bool split = SPLIT;   // (a split launch always has nsplit >= 2)
      const int col0 = nb * TBN + hc * EPI_COLS;   // this warp's first column
      float acc[EPI_COLS];
      float *stg = stage_out + warp * 32 * 32;   // this warp's 32 x 32 transpose tile
      if (EPI == EPI_RESID && !a.no_store) {
        // residual rows of this warp's 32 x 128 block into L2 now (no registers); they
        // are read (from L2) and added after the promotion sum: h_new = h + sum_p P_p
        if (row_ok) {
          const char *hrow = reinterpret_cast<const char *>(a.C + (size_t)m * a.ldc + col0);
#pragma unroll
          for (int l = 0; l < EPI_COLS * 4 / 128; ++l)
            if (col0 + l * 32 < a.N) asm volatile("prefetch.global.L2 [%0];" ::"l"(hrow + l * 128));
        }
      }
      if (EPI == EPI_QKV && !a.no_store && row_ok && col0 < a.n_q_cols + a.n_kv_cols) {
        // this row's RoPE cos/sin lines into L1 under the k loop: the epilogue reads them
        // (4 rows per instruction) once per head; each was an exposed L2 round trip
        const int pr = a.rows.pos[m];
        if (pr >= 0) {
          asm volatile("prefetch.global.L1 [%0];" ::"l"(a.rope_cos + (size_t)pr * 32));
          asm volatile("prefetch.global.L1 [%0];" ::"l"(a.rope_sin + (size_t)pr * 32));
        }
      }
      {
#pragma unroll
        for (int j = 0; j < EPI_COLS; ++j) acc[j] = 0.f;
      }
      GEMM_MARK(1);   // residual seed
      for (int kb0 = kb_lo; kb0 < kb_hi; kb0 += KPP) {
        tc::mbar_wait(&tfull[buf], buf_phase);
        GEMM_MARK(2);   // waiting for partials
        tc::fence_after();
        const uint32_t taddr = tmem_base + buf * BN + hc * EPI_COLS + ((uint32_t)(q * 32) << 16);
        if (split) {   // raw span partial -> workspace [span][M][N] (row-major per span)
          float *wp = a.ws + ((size_t)(kb0 / KPP) * a.M + m) * a.N + col0;
#pragma unroll
          for (int c = 0; c < EPI_COLS / 16; ++c) {
            uint32_t r[16];
            tc::tmem_ld16(taddr + c * 16, r);
            tc::tmem_wait_ld();
            if (row_ok && col0 + c * 16 < a.N)   // N % 16 == 0: whole 16-column groups
#pragma unroll
              for (int j = 0; j < 16; j += 4)
                __stcg(reinterpret_cast<float4 *>(wp + c * 16 + j),
                       make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                                   __uint_as_float(r[j + 3])));
          }
        } else {
#pragma unroll
          for (int c = 0; c < EPI_COLS / 16; ++c) {
            uint32_t r[16];
            tc::tmem_ld16(taddr + c * 16, r);
            tc::tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[c * 16 + j] = __fadd_rn(acc[c * 16 + j], __uint_as_float(r[j]));
          }
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_remote(tempty_leader + buf * 8);
        if (++buf == NPART) { buf = 0; buf_phase ^= 1; }
      }
      GEMM_MARK(5);   // partials drained / written
      rms_flush();    // the previous tile's RMSNorm count: its stores drained under this k loop
      if (split) {
        // the last of the nsplit warps covering this (tile, warp) region sums every span's
        // partial in span order (= the unsplit promotion sum) and runs the epilogue
        if (!__any_sync(0xffffffffu, row_ok) || col0 >= a.N) continue;   // same decision in every split
        __threadfence();
        __syncwarp();
        int last = 0;
        if (lane == 0) {
          int *ctr = a.fix_ctr + ((size_t)tile * 2 + rank) * EPI_WARPS + warp;
          last = atomicAdd(ctr, 1) == nsplit - 1;
          if (last) *ctr = 0;   // every arrival of this launch is in: reset for the next launch
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (!last) continue;
        __threadfence();
      }
      // split-K fixup (only the last warp of a region gets here): dst[0..31] (lane = row) =
      // (((0 + P_0) + P_1) + ...) of columns cc..cc+31, exactly the unsplit promotion sum.
      // Folded with lane = column (coalesced 128 B workspace rows), every span of SK_ROWS
      // rows in flight, through the warp's smem tile; done per epilogue block just before
      // the block is consumed, so no more than one block of sums is live at a time.
      auto fold32 = [&](float *dst, int cc) {
        const int nr = min(32, a.M - row0);
        const size_t sstride = (size_t)a.M * a.N;
        const float *col_base = a.ws + col0 + cc + lane;
        for (int r0 = 0; r0 < nr; r0 += SK_ROWS) {
          float v[SK_ROWS][SK_MAX_SPANS];
#pragma unroll
          for (int rr = 0; rr < SK_ROWS; ++rr)
#pragma unroll
            for (int sp = 0; sp < SK_MAX_SPANS; ++sp)
              v[rr][sp] = (sp < nspan && r0 + rr < nr)
                              ? __ldcg(col_base + sp * sstride + (size_t)(row0 + r0 + rr) * a.N)
                              : 0.f;
#pragma unroll
          for (int rr = 0; rr < SK_ROWS; ++rr) {
            float sum = 0.f;
#pragma unroll
            for (int sp = 0; sp < SK_MAX_SPANS; ++sp)
              if (sp < nspan) sum = __fadd_rn(sum, v[rr][sp]);
            if (r0 + rr < nr) stg[(r0 + rr) * 32 + (lane ^ (r0 + rr))] = sum;
          }
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 32; ++j) dst[j] = stg[lane * 32 + (j ^ lane)];
        __syncwarp();
      };
      GEMM_MARK(3);   // draining partials
      if (a.no_store) continue;
      if (EPI == EPI_RESID) {   // residual: h += acc and the next tf32 planes, by 32-column slices
#pragma unroll
        for (int sl = 0; sl < EPI_COLS / 32; ++sl) {
          const int cb = nb * TBN + hc * EPI_COLS + sl * 32;
          if (cb >= a.N) continue;                              // warp-uniform
          // (TMA stores measured slower here: three serialized stores per slice)
          const size_t o = (size_t)m * a.ldc + cb;
          if (split) fold32(acc + sl * 32, sl * 32);
          store_rows32<ST_RESID>(stg, acc + sl * 32, row_ok ? a.C + o : nullptr, a.C_hi + o, a.C_lo + o, lane,
                                 a.ssq_out && row0 < a.M ? a.ssq_out + (size_t)(cb / 32) * a.ssq_ld + row0 : nullptr);
        }
        if (a.ssq_out && col0 < a.N && row0 < a.M) rms_pend = row0;   // counted at the next tile (see rms_flush)
      } else {
        static_assert(EPI == EPI_RESID || EPI_COLS % 64 == 0, "64-column epilogue blocks");
#pragma unroll
      for (int half = 0; half < EPI_COLS / 64; ++half) {
        const int cb = nb * TBN + hc * EPI_COLS + half * 64;   // first column of this 64-wide block
        if (cb >= a.N) continue;                              // warp-uniform
        float *x = acc + half * 64;   // in place: the block's partial sums are dead after it
        if (split) {
          fold32(x, half * 64);
          fold32(x + 32, half * 64 + 32);
        }
        {
#pragma unroll
          for (int j = 0; j < 64; ++j) x[j] = __fmul_rn(x[j], rs);
          if (EPI == EPI_HEAD) {   // logits through TMA bulk tensor stores (rows >= M clipped)
            tma_store32(stg, &tmC0, cb, row0, x, lane);
            tma_store32(stg, &tmC0, cb + 32, row0, x + 32, lane);
          } else if (EPI == EPI_SWIGLU) {
            // columns [cb, cb+32) are gate rows, [cb+32, cb+64) the matching up rows
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float g = x[j], up = x[32 + j];
              // silu(g) = g / (1 + e^-g) on the SFU (ex2, fast divide): ~2 ulp, same code in prefill and decode
              const float sg = __fdividef(g, __fadd_rn(1.f, tc::ex2(__fmul_rn(g, -1.44269504088896341f))));
              x[j] = __fmul_rn(sg, up);
            }
            tma_store32_planes(stg, &tmC1, &tmC2, cb / 2, row0, x, lane);   // act tf32 planes
          } else {  // EPI_QKV
            const int pos = row_ok ? a.rows.pos[m] : -1;
            const int nq = a.n_q_cols, nkv = a.n_kv_cols;
            const bool rope = cb < nq + nkv;   // q or k head (warp-uniform): RoPE on the rotate-half pairs
            size_t o = 0;
            bool ring = false, isk = false;
            if (cb < nq) {
              o = (size_t)m * a.ldc + cb;
            } else if (pos >= 0) {
              ring = true;
              isk = cb < nq + nkv;
              const int kvh = (cb - nq - (isk ? 0 : nkv)) / 64;
              o = a.ring.off(a.rows.chunk[m], a.layer, pos) + kvh * 64;
            }
            float *dh = pos < 0 ? nullptr : (ring ? (isk ? a.ring.k_hi : a.ring.v_hi) : a.C_hi) + o;
            float *dl = pos < 0 ? nullptr : (ring ? (isk ? a.ring.k_lo : a.ring.v_lo) : a.C_lo) + o;
            store_head64<true>(stg, x, pos, rope, a.rope_cos, a.rope_sin, dh, dl, lane);
          }
        }
      }
      }
      GEMM_MARK(4);   // output
    }
  }
  if ((EPI == EPI_HEAD || EPI == EPI_SWIGLU) && warp < EPI_WARPS && lane == 0)
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // bulk stores complete before exit
  tc::fence_before();
  tc::cluster_sync();          // no CTA leaves while its pair may still signal or read it
  tc::fence_after();
  if (warp == W_TMA) tc::tmem_dealloc_pair(tmem_base, TMEM_COLS);
  if (threadIdx.x == 0) {            // last CTA out resets the tile counter for the next launch
    __threadfence();
    if (atomicAdd(a.tile_ctr + 1, 1) == (int)gridDim.x - 1) {
      a.tile_ctr[0] = 0;
      a.tile_ctr[1] = 0;
      __threadfence();
    }
  }
}

// ------------------------------------------------------------- host side ---
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// fp32 [rows, cols] row-major, box [box_rows, 32 cols], 128B swizzle; cached per (ptr, shape).
const CUtensorMap *tmap_2d(const float *ptr, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  struct Key {
    const void *p; uint64_t r, c; uint32_t b;
    bool operator==(const Key &o) const { return p == o.p && r == o.r && c == o.c && b == o.b; }
  };
  struct H {
    size_t operator()(const Key &k) const {
      return std::hash<const void *>()(k.p) ^ (k.r * 0x9E3779B97F4A7C15ull) ^ (k.c << 20) ^ k.b;
    }
  };
  static std::mutex mu;
  static std::unordered_map<Key, CUtensorMap, H> cache;
  std::lock_guard<std::mutex> lk(mu);
  Key k{ptr, rows, cols, box_rows};
  auto it = cache.find(k);
  if (it != cache.end()) return &it->second;
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 4};
  cuuint32_t box[2] = {TBK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return &cache.emplace(k, m).first->second;
}

static int g_reserved_sms = 0;
void set_reserved_sms(int n) { g_reserved_sms = n; }
static int g_splitk_mode = 1;
// programmatic dependent launch of the persistent GEMM / attention grids (NC_PDL=0: off)
static const bool g_pdl = !(std::getenv("NC_PDL") && std::getenv("NC_PDL")[0] == '0');
bool pdl_enabled() { return g_pdl; }
void set_splitk_mode(int mode) { g_splitk_mode = mode; }

// Per-device state below: nc_model_load takes a device, so one process may drive several
// GPUs; each device gets its own counters / workspace (indexed by the current device).
constexpr int kMaxDevices = 64;
static int cur_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) throw std::runtime_error("device index out of range");
  return dev;
}

static int *tile_counter() {   // {next tile, CTAs done}; zero between launches
  static int *ctrs[kMaxDevices] = {};
  int *&ctr = ctrs[cur_device()];
  if (!ctr) {
    if (cudaMalloc(&ctr, 2 * sizeof(int)) != cudaSuccess) throw std::runtime_error("cudaMalloc tile counter");
    cudaMemset(ctr, 0, 2 * sizeof(int));
    cudaDeviceSynchronize();
  }
  return ctr;
}

// split-K workspace / fixup counters: grown on demand, never while a graph is captured
static bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &st);
  return st != cudaStreamCaptureStatusNone;
}
static cudaStream_t g_launch_stream = nullptr;
static float *splitk_workspace(size_t floats) {
  static float *wss[kMaxDevices] = {};
  static size_t caps[kMaxDevices] = {};
  const int dev = cur_device();
  float *&ws = wss[dev];
  size_t &cap = caps[dev];
  if (floats > cap) {
    if (capturing(g_launch_stream)) throw std::runtime_error("split-K workspace must be sized before graph capture");
    if (ws) cudaFree(ws);
    cap = std::max(floats, (size_t)1 << 20);
    if (cudaMalloc(&ws, cap * sizeof(float)) != cudaSuccess) throw std::runtime_error("cudaMalloc split-K workspace");
  }
  return ws;
}
static int *splitk_counters(size_t n) {
  static int *ctrs[kMaxDevices] = {};
  static size_t caps[kMaxDevices] = {};
  const int dev = cur_device();
  int *&ctr = ctrs[dev];
  size_t &cap = caps[dev];
  if (n > cap) {
    if (capturing(g_launch_stream)) throw std::runtime_error("split-K counters must be sized before graph capture");
    if (ctr) cudaFree(ctr);
    cap = std::max(n, (size_t)1 << 16);
    if (cudaMalloc(&ctr, cap * sizeof(int)) != cudaSuccess) throw std::runtime_error("cudaMalloc split-K counters");
    cudaMemset(ctr, 0, cap * sizeof(int));
    cudaDeviceSynchronize();
  }
  return ctr;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <int EPI, int BN>
static void launch_tc(const TcGemmArgs &a, const TcOperands &op, cudaStream_t s) {
  g_launch_stream = s;
  static unsigned long long attr = 0;
  if (first_on_device(attr)) {
    check_launch(cudaFuncSetAttribute(gemm_tc_kernel<EPI, BN, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      TileCfg<BN>::SMEM), "gemm smem attribute");
    check_launch(cudaFuncSetAttribute(gemm_tc_kernel<EPI, BN, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      TileCfg<BN>::SMEM), "gemm smem attribute");
  }
  TcGemmArgs aa = a;
  aa.a_box = a.M <= TBM ? (a.M + 7) / 8 * 8 : 0;   // rows of the A box (0: the full 128-row tile)
  const uint32_t a_rows_box = aa.a_box ? aa.a_box : TBM;
  const CUtensorMap *ah = tmap_2d(op.A_hi, op.a_rows, a.K, a_rows_box), *al = tmap_2d(op.A_lo, op.a_rows, a.K, a_rows_box);
  const CUtensorMap *bh = tmap_2d(op.B_hi, a.N, a.K, BN / 2), *bl = tmap_2d(op.B_lo, a.N, a.K, BN / 2);
  const int tiles = ((a.M + 2 * TBM - 1) / (2 * TBM)) * ((a.N + BN - 1) / BN);
  const int pairs_avail = std::max(1, (num_sms() - g_reserved_sms) / 2);
  aa.tile_ctr = tile_counter();
  // split-K when the tile grid would leave most SMs idle (decode steps); bit-identical
  // to the unsplit sum (see the kernel header); nc_debug_set_splitk(0) disables it.
  const int nspan = (a.K / TBK + KPP - 1) / KPP;
  int nsplit = 1;
  aa.sps = 0;
  // Measured at M = 8 (tools/splitk_time.py): every launch costs ~8 us fixed and each 32-wide
  // k block ~0.9 us on one pair; the fixup's fold is a few dependent L2 round trips per 32
  // columns, so splitting wins only for long k loops (down: K = 1536, 47 -> 37 us) and
  // loses at K = 576 (25 -> 33-40 us).
  // (At M = 64 -- decode of 64 chunks -- the fixup's fold, 2 rows per round trip over 32 rows
  // per warp, made the split down projection 76 us against ~37 unsplit: split only few rows.)
  if (g_splitk_mode != 0 && nspan >= SK_MIN_SPANS && nspan <= SK_MAX_SPANS && 2 * tiles <= pairs_avail &&
      a.M <= SK_MAX_ROWS && !a.no_store && a.N % 32 == 0) {
    nsplit = std::min(nspan, pairs_avail / tiles);
    aa.sps = (nspan + nsplit - 1) / nsplit;
    nsplit = (nspan + aa.sps - 1) / aa.sps;
    if (nsplit < 2) {
      nsplit = 1;
      aa.sps = 0;
    } else {
      aa.ws = splitk_workspace((size_t)nspan * a.N * a.M);
      aa.fix_ctr = splitk_counters((size_t)tiles * 2 * TileCfg<BN>::EPI_WARPS);
    }
  }
  const int pairs = std::min(tiles * nsplit, pairs_avail);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(TileCfg<BN>::THREADS);
  cfg.dynamicSmemBytes = TileCfg<BN>::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // prologue under the previous tail
  at[1].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  // output maps of the TMA-store epilogues: rows = M (clips the tile tail), 32 x 32 boxes
  const CUtensorMap *c0 = bh, *c1 = bh, *c2 = bh;
  if (EPI == EPI_HEAD) c0 = tmap_2d(a.C, (uint64_t)a.M, (uint64_t)a.ldc, 32);
  if (EPI == EPI_SWIGLU) {
    c1 = tmap_2d(a.C_hi, (uint64_t)a.M, (uint64_t)a.ldc, 32);
    c2 = tmap_2d(a.C_lo, (uint64_t)a.M, (uint64_t)a.ldc, 32);
  }
  const cudaError_t e =
      nsplit > 1 ? cudaLaunchKernelEx(&cfg, gemm_tc_kernel<EPI, BN, true>, *ah, *al, *bh, *bl, *c0, *c1, *c2, aa)
                 : cudaLaunchKernelEx(&cfg, gemm_tc_kernel<EPI, BN, false>, *ah, *al, *bh, *bl, *c0, *c1, *c2, aa);
  if (e != cudaSuccess) throw std::runtime_error(std::string("gemm_tc launch: ") + cudaGetErrorString(e));
}

void gemm_timing_report() {
#ifdef NC_GEMM_TIMING
  unsigned long long h[32];
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(h, g_gemm_clk, sizeof(h));
  const char *nm[4] = {"qkv", "resid", "swiglu", "head"};
  for (int e = 0; e < 4; ++e) {
    const unsigned long long *x = h + 8 * e;
    const double n = (double)(x[7] ? x[7] : 1);
    if (x[7])
      fprintf(stderr,
              "gemm %-6s epilogue warp per tile (cycles): wait tile %.0f | residual prefetch %.0f | wait partials "
              "%.0f | drain %.0f | output %.0f | split write %.0f | split fixup %.0f | tiles %.0f\n",
              nm[e], x[0] / n, x[1] / n, x[2] / n, x[3] / n, x[4] / n, x[5] / n, x[6] / n, n);
  }
  unsigned long long z[32] = {};
  cudaMemcpyToSymbol(g_gemm_clk, z, sizeof(z));
#endif
}

void launch_gemm_tc(GemmEpi epi, const TcGemmArgs &a, const TcOperands &op, cudaStream_t s) {
  if (a.M <= 0) return;
  if (a.K % TBK) throw std::runtime_error("tcgen05 GEMM needs K % 32 == 0");
  switch (epi) {
    // Few rows (decode steps, M <= 128): a tile's time is its k loop of pair MMAs, which
    // cost in proportion to N (128 cycles at N = 256, 64 at N = 128), so 128-wide tiles halve
    // it and double the tiles in flight.  Each output element is the same MMA sequence
    // whatever the tile width (D15; test_splitk_bit_identity compares prefill and decode).
    case EPI_QKV:
      if (a.M <= TBM) launch_tc<EPI_QKV, NC_DECODE_BN>(a, op, s);
      else launch_tc<EPI_QKV, 192>(a, op, s);   // N = 960 = 5 x 192: three heads per tile, no padding
      break;
    case EPI_RESID:
      if (a.M <= TBM) launch_tc<EPI_RESID, NC_DECODE_BN>(a, op, s);
      else launch_tc<EPI_RESID, 192>(a, op, s);   // N = 576 = 3 x 192
      break;
    case EPI_SWIGLU:
      if (a.M <= TBM) launch_tc<EPI_SWIGLU, NC_DECODE_BN>(a, op, s);
      else launch_tc<EPI_SWIGLU, 256>(a, op, s);
      break;
    case EPI_HEAD: launch_tc<EPI_HEAD, 256>(a, op, s); break;
  }
}

// ------------------------------------------------------- plane helpers ---
__global__ void split_planes_kernel(const float *__restrict__ x, float *__restrict__ hi, float *__restrict__ lo,
                                    size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float h, l;
    tc::split_tf32(x[i], h, l);
    hi[i] = h;
    lo[i] = l;
  }
}
void launch_split_planes(const float *x, float *hi, float *lo, size_t n, cudaStream_t s) {
  if (n) split_planes_kernel<<<(unsigned)std::min<size_t>((n + 255) / 256, 4096), 256, 0, s>>>(x, hi, lo, n);
}

}  // namespace nc
