// Block-window causal GQA attention on the tensor cores (
// P:482-502 retained-KV window, D9-D12), fp32-accurate via 3xTF32:
//
//   for each 128-key block b of keys [w(j), j] (blocks aligned to absolute positions;
//   the window start w(j) is a multiple of C >= 128, so no block straddles it):
//     S_b = Q K_b^T                     tcgen05 kind::tf32, 3 products x 8 k-steps, N = 128 -> TMEM
//     m  <- max(m, rowmax(S_b / 8))     (the row's two key halves exchange their maxima)
//     P_b = exp(S_b / 8 - m) (masked), l_X <- l_X alpha + rowsum(P_bX) per key half X
//     O_b = P_b V_b                     tcgen05 kind::tf32 (P from TMEM, V MN-major), K = 128 keys:
//                                       P_hi [V_hi | V_lo] as one N = 128 MMA + P_lo V_hi (N = 64)
//                                       -> one fresh TMEM partial [main | corrections] per block
//     O  <- O * alpha + (main + corr)   in fp32 RN registers (promotion, see k_gemm_tc.cu)
//   o = O / (l_A + l_B)
//
// Every row's arithmetic is the same whatever tile it is in, so decode (tiles of one row)
// reproduces prefill bit for bit (D15); later, fully masked keys are exact no-ops
// (alpha = 1, P = 0).
//
// One CTA per (128-row query tile of one chunk, q head); 384 threads:
//   warp 0  TMA: Q once (hi/lo, 64 KB), then K of each 128-key block (64 KB, one buffer)
//   warp 3  TMA: V in 64-key granules (32 KB) through a ring of 3
//   warp 1  MMA issue (whole warp, one elected lane per instruction): S(i), then PV(i-1)
//   warp 2  TMEM allocator: S (128 cols) | P_A hi,lo | P_B hi,lo (64 each) | O partial (128)
//   warps 4-7 / 8-11  softmax of key half A / B and the promotion of output dims 0-31 / 32-63,
//                     thread = query row (TMEM lane); the halves share the row max (smem)
// Measured (tools/micro): an N = 128 tf32 MMA costs 64 cycles, N = 64 costs 48-57.  Per
// 128-key block the TMEM reads -- S (64 KB) and the O partial (32 KB; 64 KB when each key
// half kept its own partial and max) by the softmax groups, P (hi twice, lo once: 192 KB) as
// the PV MMAs' A operand -- at ~64-80 B/cycle/SM are the bound: releasing each half's P
// early and double-buffering the O partial (so the next P store and the fold overlap PV)
// measured no gain (145 vs 148 TF/s) and was reverted.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <math_constants.h>

#include <algorithm>
#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>

#include "attn_tc.cuh"
#include "gemm_tc.cuh"
#include "tc_common.cuh"

namespace nc {

constexpr int AQ = 128;          // query rows per tile
constexpr int AK = 128;          // keys per block (S: one N = 128 MMA chain)
constexpr int AH = 64;           // keys per half (softmax group / PV MMA chain)
constexpr int VG = 3;            // V ring granules (64 keys each)
constexpr int Q_SUB = AQ * 128;  // one [128 rows x 32 fp32] swizzled sub-tile: 16 KB
constexpr int K_SUB = AK * 128;  // one [128 keys x 32 fp32] sub-tile: 16 KB
constexpr int KV_SUB = AH * 128; // one [64 keys x 32 fp32] sub-tile: 8 KB (TMA box, V granule part)
constexpr int Q_BYTES = 4 * Q_SUB;               // hi/lo x two 32-dim halves: 64 KB
constexpr int K_BYTES = 4 * K_SUB;               // hi/lo x two 32-dim halves: 64 KB
constexpr int V_GRAN = 4 * KV_SUB;               // V hi/lo x two 32-dim halves, 64 keys: 32 KB
constexpr int ATT_SMEM = Q_BYTES + K_BYTES + VG * V_GRAN + 1024 + 256 + 2 * 128 * 4;
constexpr int ATT_THREADS = 384;
// TMEM columns
// P half X at T_P + 128 X (hi, lo +64); the block's O partial at T_O: [P_hi V_hi | corrections]
constexpr uint32_t T_S = 0, T_P = 128, T_O = 384;

#ifdef NC_ATT_TIMING
// diagnostics build only: per-thread phase cycles accumulated in registers, flushed once per CTA
__device__ unsigned long long g_att_clk[32];
#define AT_DECL unsigned long long _acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}; long long _at = clock64()
#define AT_T(k) do { const long long _n = clock64(); _acc[k] += (unsigned long long)(_n - _at); _at = _n; } while (0)
#define AT_FLUSH(base, cond) do { if (cond) for (int _k = 0; _k < 8; ++_k) atomicAdd(&g_att_clk[(base) + _k], _acc[_k]); } while (0)
#else
#define AT_DECL do {} while (0)
#define AT_T(k) do {} while (0)
#define AT_FLUSH(base, cond) do {} while (0)
#endif

// diagnostics builds only (-DNC_ATT_ABL=k, results wrong): 1 no exponentials, 2 no O-partial
// loads in the fold, 3 no S loads, 4 no P stores, 5 no PV MMAs, 6 no S MMAs
#ifndef NC_ATT_ABL
#define NC_ATT_ABL 0
#endif

__device__ __forceinline__ int wstart(int j, int L, int C) {
  const int over = j + 1 - L;
  return over <= 0 ? 0 : C * ((over + C - 1) / C);
}

// MN-major tf32 operand descriptor.  For 32-bit MN-major operands the only
// smem layout UMMA accepts is SWIZZLE_128B_BASE32B (layout type 1: 128 B rows,
// 32 B swizzle atoms, 4-row K atoms; CUTLASS sm100_common.inl), written by TMA
// with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B.  N blocks of 32 fp32 are LBO bytes
// apart; 4-row K groups are 512 B apart (SBO).
__device__ __forceinline__ uint64_t desc_mn_sw128_32b(uint32_t saddr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)(512u >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;
  return d;
}

__device__ __forceinline__ void tma_load_4d(void *smem_dst, const CUtensorMap *m, int c0, int c1, int c2, int c3,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(tc::smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(tc::smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

constexpr int NSCH = 2;          // item schedule ring
constexpr int SCH_CONSUMERS = 10;  // V producer, MMA warp, 8 softmax warps

__global__ __launch_bounds__(ATT_THREADS, 1) void attn_tc_kernel(const __grid_constant__ CUtensorMap tmQh,
                                                                const __grid_constant__ CUtensorMap tmQl,
                                                                const __grid_constant__ CUtensorMap tmKh,
                                                                const __grid_constant__ CUtensorMap tmKl,
                                                                const __grid_constant__ CUtensorMap tmVh,
                                                                const __grid_constant__ CUtensorMap tmVl,
                                                                AttnTcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sQ = smem;                                  // [hi d0-31][hi d32-63][lo d0-31][lo d32-63], 128 rows each
  uint8_t *sK = smem + Q_BYTES;                        // same, 128 keys each (granule g at +8 KB g)
  uint8_t *sV = sK + K_BYTES;                          // VG granules: [Vh0][Vh1][Vl0][Vl1], 64 keys each
  uint64_t *bars = reinterpret_cast<uint64_t *>(sV + VG * V_GRAN);
  uint64_t *q_full = bars, *q_empty = bars + 1, *k_full = bars + 2, *k_empty = bars + 3;
  uint64_t *v_full = bars + 4, *v_empty = v_full + VG;
  uint64_t *s_full = v_empty + VG, *s_empty = s_full + 1;
  uint64_t *p_full = s_empty + 1, *pv_done = p_full + 1;   // P of both halves stored / PV done
  uint64_t *sch_full = pv_done + 1, *sch_empty = sch_full + NSCH;
  int *sch_item = reinterpret_cast<int *>(sch_empty + NSCH);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sch_item + NSCH);
  float *xmax = reinterpret_cast<float *>(tmem_slot + 4);   // [2 halves][128 rows] row-max / row-sum exchange

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = a.n_tiles * (a.heads_as_rows ? a.KV : a.H);

  if (threadIdx.x == 0) {
    tc::tma_prefetch(&tmQh); tc::tma_prefetch(&tmKh); tc::tma_prefetch(&tmVh);
    tc::mbar_init(q_full, 1); tc::mbar_init(q_empty, 1);
    tc::mbar_init(k_full, 1); tc::mbar_init(k_empty, 1);
    for (int s = 0; s < VG; ++s) { tc::mbar_init(&v_full[s], 1); tc::mbar_init(&v_empty[s], 1); }
    tc::mbar_init(s_full, 1); tc::mbar_init(s_empty, 8);
    tc::mbar_init(p_full, 8);
    tc::mbar_init(pv_done, 1);
    for (int s = 0; s < NSCH; ++s) { tc::mbar_init(&sch_full[s], 1); tc::mbar_init(&sch_empty[s], SCH_CONSUMERS); }
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  tc::pdl_launch_dependents();
  tc::pdl_wait();   // q planes and the KV ring come from the QKV GEMM

  // item -> (tile, head, geometry); every role derives the same numbers
  // item -> (tile, head, geometry); heads_as_rows: (tile, KV group), rows = the group's q heads
  const int ipt = a.heads_as_rows ? a.KV : a.H;   // items per tile
  struct Item { AttnTile t; int h, g, kb0, nkb, zc; };
  auto item_of = [&](int it) {
    Item x;
    x.t = a.tiles[it / ipt];
    if (a.heads_as_rows) {
      x.g = it % ipt;
      x.h = x.g * (a.H / a.KV);               // first q head of the group (its q row offset)
      if (x.t.nrows > 0) x.t.nrows = a.H / a.KV;
      x.t.qrow0 = x.t.qrow0 * a.H + x.h;      // row of [rows * H, 64]
    } else {
      x.h = it % a.H;
      x.g = x.h / (a.H / a.KV);
    }
    const int w = x.t.w0 >= 0 ? x.t.w0 : wstart(x.t.p0, a.window, a.slide);   // a.window = L_max
    x.kb0 = w / AK;
    const int last = a.heads_as_rows ? x.t.p0 : x.t.p0 + x.t.nrows - 1;       // the tile's last position
    x.nkb = x.t.nrows > 0 ? last / AK - x.kb0 + 1 : 0;   // 0: inactive decode chunk
    x.zc = x.t.chunk * a.n_layers + a.layer;
    return x;
  };
  // consumers: next claimed item from the schedule ring (-1 = done)
  auto next_item = [&](int jt, bool arrive) {
    const int slot = jt % NSCH;
    tc::mbar_wait(&sch_full[slot], (jt / NSCH) & 1);
    const int it = sch_item[slot];
    __syncwarp();
    if (arrive) tc::mbar_arrive(&sch_empty[slot]);
    return it;
  };

  if (warp == 0) {
    // ---------------------------------------------- scheduler + Q/K producer
    if (lane == 0) {
      int gb = 0, qi = 0;
      for (int jt = 0;; ++jt) {
        const int slot = jt % NSCH;
        tc::mbar_wait(&sch_empty[slot], ((jt / NSCH) & 1) ^ 1);
        const int claimed = atomicAdd(a.item_ctr, 1);
        const int it = claimed < n_items ? claimed : -1;
        sch_item[slot] = it;
        tc::mbar_arrive(&sch_full[slot]);
        if (it < 0) break;
        const Item x = item_of(it);
        if (x.nkb == 0) continue;
        tc::mbar_wait(q_empty, (qi & 1) ^ 1);           // all S MMAs of the previous item done
        tc::mbar_expect_tx(q_full, Q_BYTES);
        const int qc = a.heads_as_rows ? 0 : x.h * 64;   // [rows * H, 64] view: the head is the row
        tc::tma_load_2d(sQ, &tmQh, qc, x.t.qrow0, q_full);
        tc::tma_load_2d(sQ + Q_SUB, &tmQh, qc + 32, x.t.qrow0, q_full);
        tc::tma_load_2d(sQ + 2 * Q_SUB, &tmQl, qc, x.t.qrow0, q_full);
        tc::tma_load_2d(sQ + 3 * Q_SUB, &tmQl, qc + 32, x.t.qrow0, q_full);
        ++qi;
        for (int i = 0; i < x.nkb; ++i, ++gb) {
          tc::mbar_wait(k_empty, (gb & 1) ^ 1);
          const int slot_k = ((x.kb0 + i) * AK) % a.ring;   // ring is a multiple of 128: no wrap inside a block
          tc::mbar_expect_tx(k_full, K_BYTES);
#pragma unroll
          for (int gg = 0; gg < 2; ++gg) {
            tma_load_4d(sK + 0 * K_SUB + gg * KV_SUB, &tmKh, 0, x.g, slot_k + gg * AH, x.zc, k_full);
            tma_load_4d(sK + 1 * K_SUB + gg * KV_SUB, &tmKh, 32, x.g, slot_k + gg * AH, x.zc, k_full);
            tma_load_4d(sK + 2 * K_SUB + gg * KV_SUB, &tmKl, 0, x.g, slot_k + gg * AH, x.zc, k_full);
            tma_load_4d(sK + 3 * K_SUB + gg * KV_SUB, &tmKl, 32, x.g, slot_k + gg * AH, x.zc, k_full);
          }
        }
      }
    }
  } else if (warp == 3) {
    // ---------------------------------------------------------- V producer
    int st = 0;
    uint32_t ph = 0;
    for (int jt = 0;; ++jt) {
      const int it = next_item(jt, lane == 0);
      if (it < 0) break;
      const Item x = item_of(it);
      if (lane == 0)
        for (int i = 0; i < x.nkb; ++i)
#pragma unroll
          for (int gg = 0; gg < 2; ++gg) {
            tc::mbar_wait(&v_empty[st], ph ^ 1);
            uint8_t *b = sV + st * V_GRAN;
            const int slot = ((x.kb0 + i) * AK) % a.ring + gg * AH;
            tc::mbar_expect_tx(&v_full[st], V_GRAN);
            tma_load_4d(b + 0 * KV_SUB, &tmVh, 0, x.g, slot, x.zc, &v_full[st]);
            tma_load_4d(b + 1 * KV_SUB, &tmVh, 32, x.g, slot, x.zc, &v_full[st]);
            tma_load_4d(b + 2 * KV_SUB, &tmVl, 0, x.g, slot, x.zc, &v_full[st]);
            tma_load_4d(b + 3 * KV_SUB, &tmVl, 32, x.g, slot, x.zc, &v_full[st]);
            if (++st == VG) { st = 0; ph ^= 1; }
          }
      __syncwarp();
    }
  } else if (warp == 1) {
    // MMA issuer: the whole warp runs the loop on warp-uniform values; one elected
    // lane issues each tcgen05 instruction (see tc::elect_one)
    constexpr uint32_t idS = tc::idesc_tf32(AQ, AK);                  // S: K-major A and B, N = 128
    // O: B (V) MN-major.  P_hi multiplies [V_hi | V_lo] in ONE N = 128 MMA (the granule's four
    // 32-dim blocks are consecutive: an N = 128 operand), writing P_hi V_hi to T_O and P_hi V_lo
    // to T_O + 64; P_lo V_hi (N = 64) accumulates onto the latter.  An N = 64 tf32 MMA costs
    // ~55 cycles and N = 128 64 (tools/micro/mma_bench4.cu), so this is 119 cycles per k-step
    // instead of three N = 64 MMAs (165); the fold sums the two halves.
    constexpr uint32_t idO = tc::idesc_tf32(AQ, 128) | (1u << 16);
    constexpr uint32_t idC = tc::idesc_tf32(AQ, 64) | (1u << 16);
    const uint64_t q_desc = tc::desc_k_sw128(tc::smem_u32(sQ));
    const uint64_t k_desc = tc::desc_k_sw128(tc::smem_u32(sK));
    const uint64_t v_desc0 = desc_mn_sw128_32b(tc::smem_u32(sV), KV_SUB);
    auto off = [](uint32_t bytes) { return (uint64_t)(bytes >> 4); };   // descriptor address units
    int vst = 0;
    uint32_t vph = 0;
    auto issue_pv = [&](int b) {                 // O_b = P_b V_b over the block's 128 keys (b: global block)
      tc::mbar_wait(p_full, b & 1);
      const int vs0 = vst;
      tc::mbar_wait(&v_full[vst], vph);
      if (++vst == VG) { vst = 0; vph ^= 1; }
      const int vs1 = vst;
      tc::mbar_wait(&v_full[vst], vph);
      if (++vst == VG) { vst = 0; vph ^= 1; }
      tc::fence_after();
      const uint32_t dO = tmem + T_O;
      const uint64_t vd[2] = {v_desc0 + off(vs0 * V_GRAN), v_desc0 + off(vs1 * V_GRAN)};
#if NC_ATT_ABL != 5
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const uint32_t ph_t = tmem + T_P + 128 * x, pl_t = ph_t + 64;
#pragma unroll
        for (int j = 0; j < AH / 8; ++j) {
          if (tc::elect_one()) tc::mma_tf32_ts(dO, ph_t + j * 8, vd[x] + off(j * 1024), idO, (x | j) != 0);
          if (tc::elect_one()) tc::mma_tf32_ts(dO + 64, pl_t + j * 8, vd[x] + off(j * 1024), idC, 1);
        }
      }
#endif
      if (tc::elect_one()) {
        tc::mma_commit(pv_done);                   // P buffers free + O partial ready
        tc::mma_commit(&v_empty[vs0]);
        tc::mma_commit(&v_empty[vs1]);
      }
      __syncwarp();
    };
    int gb = 0, qi = 0;
    AT_DECL;
    for (int jt = 0;; ++jt) {
      const int it = next_item(jt, lane == 0);
      if (it < 0) break;
      const Item x = item_of(it);
      if (x.nkb == 0) continue;
      AT_T(6);
      tc::mbar_wait(q_full, qi & 1);
      AT_T(0);   // wait Q
      for (int i = 0; i < x.nkb; ++i, ++gb) {
        tc::mbar_wait(k_full, gb & 1);
        AT_T(1);   // wait K
        if (gb > 0) tc::mbar_wait(s_empty, (gb - 1) & 1);   // both softmax groups read S(gb-1)
        AT_T(2);   // wait s_empty
        tc::fence_after();
#if NC_ATT_ABL != 6
#pragma unroll
        for (int dsub = 0; dsub < 2; ++dsub)     // corrections first, hi*hi last (see k_gemm_tc.cu)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t adv = j * 32;
            if (tc::elect_one())
              tc::mma_tf32(tmem + T_S, q_desc + off(dsub * Q_SUB + adv), k_desc + off((2 + dsub) * K_SUB + adv),
                           idS, (dsub | j) != 0);
            if (tc::elect_one())
              tc::mma_tf32(tmem + T_S, q_desc + off((2 + dsub) * Q_SUB + adv), k_desc + off(dsub * K_SUB + adv),
                           idS, 1);
          }
#pragma unroll
        for (int dsub = 0; dsub < 2; ++dsub)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t adv = j * 32;
            if (tc::elect_one())
              tc::mma_tf32(tmem + T_S, q_desc + off(dsub * Q_SUB + adv), k_desc + off(dsub * K_SUB + adv), idS, 1);
          }
#endif
        if (tc::elect_one()) {
          tc::mma_commit(s_full);
          tc::mma_commit(k_empty);
          if (i == x.nkb - 1) tc::mma_commit(q_empty);   // Q buffer free for the next item
        }
        __syncwarp();
        AT_T(3);   // S issue
        if (i > 0) issue_pv(gb - 1);
        AT_T(4);   // PV (incl p_full/V waits)
      }
      issue_pv(gb - 1);                           // the item's last block, before the next item's S
      AT_T(4);
      ++qi;
#ifdef NC_ATT_TIMING
      _acc[7] += x.nkb;
#endif
    }
    AT_FLUSH(0, lane == 0);
  } else if (warp >= 4) {
    // ----------------------------- softmax groups (key halves) + promotion (dim halves)
    const int x = (warp - 4) >> 2;                 // key half of this softmax group = output dim half
    const int q = warp & 3, r = q * 32 + lane;     // query row of this thread (TMEM lane)
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    // scores in the log2 domain: x = S * (1/8 * log2 e); p = 2^(x - m)
    constexpr float kScale = 0.125f * 1.44269504088896341f;
    int gb = 0;
    AT_DECL;
    for (int jt = 0;; ++jt) {
      const int it = next_item(jt, lane == 0);
      if (it < 0) break;
      const Item xi = item_of(it);
      if (xi.nkb == 0) continue;
      AT_T(6);   // item gap
      const int j = a.heads_as_rows ? xi.t.p0 : xi.t.p0 + r;   // this row's position
      float O[32];                                 // output dims [32 x, 32 x + 32) of row r
#pragma unroll
      for (int d = 0; d < 32; ++d) O[d] = 0.f;
      float m = -CUDART_INF_F, l = 0.f, alpha_prev = 1.f;
      auto fold = [&](float al) {                  // O <- O * alpha + O_partial  (fp32 RN promotion)
#pragma unroll
        for (int hd = 0; hd < 2; ++hd) {           // 16 dims at a time: 32 live registers, not 64
          uint32_t x0[16], x1[16];
#if NC_ATT_ABL == 2
          for (int d = 0; d < 16; ++d) { x0[d] = __float_as_uint(al); x1[d] = 0u; }
#else
          tc::tmem_ld16(tmem + T_O + 32 * x + 16 * hd + lane_off, x0);
          tc::tmem_ld16(tmem + T_O + 64 + 32 * x + 16 * hd + lane_off, x1);
          tc::tmem_wait_ld();
#endif
#pragma unroll
          for (int d = 0; d < 16; ++d)
            O[16 * hd + d] = __fmaf_rn(O[16 * hd + d], al, __fadd_rn(__uint_as_float(x0[d]), __uint_as_float(x1[d])));
        }
      };
      // a warp whose 32 rows are all past the tile's rows (decode tiles hold 1-3 rows; ragged
      // tails) skips its TMEM loads, exponentials, P stores and folds -- the MMAs compute its
      // rows from whatever P holds, and those rows are never stored (rows are independent) --
      // but keeps every barrier arrival
      const bool idle = q * 32 >= xi.t.nrows;
      for (int i = 0; i < xi.nkb; ++i, ++gb) {
        tc::mbar_wait(s_full, gb & 1);
        AT_T(0);   // wait S
        tc::fence_after();
        const int key0 = (xi.kb0 + i) * AK + AH * x;
        float xs[2][32];
        float mloc = -CUDART_INF_F;
        if (!idle) {
          uint32_t sr[2][32];
#if NC_ATT_ABL == 3
          for (int k = 0; k < 32; ++k) { sr[0][k] = __float_as_uint(0.01f * (k ^ lane)); sr[1][k] = __float_as_uint(0.02f * (k ^ lane)); }
#else
          tc::tmem_ld32(tmem + T_S + 64 * x + lane_off, sr[0]);
          tc::tmem_ld32(tmem + T_S + 64 * x + lane_off + 32, sr[1]);
          tc::tmem_wait_ld();
#endif
          if (key0 + AH - 1 <= j) {              // whole half inside the window: no masking
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
#pragma unroll
              for (int k = 0; k < 32; ++k) xs[hh][k] = __uint_as_float(sr[hh][k]);
          } else {
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
#pragma unroll
              for (int k = 0; k < 32; ++k)
                xs[hh][k] = key0 + 32 * hh + k <= j ? __uint_as_float(sr[hh][k]) : -CUDART_INF_F;
          }
          // max on the raw scores (kScale > 0, RN monotone: exact), as a tree
          float tt[32];
#pragma unroll
          for (int k = 0; k < 32; ++k) tt[k] = fmaxf(xs[0][k], xs[1][k]);
#pragma unroll
          for (int w2 = 16; w2 >= 1; w2 >>= 1)
#pragma unroll
            for (int k = 0; k < w2; ++k) tt[k] = fmaxf(tt[k], tt[k + w2]);
          mloc = __fmul_rn(tt[0], kScale);
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(s_empty);
        // the row's two halves exchange their maxima
        xmax[128 * x + r] = mloc;
        named_bar(3, 256);
        const float mb = fmaxf(xmax[r], xmax[128 + r]);   // same operand order in both halves
        named_bar(3, 256);                         // both read before the next exchange writes
        float alpha = 1.f;
        if (!idle) {
          const float mn = fmaxf(m, mb);
          alpha = (mn == -CUDART_INF_F) ? 1.f : tc::ex2(__fsub_rn(m, mn));
          const float nmn = mn == -CUDART_INF_F ? 0.f : -mn;
          float ps4[4] = {0.f, 0.f, 0.f, 0.f};   // 4 independent partial sums (latency), fixed order
#pragma unroll
          for (int hh = 0; hh < 2; ++hh)
#pragma unroll
            for (int k = 0; k < 32; ++k) {
#if NC_ATT_ABL == 1
              xs[hh][k] = __fmaf_rn(xs[hh][k], kScale, nmn);
#else
              xs[hh][k] = tc::ex2(__fmaf_rn(xs[hh][k], kScale, nmn));   // masked: ex2(-inf) = 0
#endif
              ps4[k & 3] = __fadd_rn(ps4[k & 3], xs[hh][k]);
            }
          const float ps = __fadd_rn(__fadd_rn(ps4[0], ps4[1]), __fadd_rn(ps4[2], ps4[3]));
          l = __fmaf_rn(l, alpha, ps);
          m = mn;
        }
        AT_T(1);   // S load + max/exp/sum
        // the P buffers and the O partial were last used by PV(gb-1): wait for it (within the
        // item; the previous item's last PV was waited for at its end), store P, fold
        if (i >= 1) {
          tc::mbar_wait(pv_done, (gb - 1) & 1);
          tc::fence_after();
        }
        AT_T(2);   // wait PV(i-1)
        if (!idle) {
          const uint32_t ph_t = tmem + T_P + 128 * x + lane_off;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh)
#pragma unroll
            for (int qq = 0; qq < 2; ++qq) {   // 16 columns at a time: 32 live plane registers
              uint32_t hi[16], lo[16];
#pragma unroll
              for (int k = 0; k < 16; ++k) {
                float fh, fl;
                tc::split_tf32(xs[hh][16 * qq + k], fh, fl);
                hi[k] = __float_as_uint(fh);
                lo[k] = __float_as_uint(fl);
              }
#if NC_ATT_ABL == 4
              if (hi[0] == 0x7fffffffu && lo[1] == 0x7fffffffu) tc::tmem_st16(ph_t + 32 * hh + 16 * qq, hi);
#else
              tc::tmem_st16(ph_t + 32 * hh + 16 * qq, hi);
              tc::tmem_st16(ph_t + 64 + 32 * hh + 16 * qq, lo);
#endif
            }
          if (i >= 1) fold(alpha_prev);
          tc::tmem_wait_st();
        }
        alpha_prev = alpha;
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(p_full);
        AT_T(3);   // P store + fold
      }
      tc::mbar_wait(pv_done, (gb - 1) & 1);
      AT_T(4);   // wait last PV
      tc::fence_after();
      if (!idle) fold(alpha_prev);
      // row sum: the two halves' partial sums (same order in both), then this half's dims
      xmax[128 * x + r] = l;
      named_bar(3, 256);
      const float lt = __fadd_rn(xmax[r], xmax[128 + r]);
      named_bar(3, 256);
      const float rl = __frcp_rn(lt);              // o = O * (1 / l): one reciprocal per row
      const bool row_ok = r < xi.t.nrows;
      const size_t ob = a.heads_as_rows ? (size_t)(xi.t.qrow0 + r) * 64 + 32 * x
                                        : (size_t)(xi.t.qrow0 + r) * a.ldo + xi.h * 64 + 32 * x;
      if (row_ok) {
#pragma unroll
        for (int d = 0; d < 32; d += 4) {
          float4 hi, lo, v;
          v.x = __fmul_rn(O[d], rl);
          v.y = __fmul_rn(O[d + 1], rl);
          v.z = __fmul_rn(O[d + 2], rl);
          v.w = __fmul_rn(O[d + 3], rl);
          tc::split_tf32(v.x, hi.x, lo.x); tc::split_tf32(v.y, hi.y, lo.y);
          tc::split_tf32(v.z, hi.z, lo.z); tc::split_tf32(v.w, hi.w, lo.w);
          *reinterpret_cast<float4 *>(a.o_hi + ob + d) = hi;
          *reinterpret_cast<float4 *>(a.o_lo + ob + d) = lo;
        }
      }
      AT_T(5);   // merge + output
#ifdef NC_ATT_TIMING
      _acc[7] += xi.nkb;
#endif
    }
    AT_FLUSH(x == 0 ? 8 : 16, lane == 0 && q == 0);
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 2) tc::tmem_dealloc(tmem, 512);
  if (threadIdx.x == 0) {            // last CTA out resets the item counter for the next launch
    __threadfence();
    if (atomicAdd(a.item_ctr + 1, 1) == (int)gridDim.x - 1) {
      a.item_ctr[0] = 0;
      a.item_ctr[1] = 0;
      __threadfence();
    }
  }
}

// ------------------------------------------------------------- host side ---
void attn_timing_report() {
#ifdef NC_ATT_TIMING
  unsigned long long h[32];
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(h, g_att_clk, sizeof(h));
  const char *nm[3] = {"MMA   ", "soft A", "soft B"};
  const char *ph[3][7] = {{"wait Q", "wait K", "wait s_empty", "S issue", "PV", "-", "item gap"},
                          {"wait S", "ld+exp", "wait PV", "store+fold", "wait last PV", "merge+out", "item gap"},
                          {"wait S", "ld+exp", "wait PV", "store+fold", "wait last PV", "merge+out", "item gap"}};
  for (int w = 0; w < 3; ++w) {
    const unsigned long long *x = h + 8 * w;
    const double n = (double)(x[7] ? x[7] : 1);
    fprintf(stderr, "attn %s per block:", nm[w]);
    for (int k = 0; k < 7; ++k) fprintf(stderr, " %s %.0f |", ph[w][k], x[k] / n);
    fprintf(stderr, " (blocks %.0f)\n", n);
  }
  unsigned long long z[32] = {};
  cudaMemcpyToSymbol(g_att_clk, z, sizeof(z));
#endif
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn2() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess || !p)
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

static const CUtensorMap *tmap_nd(const float *ptr, int rank, const uint64_t *dims, const uint32_t *box,
                                 CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  struct Key {
    const void *p; int r; uint64_t d[4]; uint32_t b[4]; int sw;
    bool operator==(const Key &o) const {
      return p == o.p && r == o.r && sw == o.sw && !memcmp(d, o.d, sizeof(d)) && !memcmp(b, o.b, sizeof(b));
    }
  };
  struct H {
    size_t operator()(const Key &k) const {
      size_t x = std::hash<const void *>()(k.p);
      for (int i = 0; i < 4; ++i) x = x * 1315423911u ^ k.d[i] ^ ((size_t)k.b[i] << 32);
      return x;
    }
  };
  static std::mutex mu;
  static std::unordered_map<Key, CUtensorMap, H> cache;
  std::lock_guard<std::mutex> lk(mu);
  Key k{ptr, rank, {0, 0, 0, 0}, {0, 0, 0, 0}, (int)swz};
  for (int i = 0; i < rank; ++i) { k.d[i] = dims[i]; k.b[i] = box[i]; }
  auto it = cache.find(k);
  if (it != cache.end()) return &it->second;
  CUtensorMap m;
  cuuint64_t gd[4], gs[3];
  cuuint32_t bx[4], es[4] = {1, 1, 1, 1};
  uint64_t stride = 4;
  for (int i = 0; i < rank; ++i) {
    gd[i] = dims[i];
    bx[i] = box[i];
    if (i > 0) gs[i - 1] = stride;
    stride *= dims[i];
  }
  CUresult r = encode_fn2()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<float *>(ptr), gd, gs, bx, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled (attention) failed: " + std::to_string((int)r));
  return &cache.emplace(k, m).first->second;
}

void launch_attention_tc(const AttnTcArgs &a, cudaStream_t s) {
  if (a.n_tiles <= 0) return;
  static unsigned long long attr = 0;
  if (first_on_device(attr))
    check_launch(cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ATT_SMEM),
                 "attention smem attribute");
  const uint64_t qd[2] = {a.heads_as_rows ? 64ull : (uint64_t)a.ldq,
                          a.heads_as_rows ? (uint64_t)a.q_rows * a.H : (uint64_t)a.q_rows};
  const uint32_t qb[2] = {32, AQ};
  if (a.heads_as_rows && a.ldq != a.H * 64) throw std::runtime_error("heads_as_rows needs ldq == H * 64");
  const uint64_t kd[4] = {64, (uint64_t)a.KV, (uint64_t)a.ring, (uint64_t)a.n_chunks * a.n_layers};
  const uint32_t kbx[4] = {32, 1, AH, 1};   // 64-key granules (a 128-key K block is two)
  const CUtensorMap *qh = tmap_nd(a.q_hi, 2, qd, qb), *ql = tmap_nd(a.q_lo, 2, qd, qb);
  const CUtensorMap *kh = tmap_nd(a.k_hi, 4, kd, kbx), *kl = tmap_nd(a.k_lo, 4, kd, kbx);
  const CUtensorMap *vh = tmap_nd(a.v_hi, 4, kd, kbx, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  const CUtensorMap *vl = tmap_nd(a.v_lo, 4, kd, kbx, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  // {next item, CTAs done}, zero between launches (last CTA resets); one per device, since
  // one process may drive models on several GPUs (nc_model_load takes a device)
  constexpr int kMaxDevices = 64;
  static int *ctrs[kMaxDevices] = {};
  static int sms[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) throw std::runtime_error("device index out of range");
  int *&ctr = ctrs[dev];
  int &n_sms = sms[dev];
  if (!ctr) {
    if (cudaMalloc(&ctr, 2 * sizeof(int)) != cudaSuccess) throw std::runtime_error("cudaMalloc attention counter");
    cudaMemset(ctr, 0, 2 * sizeof(int));
    cudaDeviceSynchronize();
    cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  AttnTcArgs aa = a;
  aa.item_ctr = ctr;
  const int grid = std::min(a.n_tiles * (a.heads_as_rows ? a.KV : a.H), n_sms);   // persistent: one CTA per SM claims items
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(ATT_THREADS);
  cfg.dynamicSmemBytes = ATT_SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  check_launch(cudaLaunchKernelEx(&cfg, attn_tc_kernel, *qh, *ql, *kh, *kl, *vh, *vl, aa), "attention launch");
}

}  // namespace nc
