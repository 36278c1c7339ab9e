// Block-window causal GQA attention on the tensor cores (
// P:482-502 retained-KV window, D9-D12), fp32-accurate via 3xTF32:
//
//   for each 64-key block b of keys [w(j), j] (blocks aligned to absolute positions):
//     S_b  = Q K_b^T              tcgen05 kind::tf32, 3 products x 8 k-steps  -> TMEM
//     m_b  = max(m_{b-1}, rowmax(S_b / 8)), P_b = exp(S_b/8 - m_b) (masked), l updated
//     O_b  = P_b V_b              tcgen05 kind::tf32 (V as an MN-major B operand) -> fresh TMEM partial
//     O   <- O * exp(m_{b-1} - m_b) + O_b     in fp32 RN registers (promotion, see k_gemm_tc.cu)
//   o = O / l
//
// One CTA per (128-row query tile of one chunk, q head); 256 threads:
//   warp 0 TMA: Q once, then K_hi/K_lo per 64-key block (3 stages, freed when S(i) completes)
//   warp 3 TMA: V_hi/V_lo per 64-key block (2 stages, freed when PV(i) completes) -- split so
//          the K loads run ahead of the late V consumer (one shared ring stalled S on the loads)
//   warp 1 tcgen05.mma issuer; warp 2 TMEM allocator;
//   warps 4-7 softmax + promotion, thread = query row (TMEM lane); P (hi/lo) goes back
//   into TMEM (tcgen05.st) and is the A operand of the PV MMA.
// Two-deep software pipeline (S, P and O partials double-buffered in TMEM): S(i)
// is issued before PV(i-1), so the softmax of block i overlaps the PV of block i-1.
// Measured: a kind::tf32 M128 MMA costs >= ~64 cycles even at N = 32, so 64-key
// blocks (S: N = 64) halve the score-MMA cost of 32-key blocks.
// A row's arithmetic depends only on its own q row and the key blocks up to its
// position (later, fully masked blocks are exact no-ops: alpha = 1, P = 0), so the
// decode step (tiles of one row) reproduces the prefill bit for bit (D15).
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
#include "tc_common.cuh"

namespace nc {

constexpr int AQ = 128;          // query rows per tile
constexpr int AK = 64;           // keys per block
constexpr int KST = 3;           // K stages
constexpr int VST = 2;           // V stages
constexpr int Q_SUB = AQ * 128;  // one [128 rows x 32 fp32] swizzled sub-tile: 16 KB
constexpr int KV_SUB = AK * 128; // one [64 keys x 32 fp32] sub-tile: 8 KB
constexpr int Q_BYTES = 4 * Q_SUB;               // hi/lo x two 32-dim halves: 64 KB
constexpr int K_STAGE = 4 * KV_SUB;              // K hi/lo x two 32-dim halves: 32 KB
constexpr int V_STAGE = 4 * KV_SUB;              // V hi/lo x two 32-dim halves: 32 KB
constexpr int ATT_SMEM = Q_BYTES + KST * K_STAGE + VST * V_STAGE + 1024 + 256;
constexpr int ATT_THREADS = 256;
// TMEM columns: S[2] (64 each) | P[2] (hi 64 + lo 64 each) | O partial[2] (64 each) = 512
constexpr uint32_t T_S = 0, T_P = 128, T_O = 384;

#ifdef NC_ATT_TIMING
// diagnostics build only: per-phase cycle sums (softmax warp 4 lane 0, MMA thread)
__device__ unsigned long long g_att_clk[16];
#define ATT_T0() const long long _t0 = clock64()
#define ATT_ACC(i, t) atomicAdd(&g_att_clk[i], (unsigned long long)(clock64() - (t)))
#else
#define ATT_T0()
#define ATT_ACC(i, t)
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

__global__ __launch_bounds__(ATT_THREADS, 1) void attn_tc_kernel(const __grid_constant__ CUtensorMap tmQh,
                                                                const __grid_constant__ CUtensorMap tmQl,
                                                                const __grid_constant__ CUtensorMap tmKh,
                                                                const __grid_constant__ CUtensorMap tmKl,
                                                                const __grid_constant__ CUtensorMap tmVh,
                                                                const __grid_constant__ CUtensorMap tmVl,
                                                                AttnTcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sQ = smem;                                  // [hi d0-31][hi d32-63][lo d0-31][lo d32-63]
  uint8_t *sK = smem + Q_BYTES;                        // per stage: Kh0 Kh1 Kl0 Kl1
  uint8_t *sV = sK + KST * K_STAGE;                     // per stage: Vh0 Vh1 Vl0 Vl1
  uint64_t *bars = reinterpret_cast<uint64_t *>(sV + VST * V_STAGE);
  uint64_t *q_full = bars, *k_full = bars + 1, *k_empty = k_full + KST, *v_full = k_empty + KST,
           *v_empty = v_full + VST;
  uint64_t *s_full = v_empty + VST, *s_empty = s_full + 2, *p_full = s_empty + 2, *p_empty = p_full + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(p_empty + 2);

  const AttnTile t = a.tiles[blockIdx.x];
  if (t.nrows <= 0) return;                        // inactive chunk in a decode step
  const int h = blockIdx.y, g = h / (a.H / a.KV);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w = wstart(t.p0, a.window, a.slide);
  const int kb0 = w / AK, kb1 = (t.p0 + t.nrows - 1) / AK;
  const int nkb = kb1 - kb0 + 1;
  const int zc = t.chunk * a.n_layers + a.layer;   // (chunk, layer) coordinate of the ring maps

  if (threadIdx.x == 0) {
    tc::tma_prefetch(&tmQh); tc::tma_prefetch(&tmKh); tc::tma_prefetch(&tmVh);
    tc::mbar_init(q_full, 1);
    for (int s = 0; s < KST; ++s) { tc::mbar_init(&k_full[s], 1); tc::mbar_init(&k_empty[s], 1); }
    for (int s = 0; s < VST; ++s) { tc::mbar_init(&v_full[s], 1); tc::mbar_init(&v_empty[s], 1); }
    for (int s = 0; s < 2; ++s) { tc::mbar_init(&s_full[s], 1); tc::mbar_init(&s_empty[s], 4); }
    for (int s = 0; s < 2; ++s) { tc::mbar_init(&p_full[s], 4); tc::mbar_init(&p_empty[s], 1); }
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
#ifdef NC_ATT_TIMING
  const long long t_cta = clock64();
#endif

  if (warp == 0) {
    if (lane == 0) {
      tc::mbar_expect_tx(q_full, Q_BYTES);
      tc::tma_load_2d(sQ, &tmQh, h * 64, t.qrow0, q_full);
      tc::tma_load_2d(sQ + Q_SUB, &tmQh, h * 64 + 32, t.qrow0, q_full);
      tc::tma_load_2d(sQ + 2 * Q_SUB, &tmQl, h * 64, t.qrow0, q_full);
      tc::tma_load_2d(sQ + 3 * Q_SUB, &tmQl, h * 64 + 32, t.qrow0, q_full);
      int st = 0;
      uint32_t ph = 0;
      for (int i = 0; i < nkb; ++i) {
        tc::mbar_wait(&k_empty[st], ph ^ 1);
        uint8_t *b = sK + st * K_STAGE;
        const int slot = ((kb0 + i) * AK) % a.ring;
        tc::mbar_expect_tx(&k_full[st], K_STAGE);
        tma_load_4d(b + 0 * KV_SUB, &tmKh, 0, g, slot, zc, &k_full[st]);
        tma_load_4d(b + 1 * KV_SUB, &tmKh, 32, g, slot, zc, &k_full[st]);
        tma_load_4d(b + 2 * KV_SUB, &tmKl, 0, g, slot, zc, &k_full[st]);
        tma_load_4d(b + 3 * KV_SUB, &tmKl, 32, g, slot, zc, &k_full[st]);
        if (++st == KST) { st = 0; ph ^= 1; }
      }
    }
  } else if (warp == 3) {
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int i = 0; i < nkb; ++i) {
        tc::mbar_wait(&v_empty[st], ph ^ 1);
        uint8_t *b = sV + st * V_STAGE;
        const int slot = ((kb0 + i) * AK) % a.ring;
        tc::mbar_expect_tx(&v_full[st], V_STAGE);
        tma_load_4d(b + 0 * KV_SUB, &tmVh, 0, g, slot, zc, &v_full[st]);
        tma_load_4d(b + 1 * KV_SUB, &tmVh, 32, g, slot, zc, &v_full[st]);
        tma_load_4d(b + 2 * KV_SUB, &tmVl, 0, g, slot, zc, &v_full[st]);
        tma_load_4d(b + 3 * KV_SUB, &tmVl, 32, g, slot, zc, &v_full[st]);
        if (++st == VST) { st = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // MMA issuer: the whole warp runs the loop on warp-uniform values; one elected
    // lane issues each tcgen05 instruction (see tc::elect_one)
    constexpr uint32_t idS = tc::idesc_tf32(AQ, AK);                  // S: K-major A and B
    constexpr uint32_t idO = tc::idesc_tf32(AQ, 64) | (1u << 16);     // O: B (V) MN-major
    tc::mbar_wait(q_full, 0);
    tc::fence_after();
    const uint64_t q_desc = tc::desc_k_sw128(tc::smem_u32(sQ));
    const uint64_t k_desc0 = tc::desc_k_sw128(tc::smem_u32(sK));
    const uint64_t v_desc0 = desc_mn_sw128_32b(tc::smem_u32(sV), KV_SUB);
    // descriptor start addresses are in 16-byte units: constant byte offsets add as (bytes >> 4)
    auto off = [](uint32_t bytes) { return (uint64_t)(bytes >> 4); };
    int st = 0;
    uint32_t ph = 0;
    uint32_t sph[2] = {0, 0}, pph[2] = {0, 0};
    int vst = 0;
    uint32_t vph = 0;
    auto issue_pv = [&](int b) {                 // O_b = P_b V_b (P from TMEM) into O partial b%2
      const int pb = b & 1;
      tc::mbar_wait(&p_full[pb], pph[pb]);
      pph[pb] ^= 1;
      tc::mbar_wait(&v_full[vst], vph);
      tc::fence_after();
      const uint32_t ph_t = tmem + T_P + pb * 128, pl_t = ph_t + 64;
      const uint64_t vd = v_desc0 + off(vst * V_STAGE);
      const uint32_t dO = tmem + T_O + pb * 64;
#pragma unroll
      for (int j = 0; j < AK / 8; ++j) {          // corrections first, hi*hi last (see k_gemm_tc.cu)
        if (tc::elect_one()) tc::mma_tf32_ts(dO, ph_t + j * 8, vd + off(2 * KV_SUB + j * 1024), idO, j != 0);
        if (tc::elect_one()) tc::mma_tf32_ts(dO, pl_t + j * 8, vd + off(j * 1024), idO, 1);
      }
#pragma unroll
      for (int j = 0; j < AK / 8; ++j)
        if (tc::elect_one()) tc::mma_tf32_ts(dO, ph_t + j * 8, vd + off(j * 1024), idO, 1);
      if (tc::elect_one()) {
        tc::mma_commit(&p_empty[pb]);             // P buffer free + O partial ready
        tc::mma_commit(&v_empty[vst]);
      }
      __syncwarp();
      if (++vst == VST) { vst = 0; vph ^= 1; }
    };
    for (int i = 0; i < nkb; ++i) {
      tc::mbar_wait(&k_full[st], ph);
      const int sb = i & 1;
      tc::mbar_wait(&s_empty[sb], sph[sb] ^ 1);
      sph[sb] ^= 1;
      tc::fence_after();
      const uint64_t kd = k_desc0 + off(st * K_STAGE);
      const uint32_t dS = tmem + T_S + sb * AK;
#pragma unroll
      for (int dsub = 0; dsub < 2; ++dsub)     // corrections first, hi*hi last (see k_gemm_tc.cu)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t adv = j * 32;
          if (tc::elect_one())
            tc::mma_tf32(dS, q_desc + off(dsub * Q_SUB + adv), kd + off((2 + dsub) * KV_SUB + adv), idS,
                         (dsub | j) != 0);
          if (tc::elect_one())
            tc::mma_tf32(dS, q_desc + off((2 + dsub) * Q_SUB + adv), kd + off(dsub * KV_SUB + adv), idS, 1);
        }
#pragma unroll
      for (int dsub = 0; dsub < 2; ++dsub)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t adv = j * 32;
          if (tc::elect_one())
            tc::mma_tf32(dS, q_desc + off(dsub * Q_SUB + adv), kd + off(dsub * KV_SUB + adv), idS, 1);
        }
      if (tc::elect_one()) {
        tc::mma_commit(&s_full[sb]);
        tc::mma_commit(&k_empty[st]);
      }
      __syncwarp();
      if (i > 0) issue_pv(i - 1);
      if (++st == KST) { st = 0; ph ^= 1; }
    }
    issue_pv(nkb - 1);
  } else if (warp >= 4) {
    const int q = warp & 3, r = q * 32 + lane;     // query row of this thread (TMEM lane)
    const bool valid = r < t.nrows;
    const int j = t.p0 + r;
    float O[64];
#pragma unroll
    for (int d = 0; d < 64; ++d) O[d] = 0.f;
    float m = -CUDART_INF_F, l = 0.f;
    float alpha_hist[2] = {1.f, 1.f};              // alpha of blocks b with b%2 == index
    uint32_t sph[2] = {0, 0}, pph[2] = {0, 0};
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    auto fold_wait = [&](int b) {                  // PV(b) complete: P buffer b%2 free, O partial b%2 ready
      const int pb = b & 1;
      tc::mbar_wait(&p_empty[pb], pph[pb]);
      pph[pb] ^= 1;
      tc::fence_after();
    };
    auto fold_apply = [&](int b) {                 // O <- O * alpha_b + O_b  (fp32 RN promotion)
      const int pb = b & 1;
      uint32_t x0[32], x1[32];
      tc::tmem_ld32(tmem + T_O + pb * 64 + lane_off, x0);
      tc::tmem_ld32(tmem + T_O + pb * 64 + lane_off + 32, x1);
      tc::tmem_wait_ld();
      const float al = alpha_hist[pb];
#pragma unroll
      for (int d = 0; d < 32; ++d) {
        O[d] = __fmaf_rn(O[d], al, __uint_as_float(x0[d]));
        O[32 + d] = __fmaf_rn(O[32 + d], al, __uint_as_float(x1[d]));
      }
    };
    auto fold = [&](int b) { fold_wait(b); fold_apply(b); };
    // scores in the log2 domain: x = S * (1/8 * log2 e); p = 2^(x - m)
    constexpr float kScale = 0.125f * 1.44269504088896341f;
    for (int i = 0; i < nkb; ++i) {
      const int sb = i & 1;
#ifdef NC_ATT_TIMING
      long long tp = clock64();
#endif
      tc::mbar_wait(&s_full[sb], sph[sb]);
#ifdef NC_ATT_TIMING
      if (threadIdx.x == 128) { atomicAdd(&g_att_clk[0], (unsigned long long)(clock64() - tp)); atomicAdd(&g_att_clk[7], 1ull); }
      tp = clock64();
#endif
      sph[sb] ^= 1;
      if (a.debug == 9) {      // diagnostics: handshakes only (no TMEM traffic, no math)
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&s_empty[sb]);
        if (i >= 2) { const int pb = i & 1; tc::mbar_wait(&p_empty[pb], pph[pb]); pph[pb] ^= 1; }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&p_full[sb]);
        continue;
      }
      tc::fence_after();
      uint32_t sr[2][32];
      tc::tmem_ld32(tmem + T_S + sb * AK + lane_off, sr[0]);
      tc::tmem_ld32(tmem + T_S + sb * AK + lane_off + 32, sr[1]);
      tc::tmem_wait_ld();
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&s_empty[sb]);
      const int key0 = (kb0 + i) * AK;
      // raw scores; masked keys -> -inf.  Max first on the raw scores (kScale > 0 and RN
      // rounding is monotone, so max(S) * kScale == max(S * kScale) exactly), as a tree.
      float x[2][32];
      if (key0 + AK - 1 <= j) {              // whole block inside the window: no masking
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
#pragma unroll
          for (int k = 0; k < 32; ++k) x[hh][k] = __uint_as_float(sr[hh][k]);
      } else {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
#pragma unroll
          for (int k = 0; k < 32; ++k)
            x[hh][k] = key0 + 32 * hh + k <= j ? __uint_as_float(sr[hh][k]) : -CUDART_INF_F;
      }
      float t[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) t[k] = fmaxf(x[0][k], x[1][k]);
#pragma unroll
      for (int w2 = 16; w2 >= 1; w2 >>= 1)
#pragma unroll
        for (int k = 0; k < w2; ++k) t[k] = fmaxf(t[k], t[k + w2]);
      const float mb = __fmul_rn(t[0], kScale);
      const float mn = fmaxf(m, mb);
      const float alpha = (mn == -CUDART_INF_F) ? 1.f : tc::ex2(__fsub_rn(m, mn));
      // p = 2^(S * kScale - m) with one FFMA per score; -inf scores give ex2(-inf) = 0.
      // (mn == -inf only when every key so far is masked: p = 0 then too.)
      const float nmn = mn == -CUDART_INF_F ? 0.f : -mn;
      float ps4[4] = {0.f, 0.f, 0.f, 0.f};   // 4 independent partial sums (latency), fixed order
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          x[hh][k] = tc::ex2(__fmaf_rn(x[hh][k], kScale, nmn));
          ps4[k & 3] = __fadd_rn(ps4[k & 3], x[hh][k]);
        }
      const float ps = __fadd_rn(__fadd_rn(ps4[0], ps4[1]), __fadd_rn(ps4[2], ps4[3]));
      l = __fmaf_rn(l, alpha, ps);
      m = mn;
#ifdef NC_ATT_TIMING
      if (threadIdx.x == 128) atomicAdd(&g_att_clk[1], (unsigned long long)(clock64() - tp));
      tp = clock64();
#endif
      // P buffer i%2 was last read by PV(i-2): wait for it, store P(i), then fold O
      // partial i-2 while the stores drain
      if (i >= 2) fold_wait(i - 2);
      const uint32_t ph_t = tmem + T_P + sb * 128 + lane_off;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          float fh, fl;
          tc::split_tf32(x[hh][k], fh, fl);
          hi[k] = __float_as_uint(fh);
          lo[k] = __float_as_uint(fl);
        }
        tc::tmem_st32(ph_t + 32 * hh, hi);
        tc::tmem_st32(ph_t + 64 + 32 * hh, lo);
      }
#ifdef NC_ATT_TIMING
      if (threadIdx.x == 128) atomicAdd(&g_att_clk[3], (unsigned long long)(clock64() - tp));
      tp = clock64();
#endif
      if (i >= 2) fold_apply(i - 2);
      alpha_hist[sb] = alpha;
      tc::tmem_wait_st();
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&p_full[sb]);
#ifdef NC_ATT_TIMING
      if (threadIdx.x == 128) atomicAdd(&g_att_clk[2], (unsigned long long)(clock64() - tp));
#endif
    }
    if (a.debug == 9) {
      for (int b = (nkb >= 2 ? nkb - 2 : 0); b < nkb; ++b) { const int pb = b & 1; tc::mbar_wait(&p_empty[pb], pph[pb]); pph[pb] ^= 1; }
    } else {
      if (nkb >= 2) fold(nkb - 2);
      fold(nkb - 1);
    }
    if (valid) {
      const size_t ob = (size_t)(t.qrow0 + r) * a.ldo + h * 64;
#pragma unroll
      for (int d = 0; d < 64; d += 4) {
        float4 hi, lo, v;
        v.x = __fdiv_rn(O[d], l); v.y = __fdiv_rn(O[d + 1], l);
        v.z = __fdiv_rn(O[d + 2], l); v.w = __fdiv_rn(O[d + 3], l);
        tc::split_tf32(v.x, hi.x, lo.x); tc::split_tf32(v.y, hi.y, lo.y);
        tc::split_tf32(v.z, hi.z, lo.z); tc::split_tf32(v.w, hi.w, lo.w);
        *reinterpret_cast<float4 *>(a.o_hi + ob + d) = hi;
        *reinterpret_cast<float4 *>(a.o_lo + ob + d) = lo;
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 2) tc::tmem_dealloc(tmem, 512);
#ifdef NC_ATT_TIMING
  if (threadIdx.x == 0) { atomicAdd(&g_att_clk[11], (unsigned long long)(clock64() - t_cta)); atomicAdd(&g_att_clk[12], 1ull); }
#endif
}

#ifdef NC_ATT_TIMING
void attn_timing_report() {
  unsigned long long h[16];
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(h, g_att_clk, sizeof(h));
  const double nb = (double)(h[7] ? h[7] : 1), nc = (double)(h[12] ? h[12] : 1);
  fprintf(stderr,
          "attn timing per block (softmax warp): wait S %.0f | max/exp/sum %.0f | fold+wait_st %.0f (wait %.0f) | "
          "pwait+split+st %.0f ; MMA thread per block: wait kv %.0f, wait s_empty %.0f, wait p_full %.0f ; per CTA %.0f "
          "cycles, %.1f blocks\n",
          h[0] / nb, h[1] / nb, h[2] / nb, h[4] / nb, h[3] / nb, h[9] / nb, h[10] / nb, h[8] / nb, h[11] / nc, nb / nc);
  cudaMemset(g_att_clk, 0, 0);
  unsigned long long z[16] = {};
  cudaMemcpyToSymbol(g_att_clk, z, sizeof(z));
}
#else
void attn_timing_report() {}
#endif

// ------------------------------------------------------------- host side ---
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
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ATT_SMEM);
    attr = true;
  }
  const uint64_t qd[2] = {(uint64_t)a.ldq, (uint64_t)a.q_rows};
  const uint32_t qb[2] = {32, AQ};
  const uint64_t kd[4] = {64, (uint64_t)a.KV, (uint64_t)a.ring, (uint64_t)a.n_chunks * a.n_layers};
  const uint32_t kbx[4] = {32, 1, AK, 1};
  const CUtensorMap *qh = tmap_nd(a.q_hi, 2, qd, qb), *ql = tmap_nd(a.q_lo, 2, qd, qb);
  const CUtensorMap *kh = tmap_nd(a.k_hi, 4, kd, kbx), *kl = tmap_nd(a.k_lo, 4, kd, kbx);
  const CUtensorMap *vh = tmap_nd(a.v_hi, 4, kd, kbx, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  const CUtensorMap *vl = tmap_nd(a.v_lo, 4, kd, kbx, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  dim3 grid(a.n_tiles, a.H);
  attn_tc_kernel<<<grid, ATT_THREADS, ATT_SMEM, s>>>(*qh, *ql, *kh, *kl, *vh, *vl, a);
}

}  // namespace nc
