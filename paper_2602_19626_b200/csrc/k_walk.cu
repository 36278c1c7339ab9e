// The per-token vocab-row CDF kernel ("walk") and
// the N-gram precompute kernel.
//
// Per token i of a chunk (alg:compress P:246-267; SURVEY.md §8(c) canonical loop):
//   u_v  = z_v / tau + (f32) b_v                            (D16a)
//   pt_v = exp(u_v - max u) / sum exp(u - max u)             (softmax, fp32)
//   p_v  = pt_v                                    (i < W or N-gram off)
//        = w_l pt_v + w_n p_ng(v)                  (otherwise)
//        p_ng(v) = a0/(N+V) (c(v)+1) + sum_k a_k cnt_k(v)   (closed form of P:361-374)
//   c_v  = max(1, floor((double) p_v (T - V)))     (exact product, D5)
//   residual T - sum c added to c_argmax (lowest index on ties, D4; signed, D6)
//   encode: (cum_t, freq_t);  decode: group prefix scan + WNC target search (D27)
//   b_v -= alpha (pt_v - [v = t])  in f64            (D17)
//   mixer: lw += eta [ln pt_t, ln p_ng(t)], renormalise (D24-D26)
//   unigram c(t)++ and the order-1..4 context tables    (D18-D23)
//
// One 1024-thread CTA per chunk walks the chunk's tokens in order; thread t owns
// the float4 groups g = t, t + 1024, ... of the vocab row (coalesced loads).
//
// Compression knows every token, so the N-gram (which depends on tokens only)
// runs ahead in `ngram_pre_kernel` (one warp per chunk) and hands the walk a
// merged sparse list per token; the walk's main pass then also folds in the
// NEXT token's softmax statistics (u_{i+1} = z_{i+1} + b after this token's
// update), so a token costs one pass over the row and one block reduction.
// Decompression runs the same N-gram functions inline and the same element
// arithmetic; every float op is an explicit round-to-nearest intrinsic and
// every reduction has a fixed tree, so the decoder reproduces the encoder's
// counts bit for bit (D15).
#include <algorithm>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <cuda_runtime.h>
#include <math_constants.h>

#include <type_traits>

#include "tc_common.cuh"
#include "walk.cuh"

namespace nc {

// Threads per walk CTA, by cluster size (a token's logits stay in registers, so the thread
// count sets the register budget): 512 (16 warps, 128 registers) for the 4- and 8-CTA
// clusters of many-chunk containers -- more warps hide the per-element latency (A/B on one
// box: config3 step -0.6 %, config2 -1 %) -- and 384 (12 warps, 168 registers) for the
// 16-CTA single-stream cluster, whose CS-sized combine spills at 128 registers (512 threads:
// config2 with one chunk 119 -> 135 ms).  The thread count fixes the reduction order, and
// the cluster size is a function of V and the container's chunk count only, so encoder and
// decoder always agree.
constexpr int walk_threads(int cs) { return (cs == 4 || cs == 8) ? 512 : 384; }
constexpr int WT = 384;          // the quantize debug kernel's block
constexpr int NW = WT / 32;

struct WalkSmem {
  // per-warp partials, padded to 32 with identities (set once) so warp 0 reduces all lanes
  float red_m[32], red_s[32];
  unsigned long long red_sum[32], red_cum[32];
  float red_bv[32]; int red_bi[32]; uint32_t red_bc[32];
  uint32_t scan[32];
  float red_h[32];   // N-gram entropy partials (skip test)
  // per-token broadcast scalars
  float M, invS, a0f;
  int mix, tok, argmax, nsp;
  long long resid;
  unsigned long long target, cum_t, freq_t;
  float pt_t, png_t, p_t;
  __align__(16) NgTok lists[2];   // sparse N-gram fixups of the current / next token
};

// ------------------------------------------------------------ elementwise ---
__device__ __forceinline__ float walk_u(float z, double b, float inv_tau) { return __fmaf_rn(z, inv_tau, (float)b); }
// b <- b - alpha (p~ - 1[t]) in f64 (D17), as two steps: b - alpha p~ for every id (one DFMA),
// then + alpha for the coded token only (b_tok_fix, one thread) -- the per-element select of
// p~ - 1 was ~8 % of the walk's instructions.  Encoder and decoder both use exactly this.
__device__ __forceinline__ double b_step(double b, float pt, double alpha) {
  return __fma_rn(-alpha, (double)pt, b);
}
// the coded token's correction, applied to component j of its float4 group (b01 = ids 0-1,
// b23 = ids 2-3)
__device__ __forceinline__ void b_tok_fix(double2 &b01, double2 &b23, int j, double alpha) {
  if (j == 0) b01.x = __dadd_rn(b01.x, alpha);
  else if (j == 1) b01.y = __dadd_rn(b01.y, alpha);
  else if (j == 2) b23.x = __dadd_rn(b23.x, alpha);
  else b23.y = __dadd_rn(b23.y, alpha);
}
// c = max(1, floor(p * (T - V))) with the EXACT product (D5), in fp32 only:
// T - V < 2^24 is exact in fp32; q = floor(rn(p * TmV)) is off by at most one,
// and the sign of the exact residual p * TmV - q is that of fma(p, TmV, -q).
// floor() and the integer conversion run on the FMA/ALU pipes, no SFU-class
// FRND/F2I: for 0 <= x < 2^23, x + 2^23 rounded down holds floor(x) in its low
// mantissa bits (exact); every float >= 2^23 is an integer, read from its bits.
// rANS stream word at bit position bp (a multiple of 32; big-endian; 0 past the end, D39)
__device__ __forceinline__ unsigned long long ans_word(const uint8_t *s, unsigned long long bp,
                                                       unsigned long long nb) {
  if (bp + 32 > nb) return 0ull;
  const uint8_t *q = s + (bp >> 3);
  return ((unsigned long long)q[0] << 24) | ((unsigned long long)q[1] << 16) | ((unsigned long long)q[2] << 8) | q[3];
}
__device__ __forceinline__ uint32_t quant(float p, float TmV) {
  const float x = __fmul_rn(p, TmV);
  const float t = __fadd_rd(x, 8388608.f);
  const uint32_t xb = __float_as_uint(x);
  const bool small = x < 8388608.f;
  const float q = small ? __fsub_rn(t, 8388608.f) : x;
  const uint32_t qi = small ? __float_as_uint(t) - 0x4B000000u : ((xb & 0x7FFFFFu) | 0x800000u) << ((xb >> 23) - 150u);
  const float r = __fmaf_rn(p, TmV, -q);
  const int qs = (int)qi + (r < 0.f ? -1 : (r >= 1.f ? 1 : 0));
  return qs < 1 ? 1u : (uint32_t)qs;
}
__device__ __forceinline__ float lg2f(float x) {   // log2 on the SFU (lg2.approx.ftz)
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// f64 ln and exp for the mixer (one thread, on the per-token critical path): short fixed
// sequences instead of the libdevice routines (~2x fewer dependent f64 instructions),
// accurate to ~1e-15 relative -- the oracle's fp64 mixer is the reference (1e-4 p bar).
// ln x, x > 0 normal: x = m 2^e, m in [sqrt(1/2), sqrt(2)), ln x = e ln 2 + 2 atanh(s),
// s = (m - 1) / (m + 1), |s| <= 0.1716: the odd series to s^19 (next term < 1e-17)
__device__ __forceinline__ double ln_f64(double x) {
  const long long b = __double_as_longlong(x);
  int e = (int)((b >> 52) & 0x7ff) - 1023;
  double m = __longlong_as_double((b & 0x000fffffffffffffLL) | 0x3ff0000000000000LL);
  if (m > 1.4142135623730951) { m = __dmul_rn(m, 0.5); ++e; }
  const double s = __dmul_rn(__dadd_rn(m, -1.0), __drcp_rn(__dadd_rn(m, 1.0)));
  const double s2 = __dmul_rn(s, s);
  double p = 1.0 / 19;
  p = __fma_rn(p, s2, 1.0 / 17); p = __fma_rn(p, s2, 1.0 / 15); p = __fma_rn(p, s2, 1.0 / 13);
  p = __fma_rn(p, s2, 1.0 / 11); p = __fma_rn(p, s2, 1.0 / 9); p = __fma_rn(p, s2, 1.0 / 7);
  p = __fma_rn(p, s2, 1.0 / 5); p = __fma_rn(p, s2, 1.0 / 3);
  const double at2 = __fma_rn(__dmul_rn(2.0 * s, s2), p, 2.0 * s);   // 2 atanh(s)
  constexpr double LN2_HI = 6.93147180369123816490e-01, LN2_LO = 1.90821492927058770002e-10;
  return __fma_rn((double)e, LN2_HI, __fma_rn((double)e, LN2_LO, at2));
}
// e^-a for a >= 0: a = n ln 2 + r, |r| <= ln2 / 2, e^-r by its Taylor series to r^14
// (error < 1e-17), times 2^-n built in the exponent; 0 past a = 700 (w ~ 1e-304, 0 in fp32)
__device__ __forceinline__ double exp_neg_f64(double a) {
  if (a > 700.0) return 0.0;
  constexpr double LN2_HI = 6.93147180369123816490e-01, LN2_LO = 1.90821492927058770002e-10;
  const double n = rint(__dmul_rn(a, 1.4426950408889634));
  const double r = __fma_rn(-n, LN2_LO, __fma_rn(-n, LN2_HI, a));   // a - n ln 2
  double p = 1.0 / 87178291200.0;                                       // 1/14!
  p = __fma_rn(p, -r, 1.0 / 6227020800.0); p = __fma_rn(p, -r, 1.0 / 479001600.0);
  p = __fma_rn(p, -r, 1.0 / 39916800.0); p = __fma_rn(p, -r, 1.0 / 3628800.0);
  p = __fma_rn(p, -r, 1.0 / 362880.0); p = __fma_rn(p, -r, 1.0 / 40320.0); p = __fma_rn(p, -r, 1.0 / 5040.0);
  p = __fma_rn(p, -r, 1.0 / 720.0); p = __fma_rn(p, -r, 1.0 / 120.0); p = __fma_rn(p, -r, 1.0 / 24.0);
  p = __fma_rn(p, -r, 1.0 / 6.0); p = __fma_rn(p, -r, 0.5); p = __fma_rn(p, -r, 1.0); p = __fma_rn(p, -r, 1.0);
  return __dmul_rn(p, __longlong_as_double((long long)(1023 - (int)n) << 52));   // n <= 1010: normal 2^-n
}
// exp on the SFU (ex2.approx; relative error ~1e-6 for the |x| < 30 used here)
__device__ __forceinline__ float fexp(float x) { return tc::ex2(__fmul_rn(x, 1.44269504088896341f)); }
// Warp (max, sum-of-exp) statistics: the max first (order-free, one redux on an order-
// preserving integer key), then every lane's sum rescaled once to it and added through a
// fixed xor tree (identical in every lane) -- one exponential per lane instead of two per
// tree level.  Compression and decompression both use exactly this.
__device__ __forceinline__ uint32_t fkey(float x) {
  const uint32_t b = __float_as_uint(x);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}
__device__ __forceinline__ void ms_warp(float &tm, float &ts) {
  const float M = fkey_inv(__reduce_max_sync(0xffffffffu, fkey(tm)));
  float s = (tm == -CUDART_INF_F) ? 0.f : __fmul_rn(ts, fexp(__fsub_rn(tm, M)));
#pragma unroll
  for (int o = 16; o; o >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
  tm = M;
  ts = s;
}
// quant() for a float4 group: the x < 2^23 path for all four, and the x >= 2^23
// path (only an element with p > 1/2 reaches it) behind one warp vote, so the
// common case issues no instructions for it.  Same values as quant().
__device__ __forceinline__ void quant4(const float p[4], float TmV, uint32_t cv[4]) {
  float x[4], q[4];
  uint32_t qi[4];
  bool big = false;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    x[j] = __fmul_rn(p[j], TmV);
    const float t = __fadd_rd(x[j], 8388608.f);
    q[j] = __fsub_rn(t, 8388608.f);
    qi[j] = __float_as_uint(t) - 0x4B000000u;
    big |= !(x[j] < 8388608.f);
  }
  if (__any_sync(__activemask(), big)) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (!(x[j] < 8388608.f)) {
        const uint32_t xb = __float_as_uint(x[j]);
        q[j] = x[j];
        qi[j] = ((xb & 0x7FFFFFu) | 0x800000u) << ((xb >> 23) - 150u);
      }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float r = __fmaf_rn(p[j], TmV, -q[j]);
    const int qs = (int)qi[j] + (r < 0.f ? -1 : (r >= 1.f ? 1 : 0));
    cv[j] = qs < 1 ? 1u : (uint32_t)qs;
  }
}
// Per-thread softmax statistics of one token from its register-resident u values
// (groups k < ng): m = max u, then s = sum 2^(u log2 e - m log2 e) as four
// element-position partial sums (over groups in order) added as (s0 + s1) + (s2 + s3):
// independent chains for latency.  Encoder and decoder both use exactly this.
constexpr int NGMAX = 8;   // float4 groups per thread at most (V / CS <= 4 * NGMAX * WT)
template <int NGM>
__device__ __forceinline__ void ms_regs(const float (&u)[NGM][4], int ng, float &tm, float &ts) {
  constexpr float LOG2E = 1.44269504088896341f;
  float m4[4] = {-CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F};
#pragma unroll
  for (int k = 0; k < NGM; ++k)
    if (k < ng) {
#pragma unroll
      for (int j = 0; j < 4; ++j) m4[j] = fmaxf(m4[j], u[k][j]);
    }
  tm = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
  float s4[4] = {0.f, 0.f, 0.f, 0.f};
  if (tm != -CUDART_INF_F) {
    const float nb = -__fmul_rn(tm, LOG2E);
#pragma unroll
    for (int k = 0; k < NGM; ++k)
      if (k < ng) {
#pragma unroll
        for (int j = 0; j < 4; ++j) s4[j] = __fadd_rn(s4[j], tc::ex2(__fmaf_rn(u[k][j], LOG2E, nb)));
      }
  }
  ts = __fadd_rn(__fadd_rn(s4[0], s4[1]), __fadd_rn(s4[2], s4[3]));
}
// ms_regs that also leaves e = 2^(u log2 e - m log2 e) in place of u (m = the thread's max):
// the token's probabilities are then p~ = e * (2^((m - M) log2 e) / S) -- one exponential per
// element instead of two (compression); the decoder forms the same e from u and m (tc_pt)
template <int NGM>
__device__ __forceinline__ void ms_regs_e(float (&u)[NGM][4], int ng, float &tm, float &ts) {
  constexpr float LOG2E = 1.44269504088896341f;
  float m4[4] = {-CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F};
#pragma unroll
  for (int k = 0; k < NGM; ++k)
    if (k < ng) {
#pragma unroll
      for (int j = 0; j < 4; ++j) m4[j] = fmaxf(m4[j], u[k][j]);
    }
  tm = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
  float s4[4] = {0.f, 0.f, 0.f, 0.f};
  if (tm != -CUDART_INF_F) {
    const float nb = -__fmul_rn(tm, LOG2E);
#pragma unroll
    for (int k = 0; k < NGM; ++k)
      if (k < ng) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          u[k][j] = tc::ex2(__fmaf_rn(u[k][j], LOG2E, nb));
          s4[j] = __fadd_rn(s4[j], u[k][j]);
        }
      }
  }
  ts = __fadd_rn(__fadd_rn(s4[0], s4[1]), __fadd_rn(s4[2], s4[3]));
}
// the thread's rescale of its e values to probabilities: 2^((m - M) log2 e) / S
__device__ __forceinline__ float pt_scale(float m_thread, float M, float invS) {
  return __fmul_rn(tc::ex2(__fmul_rn(__fsub_rn(m_thread, M), 1.44269504088896341f)), invS);
}
// p~ of one element from its u, the thread's max and scale (decoder; = e * scale of the encoder)
__device__ __forceinline__ float pt_from_u(float u, float m_thread, float scale) {
  return __fmul_rn(tc::ex2(__fmaf_rn(u, 1.44269504088896341f, -__fmul_rn(m_thread, 1.44269504088896341f))), scale);
}
// p = w_l pt + w_n (a0f (c+1) + add); c (unigram count < 2^24) held exactly in fp32
// skip (confidence-based LLM skip): p = p_ng
__device__ __forceinline__ float mix_p(float pt, float a0f, float cuv, float add, float wl, float wn, float &png,
                                       bool skip = false) {
  png = __fmaf_rn(a0f, __fadd_rn(cuv, 1.f), add);
  return skip ? png : __fmaf_rn(wl, pt, __fmul_rn(wn, png));
}
constexpr float kSkipTauBits = 1.5f;   // "H(p_ng) < tau bits, with tau = 1.5"
struct Best {
  float v; int i; uint32_t c;
};
__device__ __forceinline__ void best_merge(Best &a, float v, int i, uint32_t c) {
  if (v > a.v || (v == a.v && i < a.i)) { a.v = v; a.i = i; a.c = c; }
}
// warp argmax with best_merge's order (largest p, then smallest id), order-free:
// p >= 0 compares as its bit pattern; "none" (v < 0) ranks below every p.
__device__ __forceinline__ Best best_warp(Best b) {
  const uint32_t key = b.v < 0.f ? 0u : __float_as_uint(b.v) + 1u;
  const uint32_t kmax = __reduce_max_sync(0xffffffffu, key);
  const bool cand = key == kmax;
  const uint32_t imin = __reduce_min_sync(0xffffffffu, cand ? (uint32_t)b.i : 0xffffffffu);
  const int src = __ffs(__ballot_sync(0xffffffffu, cand && (uint32_t)b.i == imin)) - 1;
  return Best{__shfl_sync(0xffffffffu, b.v, src), __shfl_sync(0xffffffffu, b.i, src),
              __shfl_sync(0xffffffffu, b.c, src)};
}

// ------------------------------------------------------------------ N-gram ---
__device__ __forceinline__ unsigned long long fnv_ctx(int k, const uint32_t *hist) {
  unsigned long long h = 0xcbf29ce484222325ull;
  const unsigned long long P = 0x100000001b3ull;
  h ^= (unsigned long long)(k & 255); h *= P;
  for (int j = 4 - k; j < 4; ++j) {
    const uint32_t t = hist[j];
#pragma unroll
    for (int by = 0; by < 4; ++by) { h ^= (t >> (8 * by)) & 255u; h *= P; }
  }
  return h ? h : 1ull;
}

// warp-parallel linear probe; returns record index or -1 (and the first empty slot).
__device__ __forceinline__ int ng_probe(const unsigned long long *keys, const uint32_t *vals, uint32_t hcap,
                                        unsigned long long key, int lane, uint32_t *empty_slot) {
  const uint32_t base = (uint32_t)(key ^ (key >> 32)) & (hcap - 1);
  for (uint32_t p = 0; p < hcap; p += 32) {
    const uint32_t idx = (base + p + lane) & (hcap - 1);
    const unsigned long long kk = keys[idx];
    const unsigned m = __ballot_sync(0xffffffffu, kk == key);
    if (m) return (int)vals[__shfl_sync(0xffffffffu, idx, __ffs(m) - 1)];
    const unsigned e = __ballot_sync(0xffffffffu, kk == 0ull);
    if (e) { *empty_slot = __shfl_sync(0xffffffffu, idx, __ffs(e) - 1); return -1; }
  }
  *empty_slot = 0xffffffffu;
  return -1;
}

// Prediction for token i (one warp): a0f and the merged sparse list, ids in order
// of first appearance over k = 1..4 then slots, adds accumulated in that order.
// `spadd` (global, zero) and `bitmap` (zero) are scratch and are left zero.
__device__ void ng_predict_warp(const WalkArgs &a, int c, uint32_t i, const uint32_t *hist, float *spadd,
                                uint32_t *bitmap, NgTok *out, int lane) {
  double mu[kMaxOrders + 1], beta[kMaxOrders + 1];
  int rec[kMaxOrders + 1];
  for (int k = 1; k <= kMaxOrders; ++k) { mu[k] = 1.0; beta[k] = 0.0; rec[k] = -1; }
  for (int k = 1; k <= (int)a.orders; ++k) {
    if (i < (uint32_t)k) continue;
    const size_t tb = (size_t)c * kMaxOrders + (k - 1);
    uint32_t es;
    const int r = ng_probe(a.ng_keys + tb * a.hcap, a.ng_vals + tb * a.hcap, a.hcap, fnv_ctx(k, hist), lane, &es);
    if (r < 0) continue;
    const NgRecord *R = a.ng_recs + tb * a.rcap + r;
    const uint32_t ns = R->nslot;
    uint32_t s = 0;
    if ((uint32_t)lane < ns) s += R->cnt[lane];
    if ((uint32_t)lane + 32 < ns) s += R->cnt[lane + 32];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const double n = (double)R->n;
    const double lam = __ddiv_rn(n, __dadd_rn(n, 5.0));
    mu[k] = __dsub_rn(1.0, __ddiv_rn(__dmul_rn(lam, (double)s), n));
    beta[k] = __ddiv_rn(lam, n);
    rec[k] = r;
  }
  double a0 = 1.0;
  for (int k = 1; k <= (int)a.orders; ++k) a0 = __dmul_rn(a0, mu[k]);
  uint32_t nout = 0;
  for (int k = 1; k <= (int)a.orders; ++k) {
    if (rec[k] < 0) continue;
    double ak = beta[k];
    for (int j = k + 1; j <= (int)a.orders; ++j) ak = __dmul_rn(ak, mu[j]);
    const size_t tb = (size_t)c * kMaxOrders + (k - 1);
    const NgRecord *R = a.ng_recs + tb * a.rcap + rec[k];
    const uint32_t ns = R->nslot;
    for (uint32_t s0 = 0; s0 < ns; s0 += 32) {
      const uint32_t s = s0 + lane;
      const bool act = s < ns;
      uint32_t tk = 0;
      bool first = false;
      if (act) {
        tk = R->tok[s];
        const float add = (float)__dmul_rn(ak, (double)R->cnt[s]);
        const uint32_t bit = 1u << (tk & 31);
        first = !(atomicOr(&bitmap[tk >> 5], bit) & bit);
        spadd[tk] = first ? add : __fadd_rn(spadd[tk], add);     // ids are unique within one order
      }
      const unsigned fm = __ballot_sync(0xffffffffu, act && first);
      if (act && first) out->tok[nout + __popc(fm & ((1u << lane) - 1))] = tk;
      nout += __popc(fm);
    }
    __syncwarp();
    __threadfence_block();
  }
  for (uint32_t j = lane; j < nout; j += 32) {
    const uint32_t tk = out->tok[j];
    out->add[j] = spadd[tk];
    spadd[tk] = 0.f;
    bitmap[tk >> 5] = 0u;
  }
  if (lane == 0) {
    out->n = nout;
    out->a0f = (float)__ddiv_rn(a0, (double)i + (double)a.V);
  }
  __syncwarp();
}

// Count update with token t after token i (one warp): P:375-387, D19-D22.
__device__ void ng_update_warp(const WalkArgs &a, int c, uint32_t i, const uint32_t *hist, uint32_t t,
                               WalkState *st, int lane) {
  for (int k = 1; k <= (int)a.orders; ++k) {
    if (i < (uint32_t)k) continue;
    const size_t tb = (size_t)c * kMaxOrders + (k - 1);
    unsigned long long *keys = a.ng_keys + tb * a.hcap;
    uint32_t *vals = a.ng_vals + tb * a.hcap;
    const unsigned long long key = fnv_ctx(k, hist);
    uint32_t es = 0xffffffffu;
    int r = ng_probe(keys, vals, a.hcap, key, lane, &es);
    if (r < 0) {
      const uint32_t used = st->nrec[k - 1];
      if (used >= a.cap || used >= a.rcap || es == 0xffffffffu) continue;   // capacity freeze (D22)
      r = (int)used;
      if (lane == 0) {
        st->nrec[k - 1] = used + 1;
        keys[es] = key; vals[es] = (uint32_t)r;
        a.ng_recs[tb * a.rcap + r].n = 0;
        a.ng_recs[tb * a.rcap + r].nslot = 0;
      }
      __syncwarp();
      __threadfence_block();
    }
    NgRecord *R = a.ng_recs + tb * a.rcap + r;
    const uint32_t ns = R->nslot;
    const bool h0 = (uint32_t)lane < ns && R->tok[lane] == t;
    const bool h1 = (uint32_t)lane + 32 < ns && R->tok[lane + 32] == t;
    const unsigned m0 = __ballot_sync(0xffffffffu, h0), m1 = __ballot_sync(0xffffffffu, h1);
    if (m0 | m1) {
      if (h0) R->cnt[lane] += 1;
      if (h1) R->cnt[lane + 32] += 1;
    } else if (ns < kSlots) {
      if (lane == 0) { R->tok[ns] = t; R->cnt[ns] = 1; R->nslot = ns + 1; }
    } else {   // evict the lowest count, ties -> lowest slot (D21)
      uint32_t bcnt = R->cnt[lane], bidx = lane;
      if (R->cnt[lane + 32] < bcnt) { bcnt = R->cnt[lane + 32]; bidx = lane + 32; }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const uint32_t oc = __shfl_xor_sync(0xffffffffu, bcnt, o), oi = __shfl_xor_sync(0xffffffffu, bidx, o);
        if (oc < bcnt || (oc == bcnt && oi < bidx)) { bcnt = oc; bidx = oi; }
      }
      if (lane == 0) { R->tok[bidx] = t; R->cnt[bidx] = 1; }
    }
    if (lane == 0) R->n += 1;
    __syncwarp();
    __threadfence_block();
  }
}

__device__ __forceinline__ void ng_hist_push(WalkState *st, uint32_t t) {
  st->hist[0] = st->hist[1]; st->hist[1] = st->hist[2]; st->hist[2] = st->hist[3]; st->hist[3] = t;
}

// ---------------------------------------------------- N-gram precompute ---
// Compression knows every token, so the N-gram side of the walk (predictions and count
// updates) runs ahead of it.  Per token it is a chain of dependent L2 round
// trips (hash probe -> record), so latency is what matters: each chunk gets FOUR warps,
// warp k-1 owning order k's table.  Per token i:
//   A  warp k: probe context k (hist) once -- the same key serves the prediction and the
//      update -- and stage the record (n, nslot, tok[64], cnt[64]) in shared memory;
//      mu_k, beta_k as in ng_predict_warp (f64)
//   -- chunk barrier --
//   B  warp 0: a0, a_k and the merged sparse list from the staged records, in the same
//      order and with the same arithmetic as ng_predict_warp (first appearance over
//      k = 1..4 then slots, adds accumulated in k order), into the ring entry
//   C  warp k: the count update of order k from the staged record, writes only (same
//      insert / increment / append / evict rules as ng_update_warp)
//   -- chunk barrier --
// so a token costs ~3 round trips instead of ~40 (one warp doing all orders twice).
// The decoder runs ng_predict_warp / ng_update_warp inline on the same tables; both
// produce identical lists and table states (round-trip tests).
constexpr int NGC = 4;           // chunks per CTA (5 warps each: 4 orders + the merge warp)
constexpr int NGWC = 5;          // warps per chunk
constexpr int NG_HASH = 512;     // merge position hash (>= 2 x kMaxSparse)
struct NgSlot {                  // one token's staged lookups (double-buffered by token parity)
  uint32_t tok[kMaxOrders][kSlots], cnt[kMaxOrders][kSlots];
  uint32_t ns[kMaxOrders];
  int r[kMaxOrders];
  double mu[kMaxOrders], beta[kMaxOrders];
};
struct NgStage {
  NgSlot slot[2];
  uint32_t hkey[NG_HASH], hpos[NG_HASH];
  uint32_t mtok[kMaxSparse];
  float madd[kMaxSparse];
};
__host__ __device__ constexpr size_t ng_group_bytes(uint32_t V) {   // one chunk's shared memory, 16 B aligned
  return (sizeof(NgStage) + ((V + 31) / 32) * 4 + 15) / 16 * 16;
}
__device__ __forceinline__ uint32_t ng_hslot(uint32_t tk) { return (tk * 2654435761u) >> (32 - 9); }

// Per token i (slot b = i & 1):
//   order warps k-1 (k = 1..4): probe context k once -- the key serves the prediction and the
//     update -- stage the record in slot b; chunk barrier; then the count update from what
//     they staged (writes only), and on to token i + 1 (staging into the other slot)
//   merge warp (the fifth): after the barrier, the merged prediction of token i from slot b
//     into the ring entry -- concurrently with the order warps' update and next lookups
// One barrier per token: slot b is rewritten (token i + 2) only after the barrier of token
// i + 1, which the merge warp reaches after finishing token i.
__global__ void ngram_pre_kernel(WalkArgs a) {
  extern __shared__ __align__(16) uint8_t ng_raw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int lc = w / NGWC, kw = w % NGWC, k = kw + 1;   // chunk in CTA; order (kw < 4) or merge warp (kw == 4)
  const bool merger = kw == kMaxOrders;
  const int e = blockIdx.x * NGC + lc;
  if (e >= a.n_entries) return;                       // whole 5-warp groups exit together
  const uint32_t nbw = (a.V + 31) / 32;
  NgStage &S = *reinterpret_cast<NgStage *>(ng_raw + (size_t)lc * ng_group_bytes(a.V));
  uint32_t *bitmap = reinterpret_cast<uint32_t *>(&S + 1);
  const int bar = 1 + lc;
  constexpr int BAR_THREADS = 32 * NGWC;
  const int c = a.chunk_of[e], count = a.count[e];
  WalkState *st = a.st + c;
  const bool active = !merger && k <= (int)a.orders;
  const size_t tb = (size_t)c * kMaxOrders + (merger ? 0 : kw);
  unsigned long long *keys = a.ng_keys + tb * a.hcap;
  uint32_t *vals = a.ng_vals + tb * a.hcap;
  NgRecord *recs = a.ng_recs + tb * a.rcap;
  if (merger) {
    for (uint32_t x = lane; x < nbw; x += 32) bitmap[x] = 0u;
    for (int x = lane; x < NG_HASH; x += 32) S.hkey[x] = 0xffffffffu;
  }
  uint32_t hist[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) hist[j] = st->hist[j];
  uint32_t nrec = merger ? 0u : st->nrec[kw];
  const uint32_t i0 = st->ng_i;
  const int64_t toff = a.tok_off[c];
  asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(BAR_THREADS) : "memory");
  for (int it = 0; it < count; ++it) {
    const uint32_t i = i0 + it;
    NgSlot &Q = S.slot[i & 1];
    if (!merger) {
      const uint32_t t = a.tokens[toff + i];   // issued early: needed only by the update
      // ---- lookup + stage (order k)
      int r = -1;
      uint32_t es = 0xffffffffu, ns = 0, n = 0;
      unsigned long long key = 0;
      uint32_t t0 = 0, t1 = 0, c0 = 0, c1 = 0;
      if (active && i >= (uint32_t)k) {
        key = fnv_ctx(k, hist);
        r = ng_probe(keys, vals, a.hcap, key, lane, &es);
        uint32_t s = 0;
        if (r >= 0) {
          const NgRecord *R = recs + r;
          ns = R->nslot;
          n = R->n;
          t0 = R->tok[lane]; t1 = R->tok[lane + 32]; c0 = R->cnt[lane]; c1 = R->cnt[lane + 32];
          Q.tok[kw][lane] = t0; Q.tok[kw][lane + 32] = t1;
          Q.cnt[kw][lane] = c0; Q.cnt[kw][lane + 32] = c1;
          if ((uint32_t)lane < ns) s += c0;
          if ((uint32_t)lane + 32 < ns) s += c1;
#pragma unroll
          for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        }
        if (lane == 0) {
          Q.r[kw] = r; Q.ns[kw] = ns;
          if (r >= 0) {
            const double nd = (double)n;
            const double lam = __ddiv_rn(nd, __dadd_rn(nd, 5.0));
            Q.mu[kw] = __dsub_rn(1.0, __ddiv_rn(__dmul_rn(lam, (double)s), nd));
            Q.beta[kw] = __ddiv_rn(lam, nd);
          } else {
            Q.mu[kw] = 1.0;
            Q.beta[kw] = 0.0;
          }
        }
      } else if (lane == 0) {
        Q.r[kw] = -1; Q.ns[kw] = 0; Q.mu[kw] = 1.0; Q.beta[kw] = 0.0;
      }
      asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(BAR_THREADS) : "memory");
      // ---- count update of order k with token t (writes only, from this warp's registers)
      if (active && i >= (uint32_t)k) {
        bool fresh = false;
        if (r < 0) {
          if (!(nrec >= a.cap || nrec >= a.rcap || es == 0xffffffffu)) {   // capacity freeze (D22)
            r = (int)nrec;
            fresh = true;
            if (lane == 0) {
              keys[es] = key;
              vals[es] = (uint32_t)r;
            }
            ++nrec;
          }
        }
        if (r >= 0) {
          NgRecord *R = recs + r;
          if (fresh) { ns = 0; n = 0; }
          const bool h0 = (uint32_t)lane < ns && t0 == t;
          const bool h1 = (uint32_t)lane + 32 < ns && t1 == t;
          const unsigned m0 = __ballot_sync(0xffffffffu, h0), m1 = __ballot_sync(0xffffffffu, h1);
          if (m0 | m1) {
            if (h0) R->cnt[lane] = c0 + 1;
            if (h1) R->cnt[lane + 32] = c1 + 1;
          } else if (ns < kSlots) {
            if (lane == 0) { R->tok[ns] = t; R->cnt[ns] = 1; R->nslot = ns + 1; }
          } else {   // evict the lowest count, ties -> lowest slot (D21)
            uint32_t bcnt = c0, bidx = lane;
            if (c1 < bcnt) { bcnt = c1; bidx = lane + 32; }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
              const uint32_t oc = __shfl_xor_sync(0xffffffffu, bcnt, o), oi = __shfl_xor_sync(0xffffffffu, bidx, o);
              if (oc < bcnt || (oc == bcnt && oi < bidx)) { bcnt = oc; bidx = oi; }
            }
            if (lane == 0) { R->tok[bidx] = t; R->cnt[bidx] = 1; }
          }
          if (lane == 0) R->n = n + 1;
        }
      }
      __syncwarp();
      __threadfence_block();
      hist[0] = hist[1]; hist[1] = hist[2]; hist[2] = hist[3]; hist[3] = t;
    } else {
      asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(BAR_THREADS) : "memory");
      // ---- merged prediction of token i (same order and arithmetic as ng_predict_warp)
      NgTok *out = a.ng_pre + (size_t)c * a.ng_ring + (i % a.ng_ring);
      if (i >= a.warmup) {
        double a0 = 1.0;
        for (int kk = 1; kk <= (int)a.orders; ++kk) a0 = __dmul_rn(a0, Q.mu[kk - 1]);
        uint32_t nout = 0;
        for (int kk = 1; kk <= (int)a.orders; ++kk) {
          if (Q.r[kk - 1] < 0) continue;
          double ak = Q.beta[kk - 1];
          for (int j = kk + 1; j <= (int)a.orders; ++j) ak = __dmul_rn(ak, Q.mu[j - 1]);
          const uint32_t ns = Q.ns[kk - 1];
          for (uint32_t s0 = 0; s0 < ns; s0 += 32) {
            const uint32_t sl = s0 + lane;
            const bool act = sl < ns;
            uint32_t tk = 0, pos = 0;
            bool first = false;
            float add = 0.f;
            if (act) {
              tk = Q.tok[kk - 1][sl];
              add = (float)__dmul_rn(ak, (double)Q.cnt[kk - 1][sl]);
              const uint32_t bit = 1u << (tk & 31);
              first = !(atomicOr(&bitmap[tk >> 5], bit) & bit);
            }
            const unsigned fm = __ballot_sync(0xffffffffu, act && first);
            if (act && first) {
              pos = nout + __popc(fm & ((1u << lane) - 1));
              S.mtok[pos] = tk;
              S.madd[pos] = add;
              uint32_t hs = ng_hslot(tk);
              while (atomicCAS(&S.hkey[hs], 0xffffffffu, tk) != 0xffffffffu) hs = (hs + 1) & (NG_HASH - 1);
              S.hpos[hs] = pos;
            }
            __syncwarp();
            if (act && !first) {   // seen in a lower order (ids are unique within one order)
              uint32_t hs = ng_hslot(tk);
              while (S.hkey[hs] != tk) hs = (hs + 1) & (NG_HASH - 1);
              pos = S.hpos[hs];
              S.madd[pos] = __fadd_rn(S.madd[pos], add);
            }
            nout += __popc(fm);
            __syncwarp();
          }
        }
        __syncwarp();
        for (uint32_t j = lane; j < nout; j += 32) {
          const uint32_t tk = S.mtok[j];
          out->tok[j] = tk;
          out->add[j] = S.madd[j];
          bitmap[tk >> 5] = 0u;
        }
        for (int x = lane; x < NG_HASH; x += 32) S.hkey[x] = 0xffffffffu;
        if (lane == 0) {
          out->n = nout;
          out->a0f = (float)__ddiv_rn(a0, (double)i + (double)a.V);
        }
        __syncwarp();
      } else if (lane == 0) {
        out->n = 0;
        out->a0f = 0.f;
      }
    }
  }
  if (!merger && lane == 0) st->nrec[kw] = nrec;
  if (kw == 0 && lane == 0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) st->hist[j] = hist[j];
    st->ng_i = i0 + (uint32_t)count;
  }
}

void launch_ngram_precompute(const WalkArgs &a, cudaStream_t s) {
  if (a.n_entries <= 0) return;
  const size_t smem = (size_t)NGC * ng_group_bytes(a.V);
  static unsigned long long attr = 0;
  if (first_on_device(attr))
    check_launch(cudaFuncSetAttribute(ngram_pre_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024),
                 "ngram smem attribute");
  ngram_pre_kernel<<<(a.n_entries + NGC - 1) / NGC, 32 * NGWC * NGC, smem, s>>>(a);
  check_launch(cudaGetLastError(), "ngram precompute launch");
}

// ---------------------------------------------------------------- walk ---
// A chunk's vocab row is split over a thread-block cluster of CS CTAs: CTA r
// owns ids [r V/CS, (r+1) V/CS) and keeps their f64 bias, unigram counts and
// N-gram fixups in shared memory; thread t of a CTA owns the local float4
// groups t, t + 1024, ...  Per token the CTAs exchange their partial
// reductions through distributed shared memory (one cluster barrier per token
// in compression) and every CTA combines them in rank order, so all CTAs hold
// identical scalars and decode (same code, same order) is bit-identical.

struct Xch {                  // one CTA's per-token partials, read by the whole cluster
  unsigned long long sum, cum;
  float bv; int bi; uint32_t bc;
  float m, s;                 // softmax statistics partial
  int has_tok; float pt_t, png_t, p_t; uint32_t freq_t;
  int found, t; unsigned long long cum_t, fq_t; float fpt, fpng, fp;
  uint32_t pad;
};
// the cluster's (max, sum) partials in rank order: max, then the rescaled sums added in order
template <int CS>
__device__ __forceinline__ void ms_cluster(const Xch *x, float &M, float &S) {
  float m = x[0].m;
#pragma unroll
  for (int r = 1; r < CS; ++r) m = fmaxf(m, x[r].m);
  float e[CS];
#pragma unroll
  for (int r = 0; r < CS; ++r) e[r] = x[r].m == -CUDART_INF_F ? 0.f : __fmul_rn(x[r].s, fexp(__fsub_rn(x[r].m, m)));
  float sum = e[0];
#pragma unroll
  for (int r = 1; r < CS; ++r) sum = __fadd_rn(sum, e[r]);
  M = m;
  S = sum;
}
constexpr int XW = sizeof(Xch) / 4;
constexpr int XWE = 14;   // compression reads only the prefix sum .. freq_t of a slot
static_assert(offsetof(Xch, freq_t) + 4 == 4 * XWE, "Xch compression prefix");
static_assert(sizeof(Xch) % 4 == 0, "Xch words");

__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cl_ld(const void *local_smem, uint32_t rank) {
  uint32_t a = tc::smem_u32(local_smem), r, v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(r) : "memory");
  return v;
}

#ifdef NC_WALK_TIMING
// diagnostics build only: encode-loop phase cycle sums (thread 0 of rank-0 CTAs)
__device__ unsigned long long g_walk_clk[8];
#define WALK_MARK(k)                                                                            \
  do {                                                                                          \
    if (tid == 0 && rank == 0) {                                                                \
      const long long _n = clock64();                                                           \
      atomicAdd(&g_walk_clk[k], (unsigned long long)(_n - _wt));                                \
      _wt = _n;                                                                                 \
    }                                                                                           \
  } while (0)
#else
#define WALK_MARK(k) do {} while (0)
#endif

// NGM: float4 groups per thread the kernel is compiled for (>= the launch's; the register
// arrays are sized by it -- 3 at V / CS = 6,144 keeps the 128-register budget spill-free).
// The arithmetic does not depend on it (loops run over the thread's ng groups).
template <int CS, int NGM, int WT_>
__global__ __launch_bounds__(WT_, 1) void walk_cl_kernel(WalkArgs a) {
  constexpr int WT = WT_;
  static_assert(CS <= 32, "the combine reads one cluster slot per lane");
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ WalkSmem sm;
  __shared__ Xch xs[2];            // own slots (token parity)
  __shared__ Xch xin[2][CS];       // the cluster's slots (token parity): gathered (decode) or pushed (encode)
  __shared__ float xh[2][CS];      // the cluster's N-gram entropy partials (token parity), pushed
  __shared__ double s_lw[2];
  __shared__ float s_w[2];
  __shared__ uint32_t s_i;
  __shared__ uint32_t s_tok[2048];   // compression: the chunk's tokens, refilled every 1,024 (ring)
  __shared__ float s_mth[WT];        // decompression: every thread's max of its u (pt_from_u of any group)
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t rank = CS > 1 ? cl_rank() : 0u;
  const int e = blockIdx.x / CS;
  const int c = a.chunk_of[e];
  const int row0 = a.row0[e], count = a.count[e];
  const uint32_t V = a.V, Vc = V / CS, vb = rank * Vc;
  const int Gc = (int)(Vc / 4);
  const int ng = tid < Gc ? (Gc - 1 - tid) / WT + 1 : 0;   // my groups tid + k WT, k < ng <= NGM
  double *b_s = reinterpret_cast<double *>(dsm);
  float *cu_s = reinterpret_cast<float *>(b_s + Vc);   // unigram counts, exact (< 2^24) as fp32
  float *sp_s = reinterpret_cast<float *>(cu_s + Vc);
  uint32_t *bitmap = reinterpret_cast<uint32_t *>(sp_s + Vc);
  uint32_t *gsum = bitmap + (Vc + 31) / 32;
  WalkState *st = a.st + c;
  const int64_t toff = a.tok_off[c];   // hoisted: the per-token loads below depend on it
  double *b_g = a.b + (size_t)c * V + vb;
  uint32_t *cu_g = a.cu + (size_t)c * V + vb;
  const bool use_ng = a.flags & 1u, use_head = a.flags & 2u;
  const bool use_skip = use_ng && (a.flags & 4u);   // confidence-based LLM skip
  const bool enc = a.mode == 0;
  const uint64_t T = 1ull << a.cdf_bits;
  const float TmV = (float)(T - V);
  const float inv_tau = a.inv_tau;
  const unsigned long long HALF = 1ull << 31, QTR = 1ull << 30;

  // ---- load this CTA's slice of the chunk state into shared memory
  for (uint32_t v = tid; v < Vc; v += WT) {
    b_s[v] = use_head ? b_g[v] : 0.0;
    cu_s[v] = use_ng ? (float)cu_g[v] : 0.f;
    sp_s[v] = 0.f;
  }
  for (uint32_t w = tid; w < (Vc + 31) / 32; w += WT) bitmap[w] = 0u;
  if (tid < 32) {
    sm.red_m[tid] = -CUDART_INF_F; sm.red_s[tid] = 0.f; sm.red_sum[tid] = 0ull; sm.red_cum[tid] = 0ull;
    sm.red_bv[tid] = -1.f; sm.red_bi[tid] = 0x7fffffff; sm.red_bc[tid] = 0u; sm.scan[tid] = 0u;
    sm.red_h[tid] = 0.f;
  }
  if (tid == 0) {
    s_lw[0] = st->lw[0]; s_lw[1] = st->lw[1];
    s_w[0] = st->wl; s_w[1] = st->wn;
    s_i = st->i;
    if (!enc && st->i == 0 && rank == 0) {
      const uint8_t *s = a.streams + a.stream_off[c];
      const unsigned long long nb = a.stream_bits[c];
      if (a.coder == 1) {   // rANS (D39): x = the first two words (the encoder's flush)
        st->value = (ans_word(s, 0, nb) << 32) | ans_word(s, 32, nb);
        st->bitpos = 64; st->low = 0; st->high = 0; st->pend = 0;
      } else {              // WNC: prime the decoder with 32 bits
        unsigned long long v = 0;
        for (int k = 0; k < 32; ++k) v = 2 * v + ((unsigned long long)k < nb ? (s[k >> 3] >> (7 - (k & 7))) & 1u : 0u);
        st->low = 0; st->high = 0xFFFFFFFFull; st->value = v; st->bitpos = 32; st->pend = 0;
      }
    }
  }
  __syncthreads();
  if (CS > 1) cl_sync();

  auto load_u = [&](const float *z, int g, float u[4]) {
    const float4 z4 = reinterpret_cast<const float4 *>(z + vb)[g];
    const double2 b01 = reinterpret_cast<const double2 *>(b_s)[2 * g];
    const double2 b23 = reinterpret_cast<const double2 *>(b_s)[2 * g + 1];
    u[0] = walk_u(z4.x, b01.x, inv_tau); u[1] = walk_u(z4.y, b01.y, inv_tau);
    u[2] = walk_u(z4.z, b23.x, inv_tau); u[3] = walk_u(z4.w, b23.y, inv_tau);
  };
  auto prob4 = [&](const float *z, int g, float mth, float scale, float wl, float wn, float a0f, int mix, bool skip,
                   float pt[4],
                   float png[4], float p[4]) {
    float u[4];
    load_u(z, g, u);
#pragma unroll
    for (int j = 0; j < 4; ++j) pt[j] = pt_from_u(u[j], mth, scale);
    if (!mix) {
#pragma unroll
      for (int j = 0; j < 4; ++j) { png[j] = 0.f; p[j] = pt[j]; }
      return;
    }
    const float4 c4 = reinterpret_cast<const float4 *>(cu_s)[g];
    const float cc[4] = {c4.x, c4.y, c4.z, c4.w};
    const uint32_t bits = (bitmap[g >> 3] >> ((g & 7) * 4)) & 15u;
    const float4 s4 = bits ? reinterpret_cast<const float4 *>(sp_s)[g] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float sa[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) p[j] = mix_p(pt[j], a0f, cc[j], sa[j], wl, wn, png[j], skip);
  };
  // CTA reduction of (m, s) into warp 0 (all lanes hold the CTA value)
  auto cta_ms = [&](float &tm, float &ts) {
    ms_warp(tm, ts);
    if (lane == 0) { sm.red_m[wid] = tm; sm.red_s[wid] = ts; }
    __syncthreads();
    if (wid == 0) {
      tm = sm.red_m[lane]; ts = sm.red_s[lane];
      ms_warp(tm, ts);
    }
  };
  auto cta_counts = [&](unsigned long long s1, unsigned long long s2, Best bb, unsigned long long &o1,
                        unsigned long long &o2, Best &ob) {   // call after the caller's __syncthreads scheme
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      best_merge(bb, __shfl_xor_sync(0xffffffffu, bb.v, o), __shfl_xor_sync(0xffffffffu, bb.i, o),
                 __shfl_xor_sync(0xffffffffu, bb.c, o));
    }
    if (lane == 0) { sm.red_sum[wid] = s1; sm.red_cum[wid] = s2; sm.red_bv[wid] = bb.v; sm.red_bi[wid] = bb.i; sm.red_bc[wid] = bb.c; }
    __syncthreads();
    if (wid == 0) {
      s1 = sm.red_sum[lane]; s2 = sm.red_cum[lane];
      Best b2{sm.red_bv[lane], sm.red_bi[lane], sm.red_bc[lane]};
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        best_merge(b2, __shfl_xor_sync(0xffffffffu, b2.v, o), __shfl_xor_sync(0xffffffffu, b2.i, o),
                   __shfl_xor_sync(0xffffffffu, b2.c, o));
      }
      o1 = s1; o2 = s2; ob = b2;
    }
  };
  // warp 0: copy every CTA's slot `par` into xin[] (DSMEM), then lane 0 combines
  auto gather = [&](int par) {
    for (int r = 0; r < CS; ++r) {
      uint32_t *dst = reinterpret_cast<uint32_t *>(&xin[par][r]);
      const uint32_t *src = reinterpret_cast<const uint32_t *>(&xs[par]);
      for (int w = lane; w < XW; w += 32) dst[w] = CS > 1 ? cl_ld(src + w, (uint32_t)r) : src[w];
    }
    __syncwarp();
  };
  auto scatter_list = [&](uint32_t i) {   // warp 0: fixups of token i inside this CTA's range
    const NgTok &L = sm.lists[i & 1];
    const int mix = (use_ng && i >= a.warmup) ? 1 : 0;
    const int n = mix ? (int)L.n : 0;
    for (int j = lane; j < n; j += 32) {
      const uint32_t tk = L.tok[j];
      if (tk >= vb && tk < vb + Vc) {
        sp_s[tk - vb] = L.add[j];
        atomicOr(&bitmap[(tk - vb) >> 5], 1u << ((tk - vb) & 31));
      }
    }
    if (lane == 0) { sm.mix = mix; sm.nsp = n; sm.a0f = mix ? L.a0f : 0.f; }
  };
  auto clear_list = [&](uint32_t i) {
    const NgTok &L = sm.lists[i & 1];
    for (int j = lane; j < sm.nsp; j += 32) {
      const uint32_t tk = L.tok[j];
      if (tk >= vb && tk < vb + Vc) { sp_s[tk - vb] = 0.f; bitmap[(tk - vb) >> 5] = 0u; }
    }
  };
  auto prefetch_pre = [&](uint32_t i) {
    const char *src = reinterpret_cast<const char *>(a.ng_pre + (size_t)c * a.ng_ring + (i % a.ng_ring));
    char *dst = reinterpret_cast<char *>(&sm.lists[i & 1]);
    for (int ofs = lane * 16; ofs < (int)sizeof(NgTok); ofs += 32 * 16)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst + ofs)),
                   "l"(src + ofs)
                   : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto prefetch_wait = [&]() { asm volatile("cp.async.wait_all;" ::: "memory"); };
  // H(p_ng) in bits of the current token (skip test; D32).  All threads call it,
  // with the token's N-gram fixups scattered; compression and decompression run this same
  // arithmetic: per thread over its groups (four element-position partial sums), lane 0 of
  // a fixed warp xor tree, the same over the warps, then the cluster's CTAs in rank order.
  auto ng_entropy = [&](int par, float a0f) -> float {
    float h4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < NGM; ++k)
      if (k < ng) {
        const int g = tid + k * WT;
        const float4 c4 = reinterpret_cast<const float4 *>(cu_s)[g];
        const uint32_t bits = (bitmap[g >> 3] >> ((g & 7) * 4)) & 15u;
        const float4 s4 = bits ? reinterpret_cast<const float4 *>(sp_s)[g] : make_float4(0.f, 0.f, 0.f, 0.f);
        const float cc[4] = {c4.x, c4.y, c4.z, c4.w}, sa[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float q = __fmaf_rn(a0f, __fadd_rn(cc[j], 1.f), sa[j]);   // p_ng(v), as in mix_p
          h4[j] = __fsub_rn(h4[j], __fmul_rn(q, lg2f(q)));
        }
      }
    float h = __fadd_rn(__fadd_rn(h4[0], h4[1]), __fadd_rn(h4[2], h4[3]));
#pragma unroll
    for (int o = 16; o; o >>= 1) h = __fadd_rn(h, __shfl_xor_sync(0xffffffffu, h, o));
    if (lane == 0) sm.red_h[wid] = h;
    __syncthreads();
    if (wid == 0) {
      h = sm.red_h[lane];
#pragma unroll
      for (int o = 16; o; o >>= 1) h = __fadd_rn(h, __shfl_xor_sync(0xffffffffu, h, o));
      if (lane == 0) {
        if (CS > 1) {
#pragma unroll
          for (int r = 0; r < CS; ++r) tc::st_cluster_s32(tc::mapa(&xh[par][rank], (uint32_t)r), __float_as_int(h));
        } else {
          xh[par][0] = h;
        }
      }
    }
    if (CS > 1) cl_sync(); else __syncthreads();
    float H = xh[par][0];
    for (int r = 1; r < CS; ++r) H = __fadd_rn(H, xh[par][r]);
    return H;
  };

  // exponential-weights mixer step (D24-D26), one thread, in f64 (SURVEY §8(c):
  // "the scalars ... are computed in f64 by one thread").  With two experts the weights depend
  // only on the log-odds d = lw_l - lw_n (the renormalisation subtracts the same lse from
  // both), so lw += eta [ln max(pt_t, 1e-12), ln max(png_t, 1e-12)] is d += eta ln(ratio) and
  // softmax(lw) = (1 / (1 + e^-d), e^-d / (1 + e^-d)) -- equal in real arithmetic to the
  // oracle's literal form.  Thread 0 of every CTA and the decoder run this same arithmetic.
  auto mixer_update = [&](float pt_t, float png_t) {
    const double r = __ddiv_rn(fmax((double)pt_t, 1e-12), fmax((double)png_t, 1e-12));
    const double d = __fma_rn(a.eta, ln_f64(r), s_lw[0]);
    s_lw[0] = d;
    s_lw[1] = 0.0;
    const double e = exp_neg_f64(fabs(d));
    const double big = __drcp_rn(__dadd_rn(1.0, e)), small = __dmul_rn(e, big);
    s_w[0] = (float)(d >= 0.0 ? big : small);
    s_w[1] = (float)(d >= 0.0 ? small : big);
  };

  if (enc) {
    // ===================================================== compression ===
    // Thread t owns the local float4 groups t, t + WT, ... (at most NGM).  The
    // current row's logits stay in registers from the previous token's pass, and
    // the next row's loads are issued first thing, so the HBM latency of the
    // (L2-cold) logits overlaps the current token's work.  Arithmetic and its
    // order are those of the decoder: (m, s) per thread in group then element
    // order, the same warp/CTA (m, s) tree as cta_ms, exact integer sums and an
    // order-free argmax; only where the values come from changed.

    const uint32_t i0 = s_i;
    // test-only full-vector dumps (a.n_dump > 0): the next dumped token index of this chunk
    uint32_t dslot = 0, drow = 0xffffffffu;
    if (a.n_dump && c == a.dump_chunk) {
      uint32_t lo = 0, hi = a.n_dump;   // first dump row >= i0
      while (lo < hi) {
        const uint32_t mid = (lo + hi) / 2;
        if (a.dump_rows[mid] < i0) lo = mid + 1; else hi = mid;
      }
      dslot = lo;
      drow = lo < a.n_dump ? a.dump_rows[lo] : 0xffffffffu;
    }
    float uc[NGM][4];   // e = 2^((u - mth) log2 e) of the current token (u = z / tau + b), from the previous pass
    float mth = -CUDART_INF_F;   // this thread's max of the current token's u
    auto zload = [&](const float *zrow, float4 (&dst)[NGM]) {
#pragma unroll
      for (int k = 0; k < NGM; ++k)
        if (k < ng) dst[k] = __ldcs(reinterpret_cast<const float4 *>(zrow + vb) + tid + k * WT);
    };
    auto u4 = [&](const float4 z4, int g, float u[4]) {
      const double2 b01 = reinterpret_cast<const double2 *>(b_s)[2 * g];
      const double2 b23 = reinterpret_cast<const double2 *>(b_s)[2 * g + 1];
      u[0] = walk_u(z4.x, b01.x, inv_tau); u[1] = walk_u(z4.y, b01.y, inv_tau);
      u[2] = walk_u(z4.z, b23.x, inv_tau); u[3] = walk_u(z4.w, b23.y, inv_tau);
    };
    // push this CTA's slot `par` (complete in xs[par]) into every CTA's xin[par][rank]
    auto push_slot = [&](int par) {   // warp 0
      const uint32_t *src = reinterpret_cast<const uint32_t *>(&xs[par]);
      uint32_t *dst = reinterpret_cast<uint32_t *>(&xin[par][rank]);
      for (int w = lane; w < XWE; w += 32) {   // compression: the prefix the combine reads
        const uint32_t v = src[w];
        if (CS > 1) {
#pragma unroll
          for (int r = 0; r < CS; ++r) tc::st_cluster_s32(tc::mapa(dst + w, (uint32_t)r), (int)v);
        } else {
          dst[w] = v;
        }
      }
    };
    if (wid == 0) {
      if (use_ng && i0 >= a.warmup) { prefetch_pre(i0); prefetch_wait(); __syncwarp(); }
      scatter_list(i0);
    }
    // softmax statistics of the first token
    {
      float4 z0[NGM];
      zload(a.logits + (size_t)row0 * a.ldl, z0);
      float tm, ts;
#pragma unroll
      for (int k = 0; k < NGM; ++k)
        if (k < ng) u4(z0[k], tid + k * WT, uc[k]);
      ms_regs_e(uc, ng, tm, ts);   // uc now holds e = 2^((u - m) log2 e)
      mth = tm;
      cta_ms(tm, ts);
      if (tid == 0) { xs[1].m = tm; xs[1].s = ts; }
      __syncthreads();
      if (wid == 0) push_slot(1);
      if (CS > 1) cl_sync(); else __syncthreads();
      if (tid == 0) {
        float M, S;
        ms_cluster<CS>(xin[1], M, S);
        sm.M = M; sm.invS = __frcp_rn(S);
      }
      __syncthreads();
    }
    // token ids through a shared ring (tokens [it, it + 1,025) loaded every 1,024 tokens,
    // coalesced): the per-token load of the next id was a dependent global round trip
    auto refill_tokens = [&](int it0) {
      for (int j = tid; j <= 1024; j += WT)
        if (it0 + j < count) s_tok[(it0 + j) & 2047] = a.tokens[toff + i0 + it0 + j];
      __syncthreads();
    };
    refill_tokens(0);
    int tok_cur = count > 0 ? (int)s_tok[0] : 0;
    // this CTA's slice of logits row r into L2 (one TMA bulk prefetch): rows are
    // prefetched two tokens ahead so the register loads one token ahead hit L2
    auto l2_prefetch_row = [&](int r) {
      if (tid == 0 && r < count)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.logits + (size_t)(row0 + r) * a.ldl + vb),
                     "r"(Vc * 4u)
                     : "memory");
    };
    l2_prefetch_row(1);
    l2_prefetch_row(2);
    for (int it = 0; it < count; ++it) {
      if (it > 0 && (it & 1023) == 0) refill_tokens(it);
#ifdef NC_WALK_TIMING
      long long _wt = clock64();
      if (tid == 0 && rank == 0) atomicAdd(&g_walk_clk[7], 1ull);
#endif
      const bool has_next = it + 1 < count;
      l2_prefetch_row(it + 3);
      float4 zn[NGM];
#if defined(NC_WALK_ABL)   // diagnostics: next row = constant (no load dependence)
      for (int k = 0; k < NGM; ++k) zn[k] = make_float4(uc[k][0], uc[k][1], uc[k][2], uc[k][3]);
#else
      if (has_next) zload(a.logits + (size_t)(row0 + it + 1) * a.ldl, zn);
#endif
      const uint32_t i = i0 + it;
      const int par = it & 1;
      const int tok = tok_cur;
      if (has_next) tok_cur = (int)s_tok[(it + 1) & 2047];
      const bool dump = drow == i;
      const int ltok = tok - (int)vb;                  // local id (may be outside [0, Vc))
      const float M = sm.M, invS = sm.invS, a0f = sm.a0f, wl = s_w[0], wn = s_w[1];
      const float scale = pt_scale(mth, M, invS);   // p~ = e * scale for this thread's elements
      const int mix = sm.mix;
      const bool skip = (use_skip && mix) ? ng_entropy(par, a0f) < kSkipTauBits : false;
      const bool pre_next = has_next && use_ng && i + 1 >= a.warmup;
      if (wid == 1 && pre_next) prefetch_pre(i + 1);
      uint32_t my_sum = 0, my_cum = 0;
      Best bb{-1.f, 0x7fffffff, 0};
      float tm = -CUDART_INF_F, ts = 0.f;   // next token's softmax statistics (after the group loop)
      const int tg = ltok >= 0 ? (ltok >> 2) : -1;
      const int gcut = ltok < 0 ? 0 : (ltok >= (int)Vc ? Gc : tg);   // local groups entirely below tok
      // p~ and the mixed p of group k (MIX: the N-gram is mixed in)
      auto probs = [&](auto MIXC, int k, int g, float (&pt)[4], float (&png)[4], float (&p)[4]) {
        constexpr bool MIX = decltype(MIXC)::value;
#pragma unroll
        for (int j = 0; j < 4; ++j) pt[j] = __fmul_rn(uc[k][j], scale);
        if (!MIX) {
#pragma unroll
          for (int j = 0; j < 4; ++j) { png[j] = 0.f; p[j] = pt[j]; }
        } else {
          const float4 c4 = reinterpret_cast<const float4 *>(cu_s)[g];
          const float cc[4] = {c4.x, c4.y, c4.z, c4.w};
          const uint32_t bits = (bitmap[g >> 3] >> ((g & 7) * 4)) & 15u;
          const float4 s4 = bits ? reinterpret_cast<const float4 *>(sp_s)[g] : make_float4(0.f, 0.f, 0.f, 0.f);
          const float sa[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) p[j] = mix_p(pt[j], a0f, cc[j], sa[j], wl, wn, png[j], skip);
        }
      };
      if (dump) {   // test-only full vectors of this token (same values as the pass below)
#pragma unroll
        for (int k = 0; k < NGM; ++k) {
          if (k >= ng) break;
          const int g = tid + k * WT;
          float pt[4], png[4], p[4];
          if (mix) probs(std::true_type{}, k, g, pt, png, p);
          else probs(std::false_type{}, k, g, pt, png, p);
          uint32_t cv[4];
          quant4(p, TmV, cv);
          const size_t o = (size_t)dslot * V + vb + 4 * g;
          *reinterpret_cast<float4 *>(a.dump_pt + o) = make_float4(pt[0], pt[1], pt[2], pt[3]);
          *reinterpret_cast<float4 *>(a.dump_p + o) = make_float4(p[0], p[1], p[2], p[3]);
          *reinterpret_cast<uint4 *>(a.dump_c + o) = make_uint4(cv[0], cv[1], cv[2], cv[3]);
        }
      }
      // the fused pass, specialised on (mix, head) so the per-group loop carries no branches on them
      auto pass = [&](auto MIXC, auto HEADC) {
        constexpr bool HEAD = decltype(HEADC)::value;
#pragma unroll
        for (int k = 0; k < NGM; ++k) {
          if (k >= ng) break;
          const int g = tid + k * WT;
          float pt[4], png[4], p[4];
          probs(MIXC, k, g, pt, png, p);
          uint32_t cv[4];
          quant4(p, TmV, cv);
          // argmax (largest p, lowest id on ties): the group's max, then its first position;
          // the winner's count is quant(p) after the loop
          const float gm = fmaxf(fmaxf(p[0], p[1]), fmaxf(p[2], p[3]));
          if (gm > bb.v) {
            bb.v = gm;
            bb.i = (int)vb + 4 * g + (p[0] == gm ? 0 : (p[1] == gm ? 1 : (p[2] == gm ? 2 : 3)));
          }
          const uint32_t gs = cv[0] + cv[1] + cv[2] + cv[3];
          my_sum += gs;
          const bool tokg = g == tg && ltok < (int)Vc;
          if (g < gcut) {
            my_cum += gs;
          } else if (tokg) {
            const int jt = ltok & 3;
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (j < jt) my_cum += cv[j];
              else if (j == jt) { xs[par].pt_t = pt[j]; xs[par].png_t = png[j]; xs[par].p_t = p[j]; xs[par].freq_t = cv[j]; }
          }
          if (HEAD) {
            double2 *bp = reinterpret_cast<double2 *>(b_s) + 2 * g;
            double2 b01 = bp[0], b23 = bp[1];
            b01.x = b_step(b01.x, pt[0], a.alpha);
            b01.y = b_step(b01.y, pt[1], a.alpha);
            b23.x = b_step(b23.x, pt[2], a.alpha);
            b23.y = b_step(b23.y, pt[3], a.alpha);
            if (tokg) b_tok_fix(b01, b23, ltok & 3, a.alpha);
            bp[0] = b01; bp[1] = b23;
            if (has_next) {   // next token's u with the updated bias (== walk_u(z, b_new)), stats in decoder order
              uc[k][0] = __fmaf_rn(zn[k].x, inv_tau, (float)b01.x); uc[k][1] = __fmaf_rn(zn[k].y, inv_tau, (float)b01.y);
              uc[k][2] = __fmaf_rn(zn[k].z, inv_tau, (float)b23.x); uc[k][3] = __fmaf_rn(zn[k].w, inv_tau, (float)b23.y);
            }
          } else if (has_next) {
            uc[k][0] = __fmul_rn(zn[k].x, inv_tau); uc[k][1] = __fmul_rn(zn[k].y, inv_tau);   // b == 0
            uc[k][2] = __fmul_rn(zn[k].z, inv_tau); uc[k][3] = __fmul_rn(zn[k].w, inv_tau);
          }
        }
      };
      if (mix) {
        if (use_head) pass(std::true_type{}, std::true_type{});
        else pass(std::true_type{}, std::false_type{});
      } else {
        if (use_head) pass(std::false_type{}, std::true_type{});
        else pass(std::false_type{}, std::false_type{});
      }
      bb.c = bb.v >= 0.f ? quant(bb.v, TmV) : 0u;   // = the quant4 count of that element
#if defined(NC_WALK_ABL) && NC_WALK_ABL >= 2   // diagnostics: no statistics
      tm = 0.f; ts = 1.f;
#else
      if (has_next) {
        ms_regs_e(uc, ng, tm, ts);
        mth = tm;
      }
#endif
      WALK_MARK(0);
      if (wid == 1 && pre_next) prefetch_wait();
      // one CTA reduction: (m, s) through the cta_ms tree, exact sums, argmax
      {
        ms_warp(tm, ts);
        const uint32_t s1 = __reduce_add_sync(0xffffffffu, my_sum), s2 = __reduce_add_sync(0xffffffffu, my_cum);
        Best wb = best_warp(bb);
        if (lane == 0) {
          sm.red_m[wid] = tm; sm.red_s[wid] = ts;
          sm.red_sum[wid] = s1; sm.red_cum[wid] = s2;
          sm.red_bv[wid] = wb.v; sm.red_bi[wid] = wb.i; sm.red_bc[wid] = wb.c;
        }
        __syncthreads();
        if (wid == 0) {
          tm = sm.red_m[lane]; ts = sm.red_s[lane];
          ms_warp(tm, ts);
          const uint32_t c1 = __reduce_add_sync(0xffffffffu, (uint32_t)sm.red_sum[lane]);
          const uint32_t c2 = __reduce_add_sync(0xffffffffu, (uint32_t)sm.red_cum[lane]);
          const Best cb = best_warp(Best{sm.red_bv[lane], sm.red_bi[lane], sm.red_bc[lane]});
          if (lane == 0) {
            Xch &x = xs[par];
            x.sum = c1; x.cum = c2; x.bv = cb.v; x.bi = cb.i; x.bc = cb.c; x.m = tm; x.s = ts;
            x.has_tok = (ltok >= 0 && ltok < (int)Vc) ? 1 : 0;
          }
          __syncwarp();
          push_slot(par);
        }
      }
      WALK_MARK(1);
      if (CS > 1) cl_sync(); else __syncthreads();
      WALK_MARK(2);
      if (wid == 0 || wid == 2 || wid == 3) {
        // the combine, split over three warps that run concurrently (same arithmetic as one
        // thread in sequence): warp 0 codes the token, warp 2 runs the mixer, warp 3 the
        // next token's softmax statistics (warp 1 swaps the N-gram fixups meanwhile)
        if (wid == 0) {
          // the CS slots across the warp's lanes: exact integer sums (order-free; a CTA's
          // count sum is <= T < 2^31), the order-free argmax, and the one slot holding the token
          const bool in = lane < CS;
          const Xch &x = xin[par][in ? lane : 0];
          const unsigned long long s1 = __reduce_add_sync(0xffffffffu, in ? (uint32_t)x.sum : 0u);
          const unsigned long long s2 = __reduce_add_sync(0xffffffffu, in ? (uint32_t)x.cum : 0u);
          const Best b2 = best_warp(in ? Best{x.bv, x.bi, x.bc} : Best{-1.f, 0x7fffffff, 0u});
          const unsigned tb = __ballot_sync(0xffffffffu, in && x.has_tok);
          const int src = tb ? __ffs(tb) - 1 : 0;
          const float p_t = tb ? __shfl_sync(0xffffffffu, x.p_t, src) : 0.f;
          const float pt_t = tb ? __shfl_sync(0xffffffffu, x.pt_t, src) : 0.f;
          const uint32_t fq = tb ? __shfl_sync(0xffffffffu, x.freq_t, src) : 0u;
          if (lane == 0) {
          const long long R = (long long)T - (long long)s1;
          if ((long long)b2.c + R < 1) st->err = 1;     // D6
          if (dump && (uint32_t)b2.i / Vc == rank)       // the argmax's final count (its owner CTA)
            a.dump_c[(size_t)dslot * V + b2.i] = (uint32_t)((long long)b2.c + R);
          const unsigned long long cum_t = s2 + (b2.i < tok ? R : 0);
          const unsigned long long freq_t = (unsigned long long)((long long)fq + (b2.i == tok ? R : 0));
          if (rank == 0) {
            const size_t oi = (size_t)toff + i;
            a.out_cum[oi] = (uint32_t)cum_t;
            a.out_freq[oi] = (uint32_t)freq_t;
            if (a.out_p) a.out_p[oi] = p_t;
            if (a.out_pt) a.out_pt[oi] = pt_t;
          }
          if (use_ng && ltok >= 0 && ltok < (int)Vc) cu_s[ltok] = __fadd_rn(cu_s[ltok], 1.f);
          }
        } else if (wid == 2 && lane == 0) {
          if (mix) {
            float pt_t = 0.f, png_t = 0.f;
            for (int r = 0; r < CS; ++r)
              if (xin[par][r].has_tok) { pt_t = xin[par][r].pt_t; png_t = xin[par][r].png_t; }
            mixer_update(pt_t, png_t);
          }
        } else if (wid == 3 && lane == 0) {
          if (has_next) {
            float nm, ns;
            ms_cluster<CS>(xin[par], nm, ns);
            sm.M = nm;
            sm.invS = __frcp_rn(ns);
          }
        }
      } else if (wid == 1) {   // N-gram fixups: this token's out, the next token's in (parallel to warp 0)
        clear_list(i);
        __syncwarp();
        if (has_next) scatter_list(i + 1);
      }
      WALK_MARK(3);
      if (dump) {
        ++dslot;
        drow = dslot < a.n_dump ? a.dump_rows[dslot] : 0xffffffffu;
      }
      __syncthreads();
      WALK_MARK(4);
    }
    if (tid == 0) s_i = i0 + count;
  } else {
    // ======================================================== decompression ===
    for (int it = 0; it < count; ++it) {
      const float *z = a.logits + (size_t)(row0 + it) * a.ldl;
      const uint32_t i = s_i;
      const int par = it & 1;
      // (1) N-gram prediction by rank 0, shared through DSMEM; decoder target.
      //     gsum (max(V/CS/4, V/32) words, idle here) is the predictor's full-vocab bitmap scratch.
      for (int w = tid; w < (int)((V + 31) / 32); w += WT) gsum[w] = 0u;
      __syncthreads();
      if (rank == 0 && wid == 0 && use_ng && i >= a.warmup) {
        uint32_t hist[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) hist[j] = st->hist[j];
        ng_predict_warp(a, c, i, hist, a.spadd + (size_t)c * V, gsum, &sm.lists[i & 1], lane);
      }
      __syncthreads();
      if (CS > 1) cl_sync();
      if (wid == 0) {
        if (rank != 0 && use_ng && i >= a.warmup) {   // copy rank 0's list (header + used entries)
          NgTok &L = sm.lists[i & 1];
          uint32_t *hdr = reinterpret_cast<uint32_t *>(&L);
          for (uint32_t w = lane; w < 4; w += 32) hdr[w] = cl_ld(hdr + w, 0u);
          const uint32_t n = cl_ld(&L.n, 0u);
          for (uint32_t j = lane; j < n; j += 32) {
            L.tok[j] = cl_ld(&L.tok[j], 0u);
            L.add[j] = __uint_as_float(cl_ld(&L.add[j], 0u));
          }
          __syncwarp();
        }
        scatter_list(i);
        if (lane == 0) {
          if (a.coder == 1) {   // rANS: the slot x mod T (D39)
            sm.target = st->value & (T - 1);
          } else {
            const unsigned long long R = st->high - st->low + 1;
            sm.target = ((st->value - st->low + 1) * T - 1) / R;
          }
        }
      }
      __syncthreads();
      // skip test for this token (same arithmetic as compression)
      const bool skip = (use_skip && sm.mix) ? ng_entropy(par, sm.a0f) < kSkipTauBits : false;
      // (2) softmax statistics
      {
        float ud[NGM][4];
#pragma unroll
        for (int k = 0; k < NGM; ++k)
          if (k < ng) load_u(z, tid + k * WT, ud[k]);
        float tm, ts;
        ms_regs(ud, ng, tm, ts);
        s_mth[tid] = tm;
        cta_ms(tm, ts);
        if (tid == 0) { xs[par].m = tm; xs[par].s = ts; }
        __syncthreads();
        if (CS > 1) cl_sync();
        if (wid == 0) {
          gather(par);
          if (lane == 0) {
            float M, S;
            ms_cluster<CS>(xin[par], M, S);
            sm.M = M; sm.invS = __frcp_rn(S);
          }
        }
        __syncthreads();
      }
      const float M = sm.M, invS = sm.invS, a0f = sm.a0f, wl = s_w[0], wn = s_w[1];
      const int mix = sm.mix;
      const float mth = s_mth[tid], scale = pt_scale(mth, M, invS);   // this thread's groups tid + k WT
      // (3) counts
      uint32_t my_sum = 0;
      Best bb{-1.f, 0x7fffffff, 0};
      for (int g = tid; g < Gc; g += WT) {
        float pt[4], png[4], p[4];
        prob4(z, g, mth, scale, wl, wn, a0f, mix, skip, pt, png, p);
        uint32_t gs = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t cv = quant(p[j], TmV);
          gs += cv;
          if (p[j] > bb.v) { bb.v = p[j]; bb.i = (int)vb + 4 * g + j; bb.c = cv; }
        }
        my_sum += gs;
        gsum[g] = gs;
      }
      {
        unsigned long long c1 = 0, c2 = 0;
        Best cb{};
        cta_counts((unsigned long long)my_sum, 0ull, bb, c1, c2, cb);
        if (tid == 0) { Xch &x = xs[par]; x.sum = c1; x.bv = cb.v; x.bi = cb.i; x.bc = cb.c; x.found = 0; }
        __syncthreads();
        if (CS > 1) cl_sync();
        if (wid == 0) {
          gather(par);
          if (lane == 0) {
            unsigned long long s1 = 0, before = 0;
            Best b2{-1.f, 0x7fffffff, 0};
            for (int r = 0; r < CS; ++r) { s1 += xin[par][r].sum; best_merge(b2, xin[par][r].bv, xin[par][r].bi, xin[par][r].bc); }
            const long long R = (long long)T - (long long)s1;
            if ((long long)b2.c + R < 1) st->err = 1;
            for (int r = 0; r < (int)rank; ++r) before += xin[par][r].sum + ((uint32_t)b2.i / Vc == (uint32_t)r ? R : 0);
            sm.resid = R;
            sm.argmax = b2.i;
            sm.cum_t = before;                           // this CTA's first cumulative count
            if ((uint32_t)b2.i / Vc == rank) gsum[(b2.i - vb) >> 2] = (uint32_t)((long long)gsum[(b2.i - vb) >> 2] + R);
          }
        }
        __syncthreads();
      }
      // (4) prefix scan over the local groups in id order, search the target
      {
        const long long R = sm.resid;
        const int am = sm.argmax - (int)vb;
        const int gpt = (Gc + WT - 1) / WT;
        const int g0 = min(Gc, tid * gpt), g1 = min(Gc, g0 + gpt);
        uint32_t adj = 0;
        for (int g = g0; g < g1; ++g) adj += gsum[g];
        uint32_t x = adj;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (lane == 31) sm.scan[wid] = x;
        __syncthreads();
        if (wid == 0) {
          uint32_t y = sm.scan[lane];
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t z2 = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += z2;
          }
          sm.scan[lane] = y;
        }
        __syncthreads();
        const unsigned long long excl = sm.cum_t + (unsigned long long)(x - adj) + (wid ? sm.scan[wid - 1] : 0u);
        const unsigned long long tgt = sm.target;
        if (adj > 0 && tgt >= excl && tgt < excl + adj) {
          unsigned long long accm = excl;
          int gf = g0;
          for (; gf < g1; ++gf) {
            if (tgt < accm + gsum[gf]) break;
            accm += gsum[gf];
          }
          float pt[4], png[4], p[4];
          const float mo = s_mth[gf % WT];   // the max of the thread that owns group gf
          prob4(z, gf, mo, pt_scale(mo, M, invS), wl, wn, a0f, mix, skip, pt, png, p);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int v = 4 * gf + j;
            unsigned long long cv = quant(p[j], TmV);
            if (v == am) cv = (unsigned long long)((long long)cv + R);
            if (tgt < accm + cv) {
              Xch &xx = xs[par];
              xx.found = 1; xx.t = (int)vb + v; xx.cum_t = accm; xx.fq_t = cv;
              xx.fpt = pt[j]; xx.fpng = png[j]; xx.fp = p[j];
              break;
            }
            accm += cv;
          }
        }
        __syncthreads();
        if (CS > 1) cl_sync();
        if (wid == 0) {
          gather(par);
          if (lane == 0) {
            int t = -1;
            for (int r = 0; r < CS; ++r)
              if (xin[par][r].found) {
                t = xin[par][r].t; sm.cum_t = xin[par][r].cum_t; sm.freq_t = xin[par][r].fq_t;
                sm.pt_t = xin[par][r].fpt; sm.png_t = xin[par][r].fpng; sm.p_t = xin[par][r].fp;
              }
            sm.tok = t;
            if (t < 0 || tgt >= T) st->err = 2;
          }
        }
        __syncthreads();
      }
      // (5) bias update with the decoded token
      const int t = sm.tok;
      const int lt = t - (int)vb;
      if (use_head)
        for (int g = tid; g < Gc; g += WT) {
          float pt[4], png[4], p[4];
          prob4(z, g, mth, scale, wl, wn, a0f, mix, skip, pt, png, p);
          double2 *bp = reinterpret_cast<double2 *>(b_s) + 2 * g;
          double2 b01 = bp[0], b23 = bp[1];
          b01.x = b_step(b01.x, pt[0], a.alpha);
          b01.y = b_step(b01.y, pt[1], a.alpha);
          b23.x = b_step(b23.x, pt[2], a.alpha);
          b23.y = b_step(b23.y, pt[3], a.alpha);
          if (lt >= 0 && (lt >> 2) == g) b_tok_fix(b01, b23, lt & 3, a.alpha);
          bp[0] = b01; bp[1] = b23;
        }
      __syncthreads();
      // (6) scalars: outputs, coder, mixer, counts, N-gram update (rank 0)
      if (wid == 0) {
        if (lane == 0) {
          const uint32_t tt = (uint32_t)max(t, 0);
          if (rank == 0) {
            const size_t oi = (size_t)toff + i;
            a.out_tok[oi] = tt;
            if (a.next_x) a.next_x[c] = tt;
            if (a.out_p) a.out_p[oi] = sm.p_t;
            if (a.out_pt) a.out_pt[oi] = sm.pt_t;
            if (a.coder == 1) {   // rANS: x = freq (x >> b) + slot - cum, then refill 32-bit words (D39)
              const uint8_t *s = a.streams + a.stream_off[c];
              const unsigned long long nb = a.stream_bits[c];
              unsigned long long x = st->value, bp = st->bitpos;
              x = sm.freq_t * (x >> a.cdf_bits) + (x & (T - 1)) - sm.cum_t;
              // a valid stream refills at most once (x >= freq (L >> b) >= 1 before it); x = 0
              // only comes from a corrupt stream and must not spin on zero words
              for (int r = 0; r < 2 && x < (1ull << 31); ++r) { x = (x << 32) | ans_word(s, bp, nb); bp += 32; }
              if (x < (1ull << 31)) st->err = 3;
              st->value = x; st->bitpos = bp;
            } else {
              const unsigned long long Rg = st->high - st->low + 1;
              unsigned long long lo = st->low, hi = st->low + ((Rg * (sm.cum_t + sm.freq_t)) >> a.cdf_bits) - 1;
              lo = lo + ((Rg * sm.cum_t) >> a.cdf_bits);
              unsigned long long val = st->value, bp = st->bitpos;
              uint32_t pend = st->pend;
              const uint8_t *s = a.streams + a.stream_off[c];
              const unsigned long long nb = a.stream_bits[c];
              for (;;) {
                if (hi < HALF) { pend = 0; }
                else if (lo >= HALF) { lo -= HALF; hi -= HALF; val -= HALF; pend = 0; }
                else if (lo >= QTR && hi < 3 * QTR) { lo -= QTR; hi -= QTR; val -= QTR; ++pend; }
                else break;
                lo = 2 * lo; hi = 2 * hi + 1;
                const unsigned long long bit = bp < nb ? (s[bp >> 3] >> (7 - (bp & 7))) & 1u : 0u;
                val = 2 * val + bit;
                ++bp;
              }
              st->low = lo; st->high = hi; st->value = val; st->bitpos = bp; st->pend = pend;
            }
          }
          if (mix) mixer_update(sm.pt_t, sm.png_t);
          if (use_ng && lt >= 0 && lt < (int)Vc) cu_s[lt] = __fadd_rn(cu_s[lt], 1.f);
          s_i = i + 1;
        }
        __syncwarp();
        clear_list(i);
        __syncwarp();
        if (rank == 0 && use_ng && t >= 0) {
          uint32_t hist[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) hist[j] = st->hist[j];
          ng_update_warp(a, c, i, hist, (uint32_t)t, st, lane);
          if (lane == 0) { ng_hist_push(st, (uint32_t)t); st->ng_i = i + 1; }
        }
      }
      __syncthreads();
    }
  }

  // ---- write the state slice back
  for (uint32_t v = tid; v < Vc; v += WT) {
    if (use_head) b_g[v] = b_s[v];
    if (use_ng) cu_g[v] = (uint32_t)cu_s[v];
  }
  if (tid == 0 && rank == 0) {
    st->lw[0] = s_lw[0]; st->lw[1] = s_lw[1];
    st->wl = s_w[0]; st->wn = s_w[1];
    st->i = s_i;
  }
  if (CS > 1) cl_sync();     // no CTA leaves while a peer may still read its shared memory
}

// Cluster size used for a vocabulary: fixed per V (never per batch), so that the
// reduction trees of compression and decompression are the same.
// CTAs per chunk: a function of the vocabulary and of the container's chunk count only, so
// compression and decompression (which reads the count from the NC05 header) agree -- the
// vocabulary partition fixes the order of the float reductions.
static int walk_cluster_size(uint32_t V, int n_chunks) {
  static const int forced = [] {   // diagnostics override NC_WALK_CS=4|8 (compress and decompress must agree)
    const char *e = std::getenv("NC_WALK_CS");
    return e ? std::atoi(e) : 0;
  }();
  if (V < 4096 || V % 64) return 1;
  if (forced == 4 || forced == 8 || forced == 16) return forced;
  // 8 CTAs per chunk for large vocabularies: halves the per-token pass (config2: walk 29.7 ->
  // 21.6 ms of kernel time, step time unchanged -- its SMs come out of the overlapped forward).
  // With one or two chunks in the container the walk is the whole critical path: a 16-CTA
  // (non-portable) cluster halves the pass again (config2 with one chunk: 1.04 -> 1.27 MB/s;
  // per token 8.0k -> 6.0k cycles).  The rule's inputs are the vocabulary and the
  // CONTAINER's chunk count (the decoder reads it from the header; a shard passes the total).
  if (n_chunks <= 2 && V >= 32768 && V % 1024 == 0) return 16;
  // Many chunks: the walk's clusters run in waves beside the next slab's forward and their
  // SM-time is what the step pays -- 4-CTA clusters hold half the SMs per chunk for ~1.4x
  // the per-token time (config3, 64 chunks: walk 772 -> 573 ms of kernel time, step
  // 4781 -> 4709 ms).  8 CTAs while one wave of clusters fits the B200's 148 SMs (a
  // constant, not the device's count: the rule must not depend on the decoding GPU).
  if (V >= 32768 && V % 256 == 0 && n_chunks * 8 <= 148) return 8;
  return 4;
}

template <int CS, int NGM>
static void launch_walk_cs(const WalkArgs &a, cudaStream_t s) {
  constexpr int WT = walk_threads(CS);
  const uint32_t Vc = a.V / CS;
  if (Vc % 4 || Vc / 4 > (uint32_t)NGM * WT)   // float4 groups, at most NGM per thread (register-resident rows)
    throw std::runtime_error("walk: vocabulary slice of " + std::to_string(Vc) +
                             " ids per CTA unsupported (needs a multiple of 4, at most 16384)");
  // b f64, cu, spadd, the slice bitmap, then gsum: the decoder's per-group counts (Vc / 4 words)
  // AND the N-gram predictor's full-vocabulary bitmap (V / 32 words; larger at 16 CTAs)
  const size_t gsum_words = std::max<size_t>(Vc / 4, (a.V + 31) / 32);
  const size_t dyn = (size_t)Vc * 8 + Vc * 4 + Vc * 4 + ((Vc + 31) / 32) * 4 + gsum_words * 4 + 64;
  static unsigned long long attr = 0;
  if (first_on_device(attr)) {
    // the largest slice this instantiation serves (4 NGM WT ids): the attribute sized to the
    // need, not the SM maximum, so 16-CTA clusters pass the cluster placement check
    const size_t vmax = (size_t)4 * NGM * WT;
    const size_t gmax = std::max<size_t>(vmax / 4, (size_t)CS * vmax / 32);   // V <= CS vmax
    const size_t dmax = vmax * 8 + vmax * 4 + vmax * 4 + ((vmax + 31) / 32) * 4 + gmax * 4 + 64;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, walk_cl_kernel<CS, NGM, WT>);
    const size_t cap = (size_t)std::max(0, optin - (int)fa.sharedSizeBytes);   // what static smem leaves
    check_launch(cudaFuncSetAttribute(walk_cl_kernel<CS, NGM, WT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)std::min(dmax, cap)),
                 "walk smem attribute");
    if (CS > 1)
      check_launch(cudaFuncSetAttribute(walk_cl_kernel<CS, NGM, WT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                   "walk cluster attribute");
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.n_entries * CS);
  cfg.blockDim = dim3(WT);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  check_launch(cudaLaunchKernelEx(&cfg, walk_cl_kernel<CS, NGM, WT>, a), "walk launch");
}

int walk_ctas_per_chunk(uint32_t V, int n_chunks) { return walk_cluster_size(V, n_chunks); }

void walk_timing_report() {
#ifdef NC_WALK_TIMING
  unsigned long long h[8];
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(h, g_walk_clk, sizeof(h));
  const double n = (double)(h[7] ? h[7] : 1);
  fprintf(stderr,
          "walk encode per token (cycles): fused pass %.0f | CTA reductions %.0f | cluster barrier %.0f | "
          "combine+mixer+lists %.0f | final sync %.0f | tokens %.0f\n",
          h[0] / n, h[1] / n, h[2] / n, h[3] / n, h[4] / n, n);
  unsigned long long z[8] = {};
  cudaMemcpyToSymbol(g_walk_clk, z, sizeof(z));
#endif
}

void launch_walk(const WalkArgs &a, cudaStream_t s) {
  if (a.n_entries <= 0) return;
  const int cs = walk_cluster_size(a.V, a.n_chunks_total);
  const int wt = walk_threads(cs);
  const uint32_t groups = (a.V / cs / 4 + wt - 1) / wt;   // float4 groups per thread
  if (cs == 16) {
    if (groups <= 2) launch_walk_cs<16, 2>(a, s);
    else launch_walk_cs<16, 4>(a, s);
  } else if (cs == 8) {
    if (groups <= 3) launch_walk_cs<8, 3>(a, s);
    else if (groups <= 4) launch_walk_cs<8, 4>(a, s);
    else launch_walk_cs<8, NGMAX>(a, s);
  } else if (cs == 4) {
    if (groups <= 6) launch_walk_cs<4, 6>(a, s);
    else launch_walk_cs<4, NGMAX>(a, s);
  } else {
    if (groups <= 2) launch_walk_cs<1, 2>(a, s);
    else launch_walk_cs<1, NGMAX>(a, s);
  }
}

__global__ void walk_init_kernel(WalkState *st, int n, double d0) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  WalkState w;
  memset(&w, 0, sizeof(w));
  w.lw[0] = d0;   // log-odds of the initial weights (0.85, 0.15); same formula as mixer_update
  w.lw[1] = 0.0;
  const double e = exp_neg_f64(fabs(d0));
  const double big = __drcp_rn(__dadd_rn(1.0, e)), small = __dmul_rn(e, big);
  w.wl = (float)(d0 >= 0.0 ? big : small);
  w.wn = (float)(d0 >= 0.0 ? small : big);
  w.high = 0xFFFFFFFFull;
  st[c] = w;
}
void launch_walk_init(WalkState *st, int n_chunks, cudaStream_t s) {
  if (n_chunks <= 0) return;
  walk_init_kernel<<<(n_chunks + 127) / 128, 128, 0, s>>>(st, n_chunks, std::log(0.85) - std::log(0.15));
}

// -------------------------------------------------- debug quantizer (D5) ---
__global__ void quantize_debug_kernel(const float *p, uint32_t V, uint32_t bits, uint32_t *counts) {
  __shared__ unsigned long long rs[NW];
  __shared__ float rv[NW]; __shared__ int ri[NW];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const float TmV = (float)((1ull << bits) - V);
  unsigned long long s = 0; float bv = -1.f; int bi = 0x7fffffff;
  for (uint32_t v = tid; v < V; v += WT) {
    const uint32_t c = quant(p[v], TmV);
    counts[v] = c; s += c;
    if (p[v] > bv || (p[v] == bv && (int)v < bi)) { bv = p[v]; bi = (int)v; }
  }
  for (int o = 16; o; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o); const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  if (lane == 0) { rs[wid] = s; rv[wid] = bv; ri[wid] = bi; }
  __syncthreads();
  if (tid == 0) {
    unsigned long long tot = 0; float v_ = -1.f; int i_ = 0x7fffffff;
    for (int w = 0; w < NW; ++w) {
      tot += rs[w];
      if (rv[w] > v_ || (rv[w] == v_ && ri[w] < i_)) { v_ = rv[w]; i_ = ri[w]; }
    }
    const long long R = (long long)(1ull << bits) - (long long)tot;
    const long long nv = (long long)counts[i_] + R;
    counts[i_] = nv < 1 ? 0u : (uint32_t)nv;   // 0 signals the D6 error to the host
  }
}
void launch_quantize_debug(const float *p, uint32_t V, uint32_t cdf_bits, uint32_t *counts, cudaStream_t s) {
  quantize_debug_kernel<<<1, WT, 0, s>>>(p, V, cdf_bits, counts);
}

}  // namespace nc
