// The per-token vocab-row CDF kernel ("walk"), v1: one 1024-thread CTA per
// chunk walks that chunk's tokens in order.
//
// Per token i of a chunk (alg:compress P:246-267; SURVEY.md §8(c) canonical loop):
//   u_v  = z_v / tau + (f32) b_v                           (D16a)
//   pt_v = exp(u_v - max u) / sum exp(u - max u)            (softmax, fp32)
//   p_v  = pt_v                                   (i < W or N-gram off)
//        = w_l pt_v + w_n p_ng(v)                 (otherwise)
//        p_ng(v) = a0 (c(v)+1)/(N+V) + sum_k a_k cnt_k(v)   (closed form of P:361-374)
//   c_v  = max(1, floor((double) p_v (T - V)))    (exact product, D5)
//   residual T - sum c added to c_argmax (lowest index on ties, D4; signed, D6)
//   encode: emit (cum_t, freq_t);  decode: prefix scan + WNC target search (D27)
//   b_v -= alpha (pt_v - [v = t])  in f64           (D17)
//   mixer: lw += eta [ln pt_t, ln p_ng(t)], renormalise (D24-D26)
//   N-gram update with t (D18-D23)
//
// Every float operation is an explicit round-to-nearest intrinsic, and encode
// and decode run the same code, so the decoder reproduces the encoder's counts
// bit for bit (D15).
#include <cuda_runtime.h>
#include <math_constants.h>

#include "walk.cuh"

namespace nc {

constexpr int WT = 1024;   // threads per CTA
constexpr int NW = WT / 32;

struct WalkSmem {
  float red_m[NW], red_s[NW];
  unsigned long long red_sum[NW], red_cum[NW];
  float red_bv[NW]; int red_bi[NW]; uint32_t red_bc[NW];
  uint32_t scan[NW];
  uint32_t sp_tok[kMaxOrders * kSlots];
  int sp_n;
  // per-token broadcast scalars
  float M, S, a0f, wl, wn;
  int mix, tok, argmax;
  long long resid;
  unsigned long long target, cum_t, freq_t;
  float pt_t, png_t, p_t;
};

__device__ __forceinline__ unsigned long long fnv_ctx(int k, const uint32_t *hist) {
  unsigned long long h = 0xcbf29ce484222325ull;
  const unsigned long long P = 0x100000001b3ull;
  h ^= (unsigned long long)(k & 255); h *= P;
  for (int j = 4 - k; j < 4; ++j) {
    uint32_t t = hist[j];
#pragma unroll
    for (int by = 0; by < 4; ++by) { h ^= (t >> (8 * by)) & 255u; h *= P; }
  }
  return h ? h : 1ull;
}

// warp-parallel linear probe; returns record index or -1 (and the first empty slot).
__device__ __forceinline__ int ng_probe(const unsigned long long *keys, const uint32_t *vals, uint32_t hcap,
                                        unsigned long long key, int lane, uint32_t *empty_slot) {
  uint32_t base = (uint32_t)(key ^ (key >> 32)) & (hcap - 1);
  for (uint32_t p = 0; p < hcap; p += 32) {
    uint32_t idx = (base + p + lane) & (hcap - 1);
    unsigned long long kk = keys[idx];
    unsigned m = __ballot_sync(0xffffffffu, kk == key);
    if (m) return (int)vals[__shfl_sync(0xffffffffu, idx, __ffs(m) - 1)];
    unsigned e = __ballot_sync(0xffffffffu, kk == 0ull);
    if (e) { *empty_slot = __shfl_sync(0xffffffffu, idx, __ffs(e) - 1); return -1; }
  }
  *empty_slot = 0xffffffffu;
  return -1;
}

__device__ __forceinline__ float walk_u(float z, double b, float inv_tau) {
  return __fmaf_rn(z, inv_tau, (float)b);
}
__device__ __forceinline__ double b_step(double b, float pt, bool is_t, double alpha) {
  return __fma_rn(-alpha, __dsub_rn((double)pt, is_t ? 1.0 : 0.0), b);
}
__device__ __forceinline__ uint32_t quant(float p, double TmV) {
  double q = floor(__dmul_rn((double)p, TmV));
  return q < 1.0 ? 1u : (uint32_t)q;
}

// Thread t owns the float4 groups g = t, t + WT, t + 2 WT, ... of the vocab row
// (coalesced 128-bit loads of z, 2 x 128-bit loads of the f64 bias).
struct Grp {
  float pt[4], png[4], p[4];
};

__global__ __launch_bounds__(WT, 1) void walk_kernel(WalkArgs a) {
  extern __shared__ uint32_t dyn[];
  const uint32_t V = a.V;
  const int G = (int)(V / 4);
  uint32_t *bitmap = dyn;                              // V/32 words: ids with N-gram fixups
  uint32_t *gsum = dyn + (V + 31) / 32;                // decode: per-group counts (G words)
  __shared__ WalkSmem sm;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int e = blockIdx.x;
  if (e >= a.n_entries) return;
  const int c = a.chunk_of[e];
  const int row0 = a.row0[e], count = a.count[e];
  if (count <= 0) return;
  WalkState *st = a.st + c;
  double *b = a.b + (size_t)c * V;
  uint32_t *cu = a.cu + (size_t)c * V;
  float *spadd = a.spadd + (size_t)c * V;
  const bool use_ng = a.flags & 1u, use_head = a.flags & 2u;
  const uint64_t T = 1ull << a.cdf_bits;
  const double TmV = (double)(T - V);
  const unsigned long long HALF = 1ull << 31, QTR = 1ull << 30;

  for (int w = tid; w < (int)((V + 31) / 32); w += WT) bitmap[w] = 0u;
  if (a.mode == 1 && tid == 0 && st->i == 0) {   // prime the decoder with 32 bits
    const uint8_t *s = a.streams + a.stream_off[c];
    unsigned long long v = 0, nb = a.stream_bits[c];
    for (int k = 0; k < 32; ++k) v = 2 * v + (k < (long long)nb ? (s[k >> 3] >> (7 - (k & 7))) & 1u : 0u);
    st->low = 0; st->high = 0xFFFFFFFFull; st->value = v; st->bitpos = 32;
  }
  __syncthreads();

  for (int it = 0; it < count; ++it) {
    const float *z = a.logits + (size_t)(row0 + it) * a.ldl;
    const uint32_t i = st->i;

    // ---------------- phase A: N-gram prediction + mixer weights (warp 0) ----
    if (wid == 0) {
      const int mix = (use_ng && i >= a.warmup) ? 1 : 0;
      int nsp = 0;
      if (mix) {
        uint32_t hist[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) hist[j] = st->hist[j];
        double mu[kMaxOrders + 1], beta[kMaxOrders + 1];
        int rec[kMaxOrders + 1];
        for (int k = 1; k <= kMaxOrders; ++k) { mu[k] = 1.0; beta[k] = 0.0; rec[k] = -1; }
        for (int k = 1; k <= (int)a.orders; ++k) {
          if (i < (uint32_t)k) continue;
          const size_t tb = ((size_t)c * kMaxOrders + (k - 1));
          uint32_t es;
          int r = ng_probe(a.ng_keys + tb * a.hcap, a.ng_vals + tb * a.hcap, a.hcap, fnv_ctx(k, hist), lane, &es);
          if (r < 0) continue;
          const NgRecord *R = a.ng_recs + tb * a.rcap + r;
          uint32_t ns = R->nslot, s = 0;
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
        for (int k = 1; k <= (int)a.orders; ++k) {
          if (rec[k] < 0) continue;
          double ak = beta[k];
          for (int j = k + 1; j <= (int)a.orders; ++j) ak = __dmul_rn(ak, mu[j]);
          const size_t tb = ((size_t)c * kMaxOrders + (k - 1));
          const NgRecord *R = a.ng_recs + tb * a.rcap + rec[k];
          const uint32_t ns = R->nslot;
          for (uint32_t s = lane; s < ns; s += 32) {
            const uint32_t tk = R->tok[s];
            spadd[tk] = __fadd_rn(spadd[tk], (float)__dmul_rn(ak, (double)R->cnt[s]));
            atomicOr(&bitmap[tk >> 5], 1u << (tk & 31));
            sm.sp_tok[nsp + s] = tk;
          }
          nsp += (int)ns;
          __syncwarp();
          __threadfence_block();
        }
        if (lane == 0) {
          const double l0 = st->lw[0], l1 = st->lw[1];
          const double mx = fmax(l0, l1);
          const double lse = __dadd_rn(mx, log(__dadd_rn(exp(__dsub_rn(l0, mx)), exp(__dsub_rn(l1, mx)))));
          sm.wl = (float)exp(__dsub_rn(l0, lse));
          sm.wn = (float)exp(__dsub_rn(l1, lse));
          sm.a0f = (float)__ddiv_rn(a0, (double)st->N + (double)V);
        }
      }
      if (lane == 0) {
        sm.mix = mix;
        sm.sp_n = nsp;
        sm.tok = (a.mode == 0) ? (int)a.tokens[a.tok_off[c] + i] : -1;
        if (a.mode == 1) {   // WNC decode target (D8)
          const unsigned long long R = st->high - st->low + 1;
          sm.target = ((st->value - st->low + 1) * T - 1) / R;
        }
      }
    }
    __syncthreads();

    const float inv_tau = a.inv_tau;
    auto load_u = [&](int g, float u[4]) {
      const float4 z4 = reinterpret_cast<const float4 *>(z)[g];
      if (use_head) {
        const double2 b01 = reinterpret_cast<const double2 *>(b)[2 * g];
        const double2 b23 = reinterpret_cast<const double2 *>(b)[2 * g + 1];
        u[0] = walk_u(z4.x, b01.x, inv_tau); u[1] = walk_u(z4.y, b01.y, inv_tau);
        u[2] = walk_u(z4.z, b23.x, inv_tau); u[3] = walk_u(z4.w, b23.y, inv_tau);
      } else {
        u[0] = walk_u(z4.x, 0.0, inv_tau); u[1] = walk_u(z4.y, 0.0, inv_tau);
        u[2] = walk_u(z4.z, 0.0, inv_tau); u[3] = walk_u(z4.w, 0.0, inv_tau);
      }
    };

    // ---------------- pass 1: max and sum of exp (per-thread online, fixed tree) ----
    {
      float tm = -CUDART_INF_F, ts = 0.f;
      for (int g = tid; g < G; g += WT) {
        float u[4];
        load_u(g, u);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (u[j] > tm) { ts = __fmaf_rn(ts, expf(__fsub_rn(tm, u[j])), 1.f); tm = u[j]; }
          else ts = __fadd_rn(ts, expf(__fsub_rn(u[j], tm)));
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const float om = __shfl_xor_sync(0xffffffffu, tm, o), os = __shfl_xor_sync(0xffffffffu, ts, o);
        const float mm = fmaxf(tm, om);
        const float e1 = (tm == -CUDART_INF_F) ? 0.f : expf(__fsub_rn(tm, mm));
        const float e2 = (om == -CUDART_INF_F) ? 0.f : expf(__fsub_rn(om, mm));
        ts = __fadd_rn(__fmul_rn(ts, e1), __fmul_rn(os, e2));
        tm = mm;
      }
      if (lane == 0) { sm.red_m[wid] = tm; sm.red_s[wid] = ts; }
      __syncthreads();
      if (wid == 0) {
        tm = sm.red_m[lane]; ts = sm.red_s[lane];
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const float om = __shfl_xor_sync(0xffffffffu, tm, o), os = __shfl_xor_sync(0xffffffffu, ts, o);
          const float mm = fmaxf(tm, om);
          const float e1 = (tm == -CUDART_INF_F) ? 0.f : expf(__fsub_rn(tm, mm));
          const float e2 = (om == -CUDART_INF_F) ? 0.f : expf(__fsub_rn(om, mm));
          ts = __fadd_rn(__fmul_rn(ts, e1), __fmul_rn(os, e2));
          tm = mm;
        }
        if (lane == 0) { sm.M = tm; sm.S = __frcp_rn(ts); }
      }
      __syncthreads();
    }
    const float M = sm.M, invS = sm.S, a0f = sm.a0f, wl = sm.wl, wn = sm.wn;
    const int mix = sm.mix, tok = sm.tok;

    // p for the 4 ids of group g (identical code in every pass that needs it)
    auto prob4 = [&](int g, Grp &q) {
      float u[4];
      load_u(g, u);
#pragma unroll
      for (int j = 0; j < 4; ++j) q.pt[j] = __fmul_rn(expf(__fsub_rn(u[j], M)), invS);
      if (!mix) {
#pragma unroll
        for (int j = 0; j < 4; ++j) { q.png[j] = 0.f; q.p[j] = q.pt[j]; }
        return;
      }
      const uint4 c4 = reinterpret_cast<const uint4 *>(cu)[g];
      const uint32_t cc[4] = {c4.x, c4.y, c4.z, c4.w};
      const uint32_t bits = (bitmap[g >> 3] >> ((g & 7) * 4)) & 15u;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float sp = (bits >> j) & 1u ? spadd[4 * g + j] : 0.f;
        q.png[j] = __fmaf_rn(a0f, (float)(cc[j] + 1u), sp);
        q.p[j] = __fmaf_rn(wl, q.pt[j], __fmul_rn(wn, q.png[j]));
      }
    };

    // ---------------- pass 2: p, counts, sums, argmax (+ b update when t is known) ----
    unsigned long long my_sum = 0, my_cum = 0;
    float bv = -1.f; int bi = 0x7fffffff; uint32_t bc = 0;
    for (int g = tid; g < G; g += WT) {
      Grp q;
      prob4(g, q);
      uint32_t gs = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int v = 4 * g + j;
        const uint32_t cv = quant(q.p[j], TmV);
        gs += cv;
        if (q.p[j] > bv) { bv = q.p[j]; bi = v; bc = cv; }
        if (a.mode == 0) {
          if (v < tok) my_cum += cv;
          if (v == tok) { sm.pt_t = q.pt[j]; sm.png_t = q.png[j]; sm.p_t = q.p[j]; sm.freq_t = cv; }
        }
      }
      my_sum += gs;
      if (a.mode == 1) gsum[g] = gs;
      if (a.mode == 0 && use_head) {
        double2 *bp = reinterpret_cast<double2 *>(b) + 2 * g;
        double2 b01 = bp[0], b23 = bp[1];
        const int v = 4 * g;
        b01.x = b_step(b01.x, q.pt[0], v == tok, a.alpha);
        b01.y = b_step(b01.y, q.pt[1], v + 1 == tok, a.alpha);
        b23.x = b_step(b23.x, q.pt[2], v + 2 == tok, a.alpha);
        b23.y = b_step(b23.y, q.pt[3], v + 3 == tok, a.alpha);
        bp[0] = b01; bp[1] = b23;
      }
    }
    {
      unsigned long long s1 = my_sum, s2 = my_cum;
      float v_ = bv; int i_ = bi; uint32_t c_ = bc;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        const float ov = __shfl_xor_sync(0xffffffffu, v_, o);
        const int oi = __shfl_xor_sync(0xffffffffu, i_, o);
        const uint32_t oc = __shfl_xor_sync(0xffffffffu, c_, o);
        if (ov > v_ || (ov == v_ && oi < i_)) { v_ = ov; i_ = oi; c_ = oc; }
      }
      if (lane == 0) { sm.red_sum[wid] = s1; sm.red_cum[wid] = s2; sm.red_bv[wid] = v_; sm.red_bi[wid] = i_; sm.red_bc[wid] = c_; }
      __syncthreads();
      if (wid == 0) {
        s1 = sm.red_sum[lane]; s2 = sm.red_cum[lane]; v_ = sm.red_bv[lane]; i_ = sm.red_bi[lane]; c_ = sm.red_bc[lane];
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          s1 += __shfl_xor_sync(0xffffffffu, s1, o);
          s2 += __shfl_xor_sync(0xffffffffu, s2, o);
          const float ov = __shfl_xor_sync(0xffffffffu, v_, o);
          const int oi = __shfl_xor_sync(0xffffffffu, i_, o);
          const uint32_t oc = __shfl_xor_sync(0xffffffffu, c_, o);
          if (ov > v_ || (ov == v_ && oi < i_)) { v_ = ov; i_ = oi; c_ = oc; }
        }
        if (lane == 0) {
          const long long R = (long long)T - (long long)s1;
          sm.resid = R;
          sm.argmax = i_;
          if ((long long)c_ + R < 1) st->err = 1;      // D6: residual would drop a count below 1
          if (a.mode == 0) {
            sm.cum_t = s2 + (i_ < tok ? R : 0);
            sm.freq_t = sm.freq_t + (i_ == tok ? R : 0);
          } else {
            gsum[i_ >> 2] = (uint32_t)((long long)gsum[i_ >> 2] + R);
          }
        }
      }
      __syncthreads();
    }

    if (a.mode == 1) {
      // ---------------- decode: prefix scan over the groups (in id order), search the target ----
      const long long R = sm.resid;
      const int am = sm.argmax;
      const int gpt = (G + WT - 1) / WT;
      const int g0 = min(G, tid * gpt), g1 = min(G, g0 + gpt);
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
        sm.scan[lane] = y;   // inclusive warp totals
      }
      __syncthreads();
      const unsigned long long excl = (unsigned long long)(x - adj) + (wid ? sm.scan[wid - 1] : 0u);
      const unsigned long long tgt = sm.target;
      if (adj > 0 && tgt >= excl && tgt < excl + adj) {
        unsigned long long accm = excl;
        int gf = g0;
        for (; gf < g1; ++gf) {
          if (tgt < accm + gsum[gf]) break;
          accm += gsum[gf];
        }
        Grp q;
        prob4(gf, q);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int v = 4 * gf + j;
          unsigned long long cv = quant(q.p[j], TmV);
          if (v == am) cv = (unsigned long long)((long long)cv + R);
          if (tgt < accm + cv) {
            sm.tok = v; sm.cum_t = accm; sm.freq_t = cv; sm.pt_t = q.pt[j]; sm.png_t = q.png[j]; sm.p_t = q.p[j];
            break;
          }
          accm += cv;
        }
      }
      if (tid == 0 && tgt >= T) st->err = 2;
      __syncthreads();
      // ---------------- decode: bias update now that t is known ----
      const int t = sm.tok;
      if (use_head)
        for (int g = tid; g < G; g += WT) {
          Grp q;
          prob4(g, q);
          double2 *bp = reinterpret_cast<double2 *>(b) + 2 * g;
          double2 b01 = bp[0], b23 = bp[1];
          const int v = 4 * g;
          b01.x = b_step(b01.x, q.pt[0], v == t, a.alpha);
          b01.y = b_step(b01.y, q.pt[1], v + 1 == t, a.alpha);
          b23.x = b_step(b23.x, q.pt[2], v + 2 == t, a.alpha);
          b23.y = b_step(b23.y, q.pt[3], v + 3 == t, a.alpha);
          bp[0] = b01; bp[1] = b23;
        }
    }

    // ---------------- phase D: outputs, coder, mixer (thread 0), N-gram update (warp 0) ----
    __syncthreads();
    const int t = sm.tok;
    if (tid == 0) {
      const size_t oi = (size_t)a.tok_off[c] + i;
      if (a.mode == 0) {
        a.out_cum[oi] = (uint32_t)sm.cum_t;
        a.out_freq[oi] = (uint32_t)sm.freq_t;
        if (a.out_p) a.out_p[oi] = sm.p_t;
      } else {
        if (t < 0) st->err = 3;
        a.out_tok[oi] = (uint32_t)max(t, 0);
        if (a.next_x) a.next_x[c] = (uint32_t)max(t, 0);
        if (a.out_p) a.out_p[oi] = sm.p_t;
        // consume the symbol (D8)
        const unsigned long long R = st->high - st->low + 1;
        unsigned long long lo = st->low, hi = st->low + ((R * (sm.cum_t + sm.freq_t)) >> a.cdf_bits) - 1;
        lo = lo + ((R * sm.cum_t) >> a.cdf_bits);
        unsigned long long val = st->value, bp = st->bitpos;
        const uint8_t *s = a.streams + a.stream_off[c];
        const unsigned long long nb = a.stream_bits[c];
        for (;;) {
          if (hi < HALF) {
          } else if (lo >= HALF) { lo -= HALF; hi -= HALF; val -= HALF; }
          else if (lo >= QTR && hi < 3 * QTR) { lo -= QTR; hi -= QTR; val -= QTR; }
          else break;
          lo = 2 * lo; hi = 2 * hi + 1;
          const unsigned long long bit = bp < nb ? (s[bp >> 3] >> (7 - (bp & 7))) & 1u : 0u;
          val = 2 * val + bit;
          ++bp;
        }
        st->low = lo; st->high = hi; st->value = val; st->bitpos = bp;
      }
      if (mix) {   // exponential-weights update, log clamp 1e-12
        double l0 = __dadd_rn(st->lw[0], __dmul_rn(a.eta, log(fmax((double)sm.pt_t, 1e-12))));
        double l1 = __dadd_rn(st->lw[1], __dmul_rn(a.eta, log(fmax((double)sm.png_t, 1e-12))));
        const double mx = fmax(l0, l1);
        const double lse = __dadd_rn(mx, log(__dadd_rn(exp(__dsub_rn(l0, mx)), exp(__dsub_rn(l1, mx)))));
        st->lw[0] = __dsub_rn(l0, lse);
        st->lw[1] = __dsub_rn(l1, lse);
      }
    }
    if (wid == 0) {
      // clear this step's fixups
      const int nsp = sm.sp_n;
      for (int k = lane; k < nsp; k += 32) {
        const uint32_t tk = sm.sp_tok[k];
        spadd[tk] = 0.f;
        bitmap[tk >> 5] = 0u;
      }
      if (use_ng && t >= 0) {
        uint32_t hist[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) hist[j] = st->hist[j];
        for (int k = 1; k <= (int)a.orders; ++k) {
          if (i < (uint32_t)k) continue;
          const size_t tb = ((size_t)c * kMaxOrders + (k - 1));
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
          }
          NgRecord *R = a.ng_recs + tb * a.rcap + r;
          const uint32_t ns = R->nslot;
          const bool h0 = (uint32_t)lane < ns && R->tok[lane] == (uint32_t)t;
          const bool h1 = (uint32_t)lane + 32 < ns && R->tok[lane + 32] == (uint32_t)t;
          const unsigned m0 = __ballot_sync(0xffffffffu, h0), m1 = __ballot_sync(0xffffffffu, h1);
          if (m0 | m1) {
            if (h0) R->cnt[lane] += 1;
            if (h1) R->cnt[lane + 32] += 1;
          } else if (ns < kSlots) {
            if (lane == 0) { R->tok[ns] = (uint32_t)t; R->cnt[ns] = 1; R->nslot = ns + 1; }
          } else {   // evict the lowest count, ties -> lowest slot (D21)
            uint32_t bcnt = R->cnt[lane], bidx = lane;
            if (R->cnt[lane + 32] < bcnt) { bcnt = R->cnt[lane + 32]; bidx = lane + 32; }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
              const uint32_t oc = __shfl_xor_sync(0xffffffffu, bcnt, o), oi2 = __shfl_xor_sync(0xffffffffu, bidx, o);
              if (oc < bcnt || (oc == bcnt && oi2 < bidx)) { bcnt = oc; bidx = oi2; }
            }
            if (lane == 0) { R->tok[bidx] = (uint32_t)t; R->cnt[bidx] = 1; }
          }
          if (lane == 0) R->n += 1;
          __syncwarp();
        }
        if (lane == 0) {
          cu[t] += 1u;
          st->N += 1;
        }
      }
      if (lane == 0) {
        st->hist[0] = st->hist[1]; st->hist[1] = st->hist[2]; st->hist[2] = st->hist[3];
        st->hist[3] = (uint32_t)max(t, 0);
        st->i = i + 1;
      }
    }
    __syncthreads();
  }
}

void launch_walk(const WalkArgs &a, cudaStream_t s) {
  if (a.n_entries <= 0) return;
  const size_t dyn = ((a.V + 31) / 32 + a.V / 4) * sizeof(uint32_t);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(walk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  walk_kernel<<<a.n_entries, WT, dyn, s>>>(a);
}

__global__ void walk_init_kernel(WalkState *st, int n, double lw0, double lw1) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  WalkState w;
  memset(&w, 0, sizeof(w));
  w.lw[0] = lw0; w.lw[1] = lw1;
  w.high = 0xFFFFFFFFull;
  st[c] = w;
}
void launch_walk_init(WalkState *st, int n_chunks, cudaStream_t s) {
  if (n_chunks <= 0) return;
  walk_init_kernel<<<(n_chunks + 127) / 128, 128, 0, s>>>(st, n_chunks, std::log(0.85), std::log(0.15));
}

// -------------------------------------------------- debug quantizer (D5) ---
__global__ void quantize_debug_kernel(const float *p, uint32_t V, uint32_t bits, uint32_t *counts) {
  __shared__ unsigned long long rs[NW];
  __shared__ float rv[NW]; __shared__ int ri[NW];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const double TmV = (double)((1ull << bits) - V);
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
