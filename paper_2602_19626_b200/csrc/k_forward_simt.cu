// Forward-pass kernels, SIMT fp32 generation (v1).
//
// Every kernel is batch-invariant per row (fixed reduction orders, no split-K,
// explicit __fmaf_rn), so the prefill and the decode step compute bit-identical
// logits for the same row (hard part H1).
//
//   embed        h = E[x]                                   (eq:lm input)
//   rms          rinv = 1/sqrt(mean(h^2) + eps)              (RMSNorm, D16)
//   gemm<EPI>    C = rinv * (A B^T) with fused epilogues:
//                  QKV    RoPE(q,k) at absolute positions (D12), q -> buffer, k/v -> KV ring
//                  RESID  h += A B^T                         (O-proj, down-proj)
//                  SWIGLU act = silu(g) * u                  (gate/up interleaved by 32 rows)
//                  HEAD   logits = rinv * (h E'^T)            (tied head, final norm folded)
//   attention    block-window causal GQA softmax(q k / 8) v over keys [w(j), j] (D9-D10)
#include <cuda_runtime.h>
#include <math_constants.h>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace nc {

// ------------------------------------------------------------------ embed ---
__global__ void embed_kernel(const uint32_t *__restrict__ x, int M, const float *__restrict__ E, int d,
                             float *__restrict__ h, float *__restrict__ h_hi, float *__restrict__ h_lo) {
  int m = blockIdx.x;
  if (m >= M) return;
  const float4 *src = reinterpret_cast<const float4 *>(E + (size_t)x[m] * d);
  float4 *dst = reinterpret_cast<float4 *>(h + (size_t)m * d);
  for (int i = threadIdx.x; i < d / 4; i += blockDim.x) {
    const float4 v = src[i];
    dst[i] = v;
    if (h_hi) {
      float4 hi, lo;
      tc::split_tf32(v.x, hi.x, lo.x); tc::split_tf32(v.y, hi.y, lo.y);
      tc::split_tf32(v.z, hi.z, lo.z); tc::split_tf32(v.w, hi.w, lo.w);
      reinterpret_cast<float4 *>(h_hi + (size_t)m * d)[i] = hi;
      reinterpret_cast<float4 *>(h_lo + (size_t)m * d)[i] = lo;
    }
  }
}
void launch_embed(const uint32_t *x, int M, const float *E, int d, float *h, float *h_hi, float *h_lo,
                  cudaStream_t s) {
  if (M > 0) embed_kernel<<<M, 128, 0, s>>>(x, M, E, d, h, h_hi, h_lo);
}

// -------------------------------------------------------------------- rms ---
__global__ void rms_kernel(const float *__restrict__ h, int M, int d, float eps, float *__restrict__ rinv) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= M) return;
  const float *row = h + (size_t)warp * d;
  float s = 0.f;
  for (int i = lane; i < d; i += 32) s = __fmaf_rn(row[i], row[i], s);
#pragma unroll
  for (int o = 16; o; o >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
  if (lane == 0) rinv[warp] = __frsqrt_rn(__fadd_rn(__fdiv_rn(s, (float)d), eps));
}
void launch_rms(const float *h, int M, int d, float eps, float *rinv, cudaStream_t s) {
  if (M > 0) rms_kernel<<<(M + 7) / 8, 256, 0, s>>>(h, M, d, eps, rinv);
}

// ------------------------------------------------------------------- gemm ---
// CTA tile 128x128, BK = 16, 256 threads, 8x8 outputs per thread.  Thread
// (tx, ty): rows ty*4+{0..3} and 64+ty*4+{0..3}; columns hb*64 + q*4 + {0..3}
// and hb*64 + 32 + q*4 + {0..3} (hb = tx/8, q = tx%8), so every thread holds
// both halves of a rotate-half RoPE pair and of a 32-interleaved gate/up pair.
constexpr int BM = 128, BN = 128, BK = 16;

template <int EPI>
__global__ __launch_bounds__(256) void gemm_simt_kernel(GemmArgs a) {
  __shared__ __align__(16) float As[BK][BM + 4];
  __shared__ __align__(16) float Bs[BK][BN + 4];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int lr = tid >> 2, lk = (tid & 3) * 4;

  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  float4 ra[2], rb[2];
  auto load = [&](int k0) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      int r = m0 + lr + 64 * u, c = n0 + lr + 64 * u;
      ra[u] = (r < a.M) ? *reinterpret_cast<const float4 *>(a.A + (size_t)r * a.lda + k0 + lk)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
      rb[u] = (c < a.N) ? *reinterpret_cast<const float4 *>(a.B + (size_t)c * a.ldb + k0 + lk)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  load(0);
  for (int k0 = 0; k0 < a.K; k0 += BK) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      As[lk + 0][lr + 64 * u] = ra[u].x; As[lk + 1][lr + 64 * u] = ra[u].y;
      As[lk + 2][lr + 64 * u] = ra[u].z; As[lk + 3][lr + 64 * u] = ra[u].w;
      Bs[lk + 0][lr + 64 * u] = rb[u].x; Bs[lk + 1][lr + 64 * u] = rb[u].y;
      Bs[lk + 2][lr + 64 * u] = rb[u].z; Bs[lk + 3][lr + 64 * u] = rb[u].w;
    }
    __syncthreads();
    if (k0 + BK < a.K) load(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[8], bv[8];
      float4 t0 = *reinterpret_cast<const float4 *>(&As[kk][ty * 4]);
      float4 t1 = *reinterpret_cast<const float4 *>(&As[kk][64 + ty * 4]);
      float4 u0 = *reinterpret_cast<const float4 *>(&Bs[kk][(tx >> 3) * 64 + (tx & 7) * 4]);
      float4 u1 = *reinterpret_cast<const float4 *>(&Bs[kk][(tx >> 3) * 64 + 32 + (tx & 7) * 4]);
      av[0] = t0.x; av[1] = t0.y; av[2] = t0.z; av[3] = t0.w;
      av[4] = t1.x; av[5] = t1.y; av[6] = t1.z; av[7] = t1.w;
      bv[0] = u0.x; bv[1] = u0.y; bv[2] = u0.z; bv[3] = u0.w;
      bv[4] = u1.x; bv[5] = u1.y; bv[6] = u1.z; bv[7] = u1.w;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = __fmaf_rn(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }

  // ---------------------------------------------------------------- epilogue
  const int cb = n0 + (tx >> 3) * 64;          // 64-wide column block of this thread
  const int cq = (tx & 7) * 4;                 // offset inside the first half
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (m >= a.M || cb >= a.N) continue;
    if (EPI == EPI_RESID) {
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float4 *p = reinterpret_cast<float4 *>(a.C + (size_t)m * a.ldc + cb + half * 32 + cq);
        float4 o = *p;
        o.x = __fadd_rn(o.x, acc[i][half * 4 + 0]); o.y = __fadd_rn(o.y, acc[i][half * 4 + 1]);
        o.z = __fadd_rn(o.z, acc[i][half * 4 + 2]); o.w = __fadd_rn(o.w, acc[i][half * 4 + 3]);
        *p = o;
      }
    } else {
      const float rs = a.rinv[m];
      float x[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = __fmul_rn(acc[i][j], rs);
      if (EPI == EPI_HEAD) {
#pragma unroll
        for (int half = 0; half < 2; ++half)
          *reinterpret_cast<float4 *>(a.C + (size_t)m * a.ldc + cb + half * 32 + cq) =
              make_float4(x[half * 4], x[half * 4 + 1], x[half * 4 + 2], x[half * 4 + 3]);
      } else if (EPI == EPI_SWIGLU) {
        float y[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float g = x[j], u = x[j + 4];
          float sg = __fdiv_rn(g, __fadd_rn(1.f, expf(-g)));
          y[j] = __fmul_rn(sg, u);
        }
        *reinterpret_cast<float4 *>(a.C + (size_t)m * a.ldc + cb / 2 + cq) = make_float4(y[0], y[1], y[2], y[3]);
      } else {  // EPI_QKV
        const int pos = a.rows.pos[m];
        if (pos < 0) continue;
        const int nq = a.n_q_cols, nkv = a.n_kv_cols;
        if (cb < nq + nkv) {  // q or k: RoPE on the rotate-half pairs (d, d+32)
          const float *cs = a.rope_cos + (size_t)pos * 32 + cq;
          const float *sn = a.rope_sin + (size_t)pos * 32 + cq;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float c = cs[j], s = sn[j], x1 = x[j], x2 = x[j + 4];
            x[j] = __fmaf_rn(x1, c, __fmul_rn(-x2, s));
            x[j + 4] = __fmaf_rn(x2, c, __fmul_rn(x1, s));
          }
        }
        float *dst;
        if (cb < nq) {
          dst = a.C + (size_t)m * a.ldc + cb;
        } else {
          const int c = a.rows.chunk[m];
          const bool isk = cb < nq + nkv;
          const int kvh = (cb - nq - (isk ? 0 : nkv)) / 64;
          dst = (isk ? a.ring.k : a.ring.v) + a.ring.off(c, a.layer, pos) + kvh * 64;
        }
        *reinterpret_cast<float4 *>(dst + cq) = make_float4(x[0], x[1], x[2], x[3]);
        *reinterpret_cast<float4 *>(dst + 32 + cq) = make_float4(x[4], x[5], x[6], x[7]);
      }
    }
  }
}

void launch_gemm(GemmEpi epi, const GemmArgs &a, cudaStream_t s) {
  if (a.M <= 0) return;
  dim3 grid((a.N + BN - 1) / BN, (a.M + BM - 1) / BM);
  switch (epi) {
    case EPI_QKV: gemm_simt_kernel<EPI_QKV><<<grid, 256, 0, s>>>(a); break;
    case EPI_RESID: gemm_simt_kernel<EPI_RESID><<<grid, 256, 0, s>>>(a); break;
    case EPI_SWIGLU: gemm_simt_kernel<EPI_SWIGLU><<<grid, 256, 0, s>>>(a); break;
    case EPI_HEAD: gemm_simt_kernel<EPI_HEAD><<<grid, 256, 0, s>>>(a); break;
  }
}

// -------------------------------------------------------------- attention ---
// One CTA per (tile of <=64 consecutive rows of one chunk, kv head).  Thread =
// (row, q head of the group).  Keys are processed in 64-key blocks aligned to
// absolute positions (ring slots), 16-key online-softmax sub-steps; a row skips
// every key after itself, so its arithmetic does not depend on the tile.
__device__ __forceinline__ int window_start_dev(int j, int L, int C) {
  int over = j + 1 - L;
  return over <= 0 ? 0 : C * ((over + C - 1) / C);
}

__global__ __launch_bounds__(192) void attention_kernel(AttnArgs a) {
  __shared__ __align__(16) float Ks[64][64];
  __shared__ __align__(16) float Vs[64][64];
  const AttnTile t = a.tiles[blockIdx.x];
  const int g = blockIdx.y, rep = a.H / a.KV;
  const int r = threadIdx.x & 63, hq = g * rep + (threadIdx.x >> 6);
  const bool valid = r < t.nrows && (threadIdx.x >> 6) < rep;
  const int j = t.p0 + r;

  float q[64], acc[64];
  if (valid) {
    const float4 *qp = reinterpret_cast<const float4 *>(a.q + (size_t)(t.qrow0 + r) * a.ldq + hq * 64);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float4 v = qp[i];
      q[4 * i] = v.x; q[4 * i + 1] = v.y; q[4 * i + 2] = v.z; q[4 * i + 3] = v.w;
    }
  }
#pragma unroll
  for (int d = 0; d < 64; ++d) acc[d] = 0.f;
  float m = -CUDART_INF_F, l = 0.f;

  const int w = window_start_dev(t.p0, a.window, a.slide);
  const int kb0 = w / 64, kb1 = (t.p0 + t.nrows - 1) / 64;
  for (int kb = kb0; kb <= kb1; ++kb) {
    __syncthreads();
    for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) {
      const int kk = i >> 4, c4 = i & 15;
      const size_t off = a.ring.off(t.chunk, a.layer, kb * 64 + kk) + g * 64;
      reinterpret_cast<float4 *>(&Ks[kk][0])[c4] = reinterpret_cast<const float4 *>(a.ring.k + off)[c4];
      reinterpret_cast<float4 *>(&Vs[kk][0])[c4] = reinterpret_cast<const float4 *>(a.ring.v + off)[c4];
    }
    __syncthreads();
    if (!valid || kb * 64 > j) continue;
    const int kmax = min(63, j - kb * 64);
    for (int sub = 0; sub < 4; ++sub) {
      if (sub * 16 > kmax) break;
      float s[16];
      float mb = -CUDART_INF_F;
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        const int key = sub * 16 + kk;
        float dot = 0.f;
        if (key <= kmax) {
#pragma unroll
          for (int d = 0; d < 64; ++d) dot = __fmaf_rn(q[d], Ks[key][d], dot);
          dot = __fmul_rn(dot, 0.125f);
        } else {
          dot = -CUDART_INF_F;
        }
        s[kk] = dot;
        mb = fmaxf(mb, dot);
      }
      const float mn = fmaxf(m, mb);
      const float sc = expf(__fsub_rn(m, mn));   // m = -inf on the first step -> 0
      l = __fmul_rn(l, sc);
#pragma unroll
      for (int d = 0; d < 64; ++d) acc[d] = __fmul_rn(acc[d], sc);
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        const int key = sub * 16 + kk;
        if (key > kmax) break;
        const float p = expf(__fsub_rn(s[kk], mn));
        l = __fadd_rn(l, p);
#pragma unroll
        for (int d = 0; d < 64; ++d) acc[d] = __fmaf_rn(p, Vs[key][d], acc[d]);
      }
      m = mn;
    }
  }
  if (valid) {
    const size_t ob = (size_t)(t.qrow0 + r) * a.ldq + hq * 64;
    float4 *op = reinterpret_cast<float4 *>(a.o + ob);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float4 v = make_float4(__fdiv_rn(acc[4 * i], l), __fdiv_rn(acc[4 * i + 1], l),
                                   __fdiv_rn(acc[4 * i + 2], l), __fdiv_rn(acc[4 * i + 3], l));
      op[i] = v;
      if (a.o_hi) {
        float4 hi, lo;
        tc::split_tf32(v.x, hi.x, lo.x); tc::split_tf32(v.y, hi.y, lo.y);
        tc::split_tf32(v.z, hi.z, lo.z); tc::split_tf32(v.w, hi.w, lo.w);
        reinterpret_cast<float4 *>(a.o_hi + ob)[i] = hi;
        reinterpret_cast<float4 *>(a.o_lo + ob)[i] = lo;
      }
    }
  }
}

void launch_attention(const AttnArgs &a, cudaStream_t s) {
  if (a.n_tiles <= 0) return;
  dim3 grid(a.n_tiles, a.KV);
  attention_kernel<<<grid, 64 * (a.H / a.KV), 0, s>>>(a);
}

}  // namespace nc
