// The forward's memory-bound row kernel (the contractions run on the tensor cores:
// k_gemm_tc.cu, k_attn_tc.cu).
//
// It is batch-invariant per row (fixed reduction orders, explicit __fmaf_rn), so the
// prefill and the decode step compute bit-identical logits for the same row (D15).
//
//   embed        h = E[x], its tf32 hi/lo planes and h's RMSNorm scale rinv (eq:lm input,
//                P:277-282).  RMSNorm (D16) has no kernel of its own: every residual GEMM
//                epilogue also forms the new h's rinv (k_gemm_tc.cu), the consuming GEMM
//                (QKV, gate/up, head) scales its rows by it; the gain is folded into that
//                projection's weights.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <stdexcept>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace nc {

// ------------------------------------------------------------------ embed ---
// h = E[x], its tf32 planes, and the RMSNorm statistics of h: the sum of squares of every
// 32-column slice, ssq[m][s] (same per-slice arithmetic as the GEMM's residual epilogue,
// store_rows32: per float4 ((x^2 + y^2) + z^2) + w^2, then an xor tree over the slice's
// 8 float4s) and rinv = 1/sqrt(sum_s ssq[s] / d + eps) (slices in order, as the residual
// epilogue's last warp forms it).  One CTA of 128 threads per row; d % 32 == 0, d <= 2048.
// ssq != nullptr enables the statistics (the slice sums stay in shared memory).
__global__ void embed_kernel(const uint32_t *__restrict__ x, int M, const float *__restrict__ E, int d,
                             float *__restrict__ h, float *__restrict__ h_hi, float *__restrict__ h_lo,
                             float *__restrict__ ssq, float *__restrict__ rinv, float eps) {
  __shared__ float part[64];   // d <= 2048
  int m = blockIdx.x;
  if (m >= M) return;
  const float4 *src = reinterpret_cast<const float4 *>(E + (size_t)x[m] * d);
  float4 *dst = reinterpret_cast<float4 *>(h + (size_t)m * d);
  for (int base = 0; base < d / 4; base += blockDim.x) {   // uniform trip count: every lane shuffles
    const int i = base + threadIdx.x;
    const bool ok = i < d / 4;
    const float4 v = ok ? src[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    if (ok) {
      dst[i] = v;
      if (h_hi) {
        float4 hi, lo;
        tc::split_tf32(v.x, hi.x, lo.x); tc::split_tf32(v.y, hi.y, lo.y);
        tc::split_tf32(v.z, hi.z, lo.z); tc::split_tf32(v.w, hi.w, lo.w);
        reinterpret_cast<float4 *>(h_hi + (size_t)m * d)[i] = hi;
        reinterpret_cast<float4 *>(h_lo + (size_t)m * d)[i] = lo;
      }
    }
    if (ssq) {
      float t = __fmaf_rn(v.w, v.w, __fmaf_rn(v.z, v.z, __fmaf_rn(v.y, v.y, __fmul_rn(v.x, v.x))));
      t = __fadd_rn(t, __shfl_xor_sync(0xffffffffu, t, 1));
      t = __fadd_rn(t, __shfl_xor_sync(0xffffffffu, t, 2));
      t = __fadd_rn(t, __shfl_xor_sync(0xffffffffu, t, 4));
      if (ok && (i & 7) == 0) part[i / 8] = t;
    }
  }
  if (ssq) {
    __syncthreads();
    if (threadIdx.x == 0) {
      float ss = 0.f;
      for (int k = 0; k < d / 32; ++k) ss = __fadd_rn(ss, part[k]);
      rinv[m] = __frsqrt_rn(__fadd_rn(__fdiv_rn(ss, (float)d), eps));
    }
  }
}
void launch_embed(const uint32_t *x, int M, const float *E, int d, float *h, float *h_hi, float *h_lo, float *ssq,
                  float *rinv, float eps, cudaStream_t s) {
  if (d > 2048) throw std::runtime_error("embed: d_model > 2048");
  if (M > 0) embed_kernel<<<M, 128, 0, s>>>(x, M, E, d, h, h_hi, h_lo, ssq, rinv, eps);
}

}  // namespace nc
