// The forward's two memory-bound row kernels (the contractions run on the tensor cores:
// k_gemm_tc.cu, k_attn_tc.cu).
//
// Both are batch-invariant per row (fixed reduction orders, explicit __fmaf_rn), so the
// prefill and the decode step compute bit-identical logits for the same row (D15).
//
//   embed        h = E[x] and its tf32 hi/lo planes          (eq:lm input)
//   rms          rinv = 1/sqrt(mean(h^2) + eps)              (RMSNorm, D16; the gain is folded
//                                                             into the following projection)
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

}  // namespace nc
