// Per-SM global store throughput of the GEMM epilogue's pattern (diagnostics):
// 148 CTAs x W warps, each warp writes R rows x 32 floats as 8 x (4 rows x 128 B) float4 stores
// into P planes (like store_rows32<ST_RESID>: h, hi, lo), rows strided by ld floats.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/store_bw store_bw.cu && /tmp/store_bw
#include <cstdio>
#include <cuda_runtime.h>

__global__ void st_kernel(float *out, int ld, int rows_per_warp, int planes, size_t plane_stride, int reps) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int c4 = lane & 7;
  for (int rep = 0; rep < reps; ++rep)
    for (int rb = 0; rb < rows_per_warp; rb += 32)
      for (int i = 0; i < 8; ++i) {
        const int r = (blockIdx.x * nw + warp) * rows_per_warp + rb + 4 * i + (lane >> 3);
        float4 v = make_float4(r, rep, i, lane);
        for (int p = 0; p < planes; ++p)
          *reinterpret_cast<float4 *>(out + p * plane_stride + (size_t)r * ld + 32 * (rep % 18) + 4 * c4) = v;
      }
}

int main() {
  const int ld = 576, W = 12, rows_per_warp = 32 * 6, planes = 3, reps = 6;
  const int M = 148 * W * rows_per_warp;
  size_t plane = (size_t)M * ld;
  float *out;
  cudaMalloc(&out, plane * planes * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int t = 0; t < 3; ++t) {
    cudaEventRecord(a);
    st_kernel<<<148, W * 32>>>(out, ld, rows_per_warp, planes, plane, reps);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double bytes = (double)148 * W * rows_per_warp * 32 * 4 * planes * reps;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("stores %.1f MB in %.3f ms: %.2f TB/s, %.1f B/cycle/SM (at %.2f GHz nominal)\n", bytes / 1e6, ms,
           bytes / ms / 1e9, bytes / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1e6);
  }
  return 0;
}
