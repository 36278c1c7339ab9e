// (a) cycles per MMA with all SMs busy: 1-CTA M128 N256 vs CTA-pair M256 N256 (tf32)
// (b) TMA streaming rate: every CTA streams `stage_kb` tiles through a 3-deep ring from an
//     L2-resident buffer (no MMA), reports bytes/cycle per SM.
#include <cstdio>
#include <cstdint>
#include <cudaTypedefs.h>
#include "tc_common.cuh"
using namespace nc;

template <int PAIR, int N = 256>
__global__ void mma_rate(int reps, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = PAIR ? tc::cluster_ctarank() : 0;
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  if (warp == 0) { if (PAIR) tc::tmem_alloc_pair(&tslot, 512); else tc::tmem_alloc(&tslot, 512); }
  tc::fence_before(); if (PAIR) tc::cluster_sync(); else __syncthreads(); tc::fence_after();
  const uint32_t tm = tslot;
  if (threadIdx.x == 32 && rank == 0) {
    const uint32_t a = tc::smem_u32(sm), b = tc::smem_u32(sm + 16384);
    const uint64_t da = tc::desc_k_sw128(a), db = tc::desc_k_sw128(b);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (PAIR) tc::mma_tf32_pair(tm + (r & 1) * 256, da, db, tc::idesc_tf32(256, 256), r >= 2);
      else tc::mma_tf32(tm + (r & 1) * 256, da, db, tc::idesc_tf32(128, N), r >= 2);
    }
    if (PAIR) tc::mma_commit_pair(&bar); else tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  } else if (threadIdx.x == 32 && rank == 1) {
    tc::mbar_wait(&bar, 0);
  }
  tc::fence_before(); if (PAIR) tc::cluster_sync(); else __syncthreads(); tc::fence_after();
  if (warp == 0) { if (PAIR) tc::tmem_dealloc_pair(tm, 512); else tc::tmem_dealloc(tm, 512); }
}

// TMA stream: box 32 fp32 x 128 rows (16 KB); a stage = n_box boxes; 3 stages
__global__ void tma_rate(const __grid_constant__ CUtensorMap m, int n_box, int iters, int rows_total,
                         long long *out) {
  extern __shared__ uint8_t raw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[3];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) tc::mbar_init(&full[i], 1);
    tc::fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int stage_bytes = n_box * 16384;
    long long t0 = clock64();
    int row = (blockIdx.x * 997) % (rows_total / 128);
    for (int it = 0; it < iters + 3; ++it) {
      const int s = it % 3;
      if (it >= 3) tc::mbar_wait(&full[s], ((it - 3) / 3) & 1);
      if (it < iters) {
        tc::mbar_expect_tx(&full[s], stage_bytes);
        for (int b = 0; b < n_box; ++b) {
          tc::tma_load_2d(sm + s * stage_bytes + b * 16384, &m, (b % 8) * 32, row * 128, &full[s]);
          row = (row + 1) % (rows_total / 128);
        }
      }
    }
    out[blockIdx.x] = clock64() - t0;
  }
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long *d; cudaMalloc(&d, 1024 * 8);
  long long h[1024];
  const int reps = 2048;
  cudaFuncSetAttribute(mma_rate<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(mma_rate<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int pass = 0; pass < 2; ++pass) {
    mma_rate<0><<<nsm, 64, 48 * 1024>>>(reps, d);
    cudaDeviceSynchronize();
  }
  cudaMemcpy(h, d, nsm * 8, cudaMemcpyDeviceToHost);
  double s = 0; for (int i = 0; i < nsm; ++i) s += h[i];
  printf("1-CTA M128 N256, %d CTAs: %.1f cycles/MMA  (%s)\n", nsm, s / nsm / reps, cudaGetErrorString(cudaGetLastError()));
  for (int pass = 0; pass < 2; ++pass) {
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(nsm); cfg.blockDim = dim3(64); cfg.dynamicSmemBytes = 48 * 1024;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1; cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, mma_rate<1>, reps, d);
    cudaDeviceSynchronize();
  }
  cudaMemcpy(h, d, nsm * 8, cudaMemcpyDeviceToHost);
  s = 0; for (int i = 0; i < nsm; i += 2) s += h[i];
  printf("pair M256 N256, %d pairs: %.1f cycles/MMA per pair  (%s)\n", nsm / 2, s / (nsm / 2) / reps,
         cudaGetErrorString(cudaGetLastError()));

  {
    cudaFuncSetAttribute(mma_rate<0, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(mma_rate<0, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int pass = 0; pass < 2; ++pass) { mma_rate<0, 64><<<nsm, 64, 48 * 1024>>>(reps, d); cudaDeviceSynchronize(); }
    cudaMemcpy(h, d, nsm * 8, cudaMemcpyDeviceToHost);
    s = 0; for (int i = 0; i < nsm; ++i) s += h[i];
    printf("1-CTA M128 N64, %d CTAs: %.1f cycles/MMA\n", nsm, s / nsm / reps);
    for (int pass = 0; pass < 2; ++pass) { mma_rate<0, 128><<<nsm, 64, 48 * 1024>>>(reps, d); cudaDeviceSynchronize(); }
    cudaMemcpy(h, d, nsm * 8, cudaMemcpyDeviceToHost);
    s = 0; for (int i = 0; i < nsm; ++i) s += h[i];
    printf("1-CTA M128 N128, %d CTAs: %.1f cycles/MMA\n", nsm, s / nsm / reps);
    for (int pass = 0; pass < 2; ++pass) { mma_rate<0, 64><<<1, 64, 48 * 1024>>>(reps, d); cudaDeviceSynchronize(); }
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("1-CTA M128 N64, 1 CTA: %.1f cycles/MMA\n", (double)h[0] / reps);
    for (int pass = 0; pass < 2; ++pass) { mma_rate<0, 256><<<1, 64, 48 * 1024>>>(reps, d); cudaDeviceSynchronize(); }
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("1-CTA M128 N256, 1 CTA: %.1f cycles/MMA  %s\n", (double)h[0] / reps, cudaGetErrorString(cudaGetLastError()));
  }
  // TMA stream from a 64 MB buffer (L2 resident after the first pass)
  const int rows = 65536, cols = 256;   // 64 MB fp32
  float *buf; cudaMalloc(&buf, (size_t)rows * cols * 4); cudaMemset(buf, 0, (size_t)rows * cols * 4);
  PFN_cuTensorMapEncodeTiled_v12000 enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}; cuuint64_t str[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {32, 128}; cuuint32_t es[2] = {1, 1};
  enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(tma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int nb : {4, 6}) {
    for (int grid : {nsm / 2, nsm}) {
      const int iters = 400;
      for (int pass = 0; pass < 2; ++pass) { tma_rate<<<grid, 32, 3 * nb * 16384 + 1024>>>(m, nb, iters, rows, d); cudaDeviceSynchronize(); }
      cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
      double mx = 0, av = 0; for (int i = 0; i < grid; ++i) { av += h[i]; if (h[i] > mx) mx = h[i]; }
      av /= grid;
      printf("TMA stream: %3d CTAs, stage %3d KB: %.1f B/cycle/SM (avg), chip %.0f B/cycle (at slowest CTA)  (%s)\n", grid,
             nb * 16, (double)iters * nb * 16384 / av, (double)grid * iters * nb * 16384 / mx,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
