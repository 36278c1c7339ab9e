// cycles per MMA under load for the attention PV shapes: one CTA (M = 128) vs a CTA pair
// (M = 256, cta_group::2), N = 64 and 128, A from TMEM (TS) with MN-major B, and SS K-major.
// Per pair the leader issues; reported cycles are per dispatch (each SM computes 128 x N x 8).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2602_19626_b200/csrc mma_bench4.cu
#include <cstdio>
#include <cstdint>
#include "tc_common.cuh"
using namespace nc;

__device__ __forceinline__ uint64_t desc_mn(uint32_t saddr, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)(512u >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;
  return d;
}
__device__ __forceinline__ void mma_ts_pair(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
               "r"(a), "l"(b), "r"(id), "r"(acc));
}

// MODE 0: SS K-major; 1: TS + MN-major B
template <int PAIR, int MODE, int N>
__global__ void rate(int reps, long long *out) {
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
    const uint32_t a = tc::smem_u32(sm), b = tc::smem_u32(sm + 65536);
    const uint32_t M = PAIR ? 256 : 128;
    const uint32_t id = tc::idesc_tf32(M, N) | (MODE == 1 ? (1u << 16) : 0u);
    const uint64_t da = tc::desc_k_sw128(a);
    const uint64_t db = MODE == 1 ? desc_mn(b, 8192) : tc::desc_k_sw128(b);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t d = tm + (r & 1) * 128;
      if (MODE == 0) {
        if (PAIR) tc::mma_tf32_pair(d, da, db, id, r >= 2);
        else tc::mma_tf32(d, da, db, id, r >= 2);
      } else {
        if (PAIR) mma_ts_pair(d, tm + 256 + (r & 7) * 8, db, id, r >= 2);
        else tc::mma_tf32_ts(d, tm + 256 + (r & 7) * 8, db, id, r >= 2);
      }
    }
    if (PAIR) tc::mma_commit_pair(&bar); else tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  if (PAIR && rank == 1 && threadIdx.x == 32) { tc::mbar_wait(&bar, 0); out[blockIdx.x] = 0; }
  tc::fence_before(); if (PAIR) tc::cluster_sync(); else __syncthreads(); tc::fence_after();
  if (warp == 0) { if (PAIR) tc::tmem_dealloc_pair(tm, 512); else tc::tmem_dealloc(tm, 512); }
}

template <int PAIR, int MODE, int N> void run(int nsm, long long *d) {
  long long h[1024];
  const int reps = 4096;
  auto k = rate<PAIR, MODE, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3(nsm); cfg.blockDim = dim3(64); cfg.dynamicSmemBytes = 160 * 1024;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = PAIR ? 2 : 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  for (int p = 0; p < 2; ++p) { cudaLaunchKernelEx(&cfg, k, reps, d); cudaDeviceSynchronize(); }
  cudaMemcpy(h, d, nsm * 8, cudaMemcpyDeviceToHost);
  double s = 0; int n = 0;
  for (int i = 0; i < nsm; ++i) if (h[i]) { s += h[i]; ++n; }
  printf("%s %-14s N=%3d: %.1f cycles/dispatch, %.0f MAC/cycle/SM  (%s)\n", PAIR ? "pair M256" : "cta  M128",
         MODE ? "TS, B MN-maj" : "SS K-major", N, s / n / reps, 128.0 * N * 8 / (s / n / reps),
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long *d; cudaMalloc(&d, 1024 * 8);
  cudaMemset(d, 0, 1024 * 8);
  run<0, 0, 128>(nsm, d); run<1, 0, 128>(nsm, d);
  run<0, 1, 64>(nsm, d); run<1, 1, 64>(nsm, d);
  run<0, 0, 64>(nsm, d); run<1, 0, 64>(nsm, d);
  run<0, 1, 128>(nsm, d); run<1, 1, 128>(nsm, d);
  return 0;
}
