// cycles per MMA under load (148 CTAs) for the attention's operand forms:
//  SS K-major (S = Q K^T), TS with MN-major B (O = P V, P from TMEM), N = 64 / 128.
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

template <int MODE, int N, int CHAIN = 0, int VARY = 0>   // MODE 0: SS K-major; 1: TS + MN-major B; 2: SS + MN-major B; 3: TS + K-major B
__global__ void rate(int reps, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  if (warp == 0) tc::tmem_alloc(&tslot, 512);
  tc::fence_before(); __syncthreads(); tc::fence_after();
  const uint32_t tm = tslot;
  if (threadIdx.x == 32) {
    const uint32_t a = tc::smem_u32(sm), b = tc::smem_u32(sm + 65536);
    const uint32_t id = tc::idesc_tf32(128, N) | ((MODE == 1 || MODE == 2) ? (1u << 16) : 0u);
    const uint64_t da = tc::desc_k_sw128(a);
    const uint64_t db = (MODE == 1 || MODE == 2) ? desc_mn(b, 8192) : tc::desc_k_sw128(b);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t d = CHAIN ? tm : tm + (r & 1) * 128;
      // VARY: walk the operands over 8 x 16 B steps of K (1024 B span of swizzled rows) like a real k loop,
      // and over 4 distinct 16 KB tiles
      const uint64_t va = VARY ? (uint64_t)(((r & 3) * 32 + ((r >> 2) & 3) * 16384) >> 4) : 0;
      const uint64_t vb = VARY ? (uint64_t)(((r & 3) * 32) >> 4) : 0;
      if (MODE == 0 || MODE == 2) tc::mma_tf32(d, da + va, db + vb, id, CHAIN ? (r > 0) : (r >= 2));
      else tc::mma_tf32_ts(d, tm + 256 + (r & 7) * 8, db, id, r >= 2);
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc::fence_before(); __syncthreads(); tc::fence_after();
  if (warp == 0) tc::tmem_dealloc(tm, 512);
}

template <int MODE, int N, int CHAIN = 0, int VARY = 0> void run(int nsm, long long *d) {
  long long h[1024];
  const int reps = 2048;
  cudaFuncSetAttribute(rate<MODE, N, CHAIN, VARY>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  for (int p = 0; p < 2; ++p) { rate<MODE, N, CHAIN, VARY><<<nsm, 64, 96 * 1024>>>(reps, d); cudaDeviceSynchronize(); }
  cudaMemcpy(h, d, nsm * 8, cudaMemcpyDeviceToHost);
  double s = 0; for (int i = 0; i < nsm; ++i) s += h[i];
  const char *nm[] = {"SS K-major", "TS, B MN-major", "SS, B MN-major", "TS, B K-major"};
  printf("%-16s N=%3d chain=%d vary=%d: %.1f cycles/MMA  (%s)\n", nm[MODE], N, CHAIN, VARY, s / nsm / reps, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long *d; cudaMalloc(&d, 1024 * 8);
  run<0, 64>(nsm, d); run<0, 64, 1>(nsm, d); run<0, 64, 0, 1>(nsm, d); run<0, 64, 1, 1>(nsm, d);
  run<0, 128, 1, 1>(nsm, d); run<0, 256, 1, 1>(nsm, d);
  run<1, 64>(nsm, d); run<1, 64, 1>(nsm, d);
  return 0;
}
