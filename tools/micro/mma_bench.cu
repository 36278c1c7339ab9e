// Microbenchmark: cycles per tcgen05.mma.kind::tf32 (M=128, K=8) vs N and vs the
// number of independent accumulators the issue stream rotates over.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2602_19626_b200/csrc mma_bench.cu
#include <cstdio>
#include <cstdint>
#include "tc_common.cuh"
using namespace nc;

template <int M, int N, int MODE>
__global__ void bench(int n_acc, int reps, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  if (warp == 0) tc::tmem_alloc(&tslot, 512);
  tc::fence_before(); __syncthreads(); tc::fence_after();
  const uint32_t tm = tslot;
  if (threadIdx.x == 32) {
    const uint32_t a = tc::smem_u32(sm), b = tc::smem_u32(sm + 16384);
    constexpr uint32_t id = MODE == 2 ? ((1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24))
                                      : tc::idesc_tf32(M, N);
    const uint64_t da = tc::desc_k_sw128(a), db = tc::desc_k_sw128(b);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const int acc = r % n_acc;
      if (MODE == 0) tc::mma_tf32(tm + acc * N, da, db, id, r >= n_acc);
      else if (MODE == 1) tc::mma_tf32_ts(tm + acc * N, tm + 256 + 0, db, id, r >= n_acc);
      else {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm + acc * N),
                     "l"(da), "l"(db), "r"(id), "r"((uint32_t)(r >= n_acc)));
      }
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[0] = t1 - t0;
  }
  tc::fence_before(); __syncthreads(); tc::fence_after();
  if (warp == 0) tc::tmem_dealloc(tm, 512);
}

template <int M, int N, int MODE> void run(int n_acc) {
  long long *d, h;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(bench<M, N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int reps = 512;
  bench<M, N, MODE><<<1, 64, 48 * 1024>>>(n_acc, reps, d);   // warm
  bench<M, N, MODE><<<1, 64, 48 * 1024>>>(n_acc, reps, d);
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const char *nm[] = {"tf32 SS", "tf32 TS", "bf16 SS K16"};
  printf("%-12s M=%3d N=%3d acc=%d  cycles/MMA=%6.1f  flop/cycle=%6.0f  %s\n", nm[MODE], M, N, n_acc, (double)h / reps,
         2.0 * M * N * (MODE == 2 ? 16 : 8) / ((double)h / reps), cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<128, 64, 0>(1); run<128, 128, 0>(1); run<128, 256, 0>(1); run<128, 256, 0>(2);
  run<64, 64, 0>(1); run<64, 128, 0>(1); run<64, 256, 0>(1);
  run<128, 64, 1>(1); run<128, 128, 1>(1); run<128, 256, 1>(1);
  run<128, 64, 2>(1); run<128, 128, 2>(1); run<128, 256, 2>(1); run<128, 256, 2>(2);
  return 0;
}
