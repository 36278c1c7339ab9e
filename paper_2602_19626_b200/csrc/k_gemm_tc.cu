// fp32-accurate GEMM on the 5th-gen tensor cores: 3xTF32 with tcgen05.mma
// kind::tf32 (SURVEY.md D14 / hard part H2), operands staged by TMA, the
// accumulator in TMEM, and the layer's epilogue fused on the TMEM read-out.
//
//   C[m, n] = epi( sum_k A[m,k] B[n,k] ),  A = A_hi + A_lo, B = B_hi + B_lo (tf32 planes)
//   per 32-wide k block: D = sum_k (A_hi B_lo + A_lo B_hi), then D += sum_k A_hi B_hi (fixed order)
//
// Precision: every tcgen05.mma that accumulates into D rounds the sum toward
// zero (measured: relative bias -1.6e-5 at K = 1536 on positive data, i.e.
// ~0.5 ulp per MMA; tools/gemm_precision.py).  So each 32-wide k block is
// accumulated in a FRESH TMEM partial (12 MMAs) and the epilogue warps add the
// partials in fp32 round-to-nearest registers ("promotion"), which restores
// ~fp32 accuracy (D14).
//
// Persistent, warp-specialised CTA (256 threads, 1 CTA / SM):
//   warp 0  TMA producer (one thread): 4 tiles per stage (A_hi, A_lo, B_hi, B_lo), 3 stages
//   warp 1  MMA issuer  (one thread): 12 tcgen05.mma per 32-wide k block into a partial buffer
//   warp 2  TMEM allocator (4 x 128 fp32 columns: rotating partial buffers)
//   warps 4-7 promotion + epilogue: tcgen05.ld partials -> fp32 RN sums -> fused epilogue -> global
// Tiles 128 x 128 are claimed dynamically (atomic counter; the last CTA to exit
// resets it), so CTAs that start late -- e.g. on SMs a concurrently running walk
// held -- find no work instead of stalling the GEMM.  Claim order streams the
// larger operand once: M-fastest when there are at least as many N tiles as M
// tiles (weights / vocab head), N-fastest otherwise (A tile reused from L2).
//
// Row results do not depend on which other rows share the tile (each output
// element is one fixed sequence of MMAs), so prefill and decode agree bit for
// bit (D15).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>

#include "gemm_tc.cuh"
#include "tc_common.cuh"

namespace nc {

constexpr int TBM = 128, TBN = 128, TBK = 32, TSTAGES = 3, NPART = 4, NSCHED = 4;
constexpr int TILE_A_BYTES = TBM * TBK * 4;   // 16 KB
constexpr int TILE_B_BYTES = TBN * TBK * 4;   // 16 KB
constexpr int STAGE_BYTES = 2 * TILE_A_BYTES + 2 * TILE_B_BYTES;
constexpr int TC_SMEM = TSTAGES * STAGE_BYTES + 1024 /*align*/ + 512 /*barriers, schedule*/;
constexpr int TC_THREADS = 256;

template <int EPI>
__global__ __launch_bounds__(TC_THREADS, 1) void gemm_tc_kernel(const __grid_constant__ CUtensorMap tmAh,
                                                                const __grid_constant__ CUtensorMap tmAl,
                                                                const __grid_constant__ CUtensorMap tmBh,
                                                                const __grid_constant__ CUtensorMap tmBl,
                                                                TcGemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + TSTAGES * STAGE_BYTES);
  uint64_t *empty = full + TSTAGES;
  uint64_t *tfull = empty + TSTAGES;
  uint64_t *tempty = tfull + NPART;
  uint64_t *sch_full = tempty + NPART, *sch_empty = sch_full + NSCHED;
  int *sch_tile = reinterpret_cast<int *>(sch_empty + NSCHED);
  uint32_t *tmem_base_smem = reinterpret_cast<uint32_t *>(sch_tile + NSCHED);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_m = (a.M + TBM - 1) / TBM, num_n = (a.N + TBN - 1) / TBN;
  const int n_tiles = num_m * num_n;
  const int nk = a.K / TBK;
  const bool m_fast = num_n >= num_m;
  auto tile_mn = [&](int t, int &mb, int &nb) {
    if (m_fast) { mb = t % num_m; nb = t / num_m; } else { nb = t % num_n; mb = t / num_n; }
  };

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmAh); tc::tma_prefetch(&tmAl); tc::tma_prefetch(&tmBh); tc::tma_prefetch(&tmBl);
    for (int s = 0; s < TSTAGES; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
    for (int s = 0; s < NPART; ++s) { tc::mbar_init(&tfull[s], 1); tc::mbar_init(&tempty[s], 4); }
    for (int s = 0; s < NSCHED; ++s) { tc::mbar_init(&sch_full[s], 1); tc::mbar_init(&sch_empty[s], 5); }
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc(tmem_base_smem, NPART * TBN);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem_base = *tmem_base_smem;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int jt = 0;; ++jt) {
        const int slot = jt % NSCHED;
        tc::mbar_wait(&sch_empty[slot], ((jt / NSCHED) & 1) ^ 1);
        const int claimed = atomicAdd(a.tile_ctr, 1);
        const int t = claimed < n_tiles ? claimed : -1;
        sch_tile[slot] = t;
        tc::mbar_arrive(&sch_full[slot]);
        if (t < 0) break;
        int mb, nb;
        tile_mn(t, mb, nb);
        for (int kb = 0; kb < nk; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t *st = smem + stage * STAGE_BYTES;
          tc::mbar_expect_tx(&full[stage], STAGE_BYTES);
          tc::tma_load_2d(st, &tmAh, kb * TBK, mb * TBM, &full[stage]);
          tc::tma_load_2d(st + TILE_A_BYTES, &tmAl, kb * TBK, mb * TBM, &full[stage]);
          tc::tma_load_2d(st + 2 * TILE_A_BYTES, &tmBh, kb * TBK, nb * TBN, &full[stage]);
          tc::tma_load_2d(st + 2 * TILE_A_BYTES + TILE_B_BYTES, &tmBl, kb * TBK, nb * TBN, &full[stage]);
          if (++stage == TSTAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_tf32(TBM, TBN);
      int stage = 0;
      uint32_t phase = 0;
      int buf = 0;
      uint32_t buf_phase = 0;
      for (int jt = 0;; ++jt) {
        const int slot = jt % NSCHED;
        tc::mbar_wait(&sch_full[slot], (jt / NSCHED) & 1);
        const int t = sch_tile[slot];
        tc::mbar_arrive(&sch_empty[slot]);
        if (t < 0) break;
        for (int kb = 0; kb < nk; ++kb) {
          tc::mbar_wait(&tempty[buf], buf_phase ^ 1);     // partial buffer drained by the epilogue
          tc::mbar_wait(&full[stage], phase);
          tc::fence_after();
          const uint32_t d = tmem_base + buf * TBN;
          const uint32_t s0 = tc::smem_u32(smem + stage * STAGE_BYTES);
          const uint64_t dah = tc::desc_k_sw128(s0), dal = tc::desc_k_sw128(s0 + TILE_A_BYTES);
          const uint64_t dbh = tc::desc_k_sw128(s0 + 2 * TILE_A_BYTES);
          const uint64_t dbl = tc::desc_k_sw128(s0 + 2 * TILE_A_BYTES + TILE_B_BYTES);
          // the small correction products first, hi*hi last: each accumulate rounds
          // toward zero relative to the running sum, which stays ~2^-11 smaller
          // while the corrections are added (4 large-magnitude truncations, not 12)
#pragma unroll
          for (int j = 0; j < TBK / 8; ++j) {
            const uint64_t adv = (uint64_t)(j * 32) >> 4;   // 8 tf32 = 32 bytes along K
            tc::mma_tf32(d, dah + adv, dbl + adv, idesc, j != 0);
            tc::mma_tf32(d, dal + adv, dbh + adv, idesc, 1);
          }
#pragma unroll
          for (int j = 0; j < TBK / 8; ++j) {
            const uint64_t adv = (uint64_t)(j * 32) >> 4;
            tc::mma_tf32(d, dah + adv, dbh + adv, idesc, 1);
          }
          tc::mma_commit(&empty[stage]);
          tc::mma_commit(&tfull[buf]);
          if (++stage == TSTAGES) { stage = 0; phase ^= 1; }
          if (++buf == NPART) { buf = 0; buf_phase ^= 1; }
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- epilogue
    const int q = warp & 3;   // TMEM lanes 32q .. 32q+31
    int buf = 0;
    uint32_t buf_phase = 0;
    for (int jt = 0;; ++jt) {
      const int slot = jt % NSCHED;
      tc::mbar_wait(&sch_full[slot], (jt / NSCHED) & 1);
      const int t = sch_tile[slot];
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&sch_empty[slot]);
      if (t < 0) break;
      int mb, nb;
      tile_mn(t, mb, nb);
      float acc[TBN];
#pragma unroll
      for (int j = 0; j < TBN; ++j) acc[j] = 0.f;
      for (int kb = 0; kb < nk; ++kb) {
        tc::mbar_wait(&tfull[buf], buf_phase);
        tc::fence_after();
        const uint32_t taddr = tmem_base + buf * TBN + ((uint32_t)(q * 32) << 16);
#pragma unroll
        for (int c = 0; c < TBN / 32; ++c) {
          uint32_t r[32];
          tc::tmem_ld32(taddr + c * 32, r);
          tc::tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[c * 32 + j] = __fadd_rn(acc[c * 32 + j], __uint_as_float(r[j]));
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&tempty[buf]);
        if (++buf == NPART) { buf = 0; buf_phase ^= 1; }
      }
      const int m = mb * TBM + q * 32 + lane;
      const bool row_ok = m < a.M;
      const float rs = (EPI != EPI_RESID && row_ok && a.rinv) ? a.rinv[m] : 1.f;
#pragma unroll
      for (int half = 0; half < TBN / 64; ++half) {
        const int cb = nb * TBN + half * 64;        // first column of this 64-wide block
        if (!row_ok || cb >= a.N) continue;
        float x[64];
#pragma unroll
        for (int j = 0; j < 64; ++j) x[j] = acc[half * 64 + j];
        if (EPI == EPI_RESID) {
          float *hp = a.C + (size_t)m * a.ldc + cb;
          float *hh = a.C_hi + (size_t)m * a.ldc + cb;
          float *hl = a.C_lo + (size_t)m * a.ldc + cb;
#pragma unroll
          for (int j = 0; j < 64; j += 4) {
            float4 o = *reinterpret_cast<float4 *>(hp + j);
            o.x = __fadd_rn(o.x, x[j]); o.y = __fadd_rn(o.y, x[j + 1]);
            o.z = __fadd_rn(o.z, x[j + 2]); o.w = __fadd_rn(o.w, x[j + 3]);
            *reinterpret_cast<float4 *>(hp + j) = o;
            float4 h4, l4;
            tc::split_tf32(o.x, h4.x, l4.x); tc::split_tf32(o.y, h4.y, l4.y);
            tc::split_tf32(o.z, h4.z, l4.z); tc::split_tf32(o.w, h4.w, l4.w);
            *reinterpret_cast<float4 *>(hh + j) = h4;
            *reinterpret_cast<float4 *>(hl + j) = l4;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 64; ++j) x[j] = __fmul_rn(x[j], rs);
          if (EPI == EPI_HEAD) {
            float *dst = a.C + (size_t)m * a.ldc + cb;
#pragma unroll
            for (int j = 0; j < 64; j += 4)
              *reinterpret_cast<float4 *>(dst + j) = make_float4(x[j], x[j + 1], x[j + 2], x[j + 3]);
          } else if (EPI == EPI_SWIGLU) {
            // columns [cb, cb+32) are gate rows, [cb+32, cb+64) the matching up rows
            float *dh = a.C_hi + (size_t)m * a.ldc + cb / 2;
            float *dl = a.C_lo + (size_t)m * a.ldc + cb / 2;
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              float4 h4, l4;
              float y[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const float g = x[j + u], up = x[32 + j + u];
                const float sg = __fdiv_rn(g, __fadd_rn(1.f, expf(-g)));
                y[u] = __fmul_rn(sg, up);
              }
              tc::split_tf32(y[0], h4.x, l4.x); tc::split_tf32(y[1], h4.y, l4.y);
              tc::split_tf32(y[2], h4.z, l4.z); tc::split_tf32(y[3], h4.w, l4.w);
              *reinterpret_cast<float4 *>(dh + j) = h4;
              *reinterpret_cast<float4 *>(dl + j) = l4;
            }
          } else {  // EPI_QKV
            const int pos = a.rows.pos[m];
            if (pos >= 0) {
              const int nq = a.n_q_cols, nkv = a.n_kv_cols;
              if (cb < nq + nkv) {   // q or k head: RoPE on the rotate-half pairs (d, d+32)
                const float *cs = a.rope_cos + (size_t)pos * 32;
                const float *sn = a.rope_sin + (size_t)pos * 32;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                  const float c = cs[j], s = sn[j], x1 = x[j], x2 = x[j + 32];
                  x[j] = __fmaf_rn(x1, c, __fmul_rn(-x2, s));
                  x[j + 32] = __fmaf_rn(x2, c, __fmul_rn(x1, s));
                }
              }
              if (a.planes) {
                float *dh, *dl;
                if (cb < nq) {
                  dh = a.C_hi + (size_t)m * a.ldc + cb;
                  dl = a.C_lo + (size_t)m * a.ldc + cb;
                } else {
                  const int ch = a.rows.chunk[m];
                  const bool isk = cb < nq + nkv;
                  const int kvh = (cb - nq - (isk ? 0 : nkv)) / 64;
                  const size_t o = a.ring.off(ch, a.layer, pos) + kvh * 64;
                  dh = (isk ? a.ring.k_hi : a.ring.v_hi) + o;
                  dl = (isk ? a.ring.k_lo : a.ring.v_lo) + o;
                }
#pragma unroll
                for (int j = 0; j < 64; j += 4) {
                  float4 h4, l4;
                  tc::split_tf32(x[j], h4.x, l4.x); tc::split_tf32(x[j + 1], h4.y, l4.y);
                  tc::split_tf32(x[j + 2], h4.z, l4.z); tc::split_tf32(x[j + 3], h4.w, l4.w);
                  *reinterpret_cast<float4 *>(dh + j) = h4;
                  *reinterpret_cast<float4 *>(dl + j) = l4;
                }
              } else {
                float *dst;
                if (cb < nq) {
                  dst = a.C + (size_t)m * a.ldc + cb;
                } else {
                  const int ch = a.rows.chunk[m];
                  const bool isk = cb < nq + nkv;
                  const int kvh = (cb - nq - (isk ? 0 : nkv)) / 64;
                  dst = (isk ? a.ring.k : a.ring.v) + a.ring.off(ch, a.layer, pos) + kvh * 64;
                }
#pragma unroll
                for (int j = 0; j < 64; j += 4)
                  *reinterpret_cast<float4 *>(dst + j) = make_float4(x[j], x[j + 1], x[j + 2], x[j + 3]);
              }
            }
          }
        }
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 2) tc::tmem_dealloc(tmem_base, NPART * TBN);
  if (threadIdx.x == 0) {            // last CTA out resets the tile counter for the next launch
    __threadfence();
    if (atomicAdd(a.tile_ctr + 1, 1) == (int)gridDim.x - 1) {
      a.tile_ctr[0] = 0;
      a.tile_ctr[1] = 0;
      __threadfence();
    }
  }
}

// ------------------------------------------------------------- host side ---
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// fp32 [rows, cols] row-major, box [box_rows, 32 cols], 128B swizzle; cached per (ptr, shape).
const CUtensorMap *tmap_2d(const float *ptr, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  struct Key {
    const void *p; uint64_t r, c; uint32_t b;
    bool operator==(const Key &o) const { return p == o.p && r == o.r && c == o.c && b == o.b; }
  };
  struct H {
    size_t operator()(const Key &k) const {
      return std::hash<const void *>()(k.p) ^ (k.r * 0x9E3779B97F4A7C15ull) ^ (k.c << 20) ^ k.b;
    }
  };
  static std::mutex mu;
  static std::unordered_map<Key, CUtensorMap, H> cache;
  std::lock_guard<std::mutex> lk(mu);
  Key k{ptr, rows, cols, box_rows};
  auto it = cache.find(k);
  if (it != cache.end()) return &it->second;
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 4};
  cuuint32_t box[2] = {TBK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return &cache.emplace(k, m).first->second;
}

static int g_reserved_sms = 0;
void set_reserved_sms(int n) { g_reserved_sms = n; }

static int *tile_counter() {   // {next tile, CTAs done}; zero between launches
  static int *ctr = nullptr;
  if (!ctr) {
    if (cudaMalloc(&ctr, 2 * sizeof(int)) != cudaSuccess) throw std::runtime_error("cudaMalloc tile counter");
    cudaMemset(ctr, 0, 2 * sizeof(int));
    cudaDeviceSynchronize();
  }
  return ctr;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <int EPI>
static void launch_tc(const TcGemmArgs &a, const TcOperands &op, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_tc_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM);
    attr = true;
  }
  const CUtensorMap *ah = tmap_2d(op.A_hi, op.a_rows, a.K, TBM), *al = tmap_2d(op.A_lo, op.a_rows, a.K, TBM);
  const CUtensorMap *bh = tmap_2d(op.B_hi, a.N, a.K, TBN), *bl = tmap_2d(op.B_lo, a.N, a.K, TBN);
  const int tiles = ((a.M + TBM - 1) / TBM) * ((a.N + TBN - 1) / TBN);
  const int grid = std::min(tiles, std::max(1, num_sms() - g_reserved_sms));
  TcGemmArgs aa = a;
  aa.tile_ctr = tile_counter();
  gemm_tc_kernel<EPI><<<grid, TC_THREADS, TC_SMEM, s>>>(*ah, *al, *bh, *bl, aa);
}

void launch_gemm_tc(GemmEpi epi, const TcGemmArgs &a, const TcOperands &op, cudaStream_t s) {
  if (a.M <= 0) return;
  if (a.K % TBK) throw std::runtime_error("tcgen05 GEMM needs K % 32 == 0");
  switch (epi) {
    case EPI_QKV: launch_tc<EPI_QKV>(a, op, s); break;
    case EPI_RESID: launch_tc<EPI_RESID>(a, op, s); break;
    case EPI_SWIGLU: launch_tc<EPI_SWIGLU>(a, op, s); break;
    case EPI_HEAD: launch_tc<EPI_HEAD>(a, op, s); break;
  }
}

// ------------------------------------------------------- plane helpers ---
__global__ void split_planes_kernel(const float *__restrict__ x, float *__restrict__ hi, float *__restrict__ lo,
                                    size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float h, l;
    tc::split_tf32(x[i], h, l);
    hi[i] = h;
    lo[i] = l;
  }
}
void launch_split_planes(const float *x, float *hi, float *lo, size_t n, cudaStream_t s) {
  if (n) split_planes_kernel<<<(unsigned)std::min<size_t>((n + 255) / 256, 4096), 256, 0, s>>>(x, hi, lo, n);
}

}  // namespace nc
