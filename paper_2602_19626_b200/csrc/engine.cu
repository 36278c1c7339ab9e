// Engine: model upload, the slabbed prefill + walk driver (compress), the
// one-row-per-chunk decode-step driver (decompress), host WNC + NC05 assembly.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <thread>

#include <nvtx3/nvToolsExt.h>

#include "engine.hpp"
#include "attn_tc.cuh"
#include "gemm_tc.cuh"

namespace nc {

// NVTX ranges around the host-side phases (visible in nsys / ncu --nvtx; header-only NVTX3,
// a no-op unless a tool injects itself)
struct Nvtx {
  explicit Nvtx(const char *name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

void check_cuda(cudaError_t e, const char *what) {
  if (e != cudaSuccess) fail(NC_ERR_BACKEND, std::string(what) + ": " + cudaGetErrorString(e));
}
void throw_launch_error(cudaError_t e, const char *what) {
  cudaGetLastError();   // clear the sticky-free launch error
  fail(NC_ERR_BACKEND, std::string(what) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------- allocator ---
static void *(*g_alloc)(size_t, void *) = nullptr;
static void (*g_free)(void *, void *) = nullptr;
static void *g_ctx = nullptr;
void set_allocator(void *(*a)(size_t, void *), void (*f)(void *, void *), void *ctx) {
  g_alloc = a; g_free = f; g_ctx = ctx;
}
// Default device allocator: a grow-only caching pool over cudaMalloc.  Every
// call allocates the same buffer sizes, so after the first call nothing is
// mapped or unmapped again (cudaMallocAsync with a zero release threshold
// re-mapped GBs of slab buffers per call).  Blocks are returned after the
// owning call has synchronised its stream.
struct DevCache {   // keyed by (device, size): a block is only reused on the device it lives on
  std::mutex mu;
  std::multimap<std::pair<int, size_t>, void *> free_;
  std::map<void *, std::pair<int, size_t>> size_;
};
static DevCache &cache() {
  static DevCache c;
  return c;
}
void *dev_alloc(size_t bytes, cudaStream_t s) {
  (void)s;
  if (bytes == 0) bytes = 16;
  bytes = (bytes + 255) & ~size_t(255);
  void *p = nullptr;
  if (g_alloc) {
    p = g_alloc(bytes, g_ctx);
    if (!p) fail(NC_ERR_NOMEM, "device allocation failed (hook)");
    return p;
  }
  DevCache &c = cache();
  int dev = 0;
  NC_CUDA(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.free_.lower_bound({dev, bytes});
    if (it != c.free_.end() && it->first.first == dev && it->first.second <= 2 * bytes) {
      p = it->second;
      c.free_.erase(it);
      return p;
    }
  }
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    // release this device's cached blocks and retry once
    std::lock_guard<std::mutex> lk(c.mu);
    for (auto it = c.free_.lower_bound({dev, 0}); it != c.free_.end() && it->first.first == dev;) {
      cudaFree(it->second);
      c.size_.erase(it->second);
      it = c.free_.erase(it);
    }
    e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) fail(NC_ERR_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  }
  std::lock_guard<std::mutex> lk(c.mu);
  c.size_[p] = {dev, bytes};
  return p;
}
void dev_free(void *p, cudaStream_t s) {
  (void)s;
  if (!p) return;
  if (g_free) { g_free(p, g_ctx); return; }
  DevCache &c = cache();
  std::lock_guard<std::mutex> lk(c.mu);
  auto it = c.size_.find(p);
  if (it == c.size_.end()) return;
  c.free_.insert({it->second, p});
}

Stats &stats() {
  static thread_local Stats st;
  return st;
}

Prof &prof() {
  static Prof p;
  return p;
}
cudaEvent_t Prof::ev() {
  if (used == pool.size()) {
    cudaEvent_t e;
    NC_CUDA(cudaEventCreate(&e));
    pool.push_back(e);
  }
  return pool[used++];
}
void Prof::begin(int cls, double w, cudaStream_t s) {
  if (!on) return;
  Rec r{cls, ev(), ev(), w};
  NC_CUDA(cudaEventRecord(r.a, s));
  recs.push_back(r);
}
void Prof::end(cudaStream_t s) {
  if (!on) return;
  NC_CUDA(cudaEventRecord(recs.back().b, s));
}
void Prof::collect() {
  for (auto &r : recs) {
    float t = 0;
    NC_CUDA(cudaEventSynchronize(r.b));
    NC_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    n[r.cls]++;
    ms[r.cls] += t;
    work[r.cls] += r.work;
  }
  recs.clear();
  used = 0;
}
void Prof::reset() {
  recs.clear();
  used = 0;
  for (int i = 0; i < K_NCLASS; ++i) { n[i] = 0; ms[i] = 0; work[i] = 0; }
}
#define PROF(cls, w, call)            \
  do {                                \
    prof().begin((cls), (w), s);      \
    call;                             \
    prof().end(s);                    \
  } while (0)

// RAII bag of device buffers for one call.  The buffers go back to the pool only after
// every stream that may still use them (the call's stream plus any registered with
// also()) has drained -- also on the error path.
struct Bag {
  cudaStream_t s;
  std::vector<cudaStream_t> extra;
  std::vector<void *> ptrs;
  explicit Bag(cudaStream_t st) : s(st) {}
  void also(cudaStream_t x) { extra.push_back(x); }
  template <class T>
  T *get(size_t n) {
    T *p = static_cast<T *>(dev_alloc(n * sizeof(T), s));
    ptrs.push_back(p);
    return p;
  }
  template <class T>
  T *upload(const std::vector<T> &v) {
    T *p = get<T>(v.size());
    if (!v.empty()) NC_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    return p;
  }
  ~Bag() {
    cudaStreamSynchronize(s);
    for (cudaStream_t x : extra) cudaStreamSynchronize(x);
    for (void *p : ptrs) dev_free(p, s);
    cudaStreamSynchronize(s);
  }
};
// RAII set of CUDA events (destroyed on every path)
struct Events {
  std::vector<cudaEvent_t> ev;
  explicit Events(size_t n) : ev(n, nullptr) {
    for (auto &e : ev) NC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDefault));
  }
  ~Events() {
    for (auto &e : ev)
      if (e) cudaEventDestroy(e);
  }
  cudaEvent_t &operator[](size_t i) { return ev[i]; }
};

// ---------------------------------------------------------- token check ---
__global__ void token_max_kernel(const uint32_t *t, size_t n, uint32_t *mx) {
  uint32_t m = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    m = max(m, t[i]);
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) atomicMax(mx, m);
}
void check_tokens_device(nc_model *m, const uint32_t *tokens_dev, size_t n, cudaStream_t s) {
  if (n == 0) return;
  NC_CUDA(cudaSetDevice(m->device));
  uint32_t *mx = static_cast<uint32_t *>(dev_alloc(4, s));
  uint32_t h = 0;
  cudaError_t e = cudaMemsetAsync(mx, 0, 4, s);
  if (e == cudaSuccess) {
    token_max_kernel<<<(unsigned)std::min<size_t>((n + 255) / 256, 1184), 256, 0, s>>>(tokens_dev, n, mx);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, mx, 4, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  dev_free(mx, s);
  NC_CUDA(e);
  stats().launches++;
  if (h >= m->s.V) fail(NC_ERR_INVALID, "token id " + std::to_string(h) + " >= vocabulary size");
}

// ------------------------------------------------------------------ model ---
void model_load(nc_model *m, const std::string &path, int device) {
  NcwFile f = read_ncw(path);
  model_setup(m, f, device);
}

void model_load_hf(nc_model *m, const std::string &dir, int device) {
  NcwFile f = read_hf(dir, m->bpe);
  model_setup(m, f, device);
}

void model_setup(nc_model *m, const NcwFile &f, int device) {
  Nvtx nv("nc.model upload");
  const Shape &s = f.s;
  if (s.dh != (uint32_t)kHeadDim) fail(NC_ERR_INVALID, "kernels are specialised to head_dim 64");
  if (s.H % s.KV || s.H / s.KV > 3) fail(NC_ERR_INVALID, "GQA group must be <= 3");
  if (s.d % 64 || s.d_ff % 64) fail(NC_ERR_INVALID, "d_model and d_ff must be multiples of 64");
  if (s.V % 128) fail(NC_ERR_INVALID, "vocab must be a multiple of 128");
  NC_CUDA(cudaSetDevice(device));
  m->device = device;
  m->s = s;
  m->vocab = f.vocab;
  m->tok.build(f.vocab, s.n_special);
  const size_t d = s.d, V = s.V, qd = (size_t)s.H * s.dh, kvd = (size_t)s.KV * s.dh, ff = s.d_ff;
  // device memory of the model: through the allocator hook when one is set (nc_set_allocator),
  // else cudaMalloc; released in model_free
  auto alloc = [&](size_t bytes) {
    void *p = nullptr;
    if (g_alloc) {
      p = g_alloc(bytes, g_ctx);
      if (!p) fail(NC_ERR_NOMEM, "device allocation failed (hook)");
    } else {
      NC_CUDA(cudaMalloc(&p, bytes));
    }
    m->owned.push_back(p);
    m->owned_hook.push_back(g_alloc != nullptr);
    return static_cast<float *>(p);
  };
  // fp32 staging buffer on the device: the tf32 planes are split from it, then it is reused
  size_t stage_n = std::max<size_t>(V * d, 2 * ff * d);
  float *stage = nullptr;
  NC_CUDA(cudaMalloc(&stage, stage_n * sizeof(float)));
  auto planes = [&](const std::vector<float> &h, float *&hi, float *&lo) {
    NC_CUDA(cudaMemcpy(stage, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice));
    hi = alloc(h.size() * 4);
    lo = alloc(h.size() * 4);
    launch_split_planes(stage, hi, lo, h.size(), nullptr);
    NC_CUDA(cudaDeviceSynchronize());
  };
  size_t off = 0;
  const float *E = f.tensor(0);
  off += V * d;
  std::vector<float> buf(E, E + V * d);
  m->E = alloc(V * d * 4);
  NC_CUDA(cudaMemcpy(m->E, buf.data(), V * d * 4, cudaMemcpyHostToDevice));
  m->wqkv_hi.resize(s.n_layers); m->wqkv_lo.resize(s.n_layers); m->wo_hi.resize(s.n_layers);
  m->wo_lo.resize(s.n_layers); m->wgu_hi.resize(s.n_layers); m->wgu_lo.resize(s.n_layers);
  m->wd_hi.resize(s.n_layers); m->wd_lo.resize(s.n_layers);
  for (uint32_t l = 0; l < s.n_layers; ++l) {
    const float *g1 = f.tensor(off); off += d;
    const float *wq = f.tensor(off); off += qd * d;
    const float *wk = f.tensor(off); off += kvd * d;
    const float *wv = f.tensor(off); off += kvd * d;
    const float *wo = f.tensor(off); off += d * qd;
    const float *g2 = f.tensor(off); off += d;
    const float *wg = f.tensor(off); off += ff * d;
    const float *wu = f.tensor(off); off += ff * d;
    const float *wd = f.tensor(off); off += d * ff;
    // [Wq; Wk; Wv] with the attention RMSNorm gain folded into the columns
    buf.assign((qd + 2 * kvd) * d, 0.f);
    for (size_t r = 0; r < qd + 2 * kvd; ++r) {
      const float *src = r < qd ? wq + r * d : (r < qd + kvd ? wk + (r - qd) * d : wv + (r - qd - kvd) * d);
      for (size_t k = 0; k < d; ++k) buf[r * d + k] = src[k] * g1[k];
    }
    planes(buf, m->wqkv_hi[l], m->wqkv_lo[l]);
    buf.assign(wo, wo + d * qd);
    planes(buf, m->wo_hi[l], m->wo_lo[l]);
    // gate/up interleaved in groups of 32 rows, MLP RMSNorm gain folded in
    buf.assign(2 * ff * d, 0.f);
    for (size_t gi = 0; gi < ff / 32; ++gi)
      for (size_t j = 0; j < 32; ++j)
        for (size_t k = 0; k < d; ++k) {
          buf[(64 * gi + j) * d + k] = wg[(32 * gi + j) * d + k] * g2[k];
          buf[(64 * gi + 32 + j) * d + k] = wu[(32 * gi + j) * d + k] * g2[k];
        }
    planes(buf, m->wgu_hi[l], m->wgu_lo[l]);
    buf.assign(wd, wd + d * ff);
    planes(buf, m->wd_hi[l], m->wd_lo[l]);
  }
  const float *gf = f.tensor(off);
  buf.assign(V * d, 0.f);
  for (size_t v = 0; v < V; ++v)
    for (size_t k = 0; k < d; ++k) buf[v * d + k] = E[v * d + k] * gf[k];
  planes(buf, m->E_head_hi, m->E_head_lo);
  cudaFree(stage);
  ensure_rope(m, 4096);
  int lo_prio = 0, hi_prio = 0;
  NC_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
  // the walk is the sequential critical path: its clusters go first when SMs free up
  NC_CUDA(cudaStreamCreateWithPriority(&m->walk_stream, cudaStreamNonBlocking, hi_prio));
  NC_CUDA(cudaStreamCreateWithFlags(&m->ng_stream, cudaStreamNonBlocking));
}

void model_free(nc_model *m) {
  cudaSetDevice(m->device);
  cudaDeviceSynchronize();
  for (size_t i = 0; i < m->owned.size(); ++i) {
    if (i < m->owned_hook.size() && m->owned_hook[i] && g_free) g_free(m->owned[i], g_ctx);
    else cudaFree(m->owned[i]);
  }
  m->owned_hook.clear();
  if (m->rope_cos) cudaFree(m->rope_cos);
  if (m->rope_sin) cudaFree(m->rope_sin);
  if (m->walk_stream) cudaStreamDestroy(m->walk_stream);
  if (m->ng_stream) cudaStreamDestroy(m->ng_stream);
  m->walk_stream = m->ng_stream = nullptr;
  m->owned.clear();
}

// cos/sin of pos * theta^(-2i/64) computed in fp64, stored fp32 (D12)
void ensure_rope(nc_model *m, int64_t max_pos) {
  if (max_pos <= m->rope_len) return;
  if (max_pos > (int64_t)INT32_MAX - 4096) fail(NC_ERR_INVALID, "positions beyond the RoPE table range");
  const int len = (int)(((max_pos + 4095) / 4096) * 4096);
  std::vector<float> c((size_t)len * 32), sn((size_t)len * 32);
  for (int p = 0; p < len; ++p)
    for (int i = 0; i < 32; ++i) {
      double inv = std::pow(m->s.rope_theta, -(2.0 * i) / 64.0);
      double ang = (double)p * inv;
      c[(size_t)p * 32 + i] = (float)std::cos(ang);
      sn[(size_t)p * 32 + i] = (float)std::sin(ang);
    }
  NC_CUDA(cudaDeviceSynchronize());
  if (m->rope_cos) cudaFree(m->rope_cos);
  if (m->rope_sin) cudaFree(m->rope_sin);
  NC_CUDA(cudaMalloc(&m->rope_cos, c.size() * 4));
  NC_CUDA(cudaMalloc(&m->rope_sin, sn.size() * 4));
  NC_CUDA(cudaMemcpy(m->rope_cos, c.data(), c.size() * 4, cudaMemcpyHostToDevice));
  NC_CUDA(cudaMemcpy(m->rope_sin, sn.data(), sn.size() * 4, cudaMemcpyHostToDevice));
  m->rope_len = len;
}

// ---------------------------------------------------------------- forward ---
struct Forward {
  nc_model *m;
  cudaStream_t s;
  int Mmax = 0;
  float *h, *rinv, *logits, *lbuf[2];
  float *ssq; int *rms_ctr;            // RMSNorm statistics of h: slice sums of squares, per-32-row counters
  float *h_hi, *h_lo, *o_hi, *o_lo, *act_hi, *act_lo;   // tf32 planes (tensor-core GEMM operands)
  float *q_hi = nullptr, *q_lo = nullptr;               // tf32 planes of q (tensor-core attention)
  int n_chunks_ = 0;
  KvRing ring{};
  // shared_ring: use another Forward's KV ring instead of allocating one (refresh re-prefill);
  // with_logits = false: no logits buffer (a forward run without the head)
  void alloc(Bag &bag, int Mmax_, int n_chunks, int ring_len, bool double_logits = false,
             const KvRing *shared_ring = nullptr, bool with_logits = true) {
    Mmax = Mmax_;
    const Shape &S = m->s;
    h = bag.get<float>((size_t)Mmax * S.d);
    rinv = bag.get<float>((size_t)Mmax);
    ssq = bag.get<float>((size_t)(S.d / 32) * ((Mmax + 31) / 32 * 32));   // [slice][row]
    rms_ctr = bag.get<int>((size_t)(Mmax + 31) / 32);
    NC_CUDA(cudaMemsetAsync(rms_ctr, 0, (size_t)(Mmax + 31) / 32 * sizeof(int), s));   // self-resetting
    h_hi = bag.get<float>((size_t)Mmax * S.d);
    h_lo = bag.get<float>((size_t)Mmax * S.d);
    o_hi = bag.get<float>((size_t)Mmax * S.H * S.dh);
    o_lo = bag.get<float>((size_t)Mmax * S.H * S.dh);
    act_hi = bag.get<float>((size_t)Mmax * S.d_ff);
    act_lo = bag.get<float>((size_t)Mmax * S.d_ff);
    logits = lbuf[0] = with_logits ? bag.get<float>((size_t)Mmax * S.V) : nullptr;
    lbuf[1] = double_logits ? bag.get<float>((size_t)Mmax * S.V) : lbuf[0];
    ring.n_layers = S.n_layers;
    ring.ring = ring_len;
    ring.kv = S.KV;
    size_t rn = (size_t)n_chunks * S.n_layers * ring_len * S.KV * S.dh;
    n_chunks_ = n_chunks;
    q_hi = bag.get<float>((size_t)Mmax * S.H * S.dh);
    q_lo = bag.get<float>((size_t)Mmax * S.H * S.dh);
    if (shared_ring) {
      ring = *shared_ring;
      return;
    }
    ring.k_hi = bag.get<float>(rn); ring.k_lo = bag.get<float>(rn);
    ring.v_hi = bag.get<float>(rn); ring.v_lo = bag.get<float>(rn);
    // The PV MMA multiplies masked keys by P = 0; a ring slot not written yet
    // (past the chunk end, or ahead of the decode position) must hold a finite
    // value or 0 * NaN poisons the row.  Masked K slots never reach P.
    NC_CUDA(cudaMemsetAsync(ring.v_hi, 0, rn * sizeof(float), s));
    NC_CUDA(cudaMemsetAsync(ring.v_lo, 0, rn * sizeof(float), s));
  }
  // embed -> n_layers x {QKV, attention, O, gate-up, down} -> head into `logits`.
  // valid = rows that are real tokens (algorithmic work), attn_flops = sum over
  // valid rows of 4*H*dh*n_ctx(j) for one layer.
  // decode_rows: every tile is one row of one chunk (decode steps): the attention packs the
  // q heads of a KV group into one tile's rows
  void run(int M, double valid, double attn_flops, const RowMeta &rows, const AttnTile *tiles, int n_tiles,
           const Params &p, cudaEvent_t ev_head, bool head = true, bool decode_rows = false) {
    const Shape &S = m->s;
    Stats &st = stats();
    const int qd = S.H * S.dh, kvd = S.KV * S.dh;
    const double d = S.d;
    PROF(K_EMBED, 4.0 * d * valid, launch_embed(rows.x, M, m->E, S.d, h, h_hi, h_lo, ssq, rinv, (float)S.eps, s));
    st.launches++;
    // RMSNorm (D16): rinv = 1/sqrt(mean(h^2) + eps) comes with h (the embedding, the residual
    // epilogues); the consuming projection scales its rows by it in its epilogue
    auto norm = [&](TcGemmArgs &g) { g.rinv = rinv; };
    auto stats_out = [&](TcGemmArgs &g) {
      g.ssq_out = ssq; g.ssq_ld = (Mmax + 31) / 32 * 32;
      g.rinv_out = rinv; g.rms_ctr = rms_ctr; g.rms_d = (float)S.d; g.rms_eps = (float)S.eps;
    };
    for (uint32_t l = 0; l < S.n_layers; ++l) {
      {  // RMSNorm scale + QKV + RoPE + KV-ring scatter (q and K/V as tf32 planes)
        TcGemmArgs g{};
        g.M = M; g.N = qd + 2 * kvd; g.K = S.d; norm(g); g.C = nullptr; g.ldc = qd;
        g.layer = (int)l; g.n_q_cols = qd; g.n_kv_cols = kvd; g.rows = rows; g.ring = ring;
        g.rope_cos = m->rope_cos; g.rope_sin = m->rope_sin;
        g.C_hi = q_hi; g.C_lo = q_lo;
        TcOperands op{h_hi, h_lo, (uint64_t)Mmax, m->wqkv_hi[l], m->wqkv_lo[l]};
        PROF(K_QKV, 2.0 * valid * (qd + 2 * kvd) * d, launch_gemm_tc(EPI_QKV, g, op, s));
      }
      {
        AttnTcArgs at{};
        at.tiles = tiles; at.n_tiles = n_tiles; at.q_hi = q_hi; at.q_lo = q_lo; at.ldq = qd; at.q_rows = Mmax;
        at.k_hi = ring.k_hi; at.k_lo = ring.k_lo; at.v_hi = ring.v_hi; at.v_lo = ring.v_lo;
        at.ring = ring.ring; at.n_chunks = n_chunks_; at.n_layers = (int)S.n_layers; at.layer = (int)l;
        at.o_hi = o_hi; at.o_lo = o_lo; at.ldo = qd;
        at.H = S.H; at.KV = S.KV; at.window = (int)p.lmax; at.slide = (int)p.slide;
        at.heads_as_rows = decode_rows ? 1 : 0;
        PROF(K_ATTN, attn_flops, launch_attention_tc(at, s));
      }
      {
        TcGemmArgs g{};
        g.M = M; g.N = S.d; g.K = qd; g.C = h; g.ldc = S.d; g.C_hi = h_hi; g.C_lo = h_lo; stats_out(g);
        TcOperands op{o_hi, o_lo, (uint64_t)Mmax, m->wo_hi[l], m->wo_lo[l]};
        PROF(K_OPROJ, 2.0 * valid * d * qd, launch_gemm_tc(EPI_RESID, g, op, s));
      }
      {
        TcGemmArgs g{};
        g.M = M; g.N = 2 * S.d_ff; g.K = S.d; norm(g); g.C_hi = act_hi; g.C_lo = act_lo; g.ldc = S.d_ff;
        TcOperands op{h_hi, h_lo, (uint64_t)Mmax, m->wgu_hi[l], m->wgu_lo[l]};
        PROF(K_GATEUP, 2.0 * valid * 2 * S.d_ff * d, launch_gemm_tc(EPI_SWIGLU, g, op, s));
        TcGemmArgs g2{};
        g2.M = M; g2.N = S.d; g2.K = S.d_ff; g2.C = h; g2.ldc = S.d; g2.C_hi = h_hi; g2.C_lo = h_lo; stats_out(g2);
        TcOperands op2{act_hi, act_lo, (uint64_t)Mmax, m->wd_hi[l], m->wd_lo[l]};
        PROF(K_DOWN, 2.0 * valid * d * S.d_ff, launch_gemm_tc(EPI_RESID, g2, op2, s));
      }
      st.launches += 5;   // QKV, attention, O, gate/up, down
    }
    if (ev_head) NC_CUDA(cudaEventRecord(ev_head, s));
    if (!head) {
      NC_CUDA(cudaGetLastError());
      return;
    }
    {
      TcGemmArgs g{};
      g.M = M; g.N = S.V; g.K = S.d; norm(g); g.C = logits; g.ldc = S.V;
      TcOperands op{h_hi, h_lo, (uint64_t)Mmax, m->E_head_hi, m->E_head_lo};
      PROF(K_HEAD, 2.0 * valid * S.V * d, launch_gemm_tc(EPI_HEAD, g, op, s));
    }
    st.launches += 1;
    NC_CUDA(cudaGetLastError());
  }
};

static double window_start_h(int64_t j, int64_t L, int64_t C) {
  int64_t over = j + 1 - L;
  return over <= 0 ? 0 : (double)(C * ((over + C - 1) / C));
}
// sum over positions [p0, p1) of n_ctx(j) = j - w(j) + 1
static double ctx_sum(int64_t p0, int64_t p1, int64_t L, int64_t C) {
  double s = 0;
  for (int64_t j = p0; j < p1; ++j) s += (double)j - window_start_h(j, L, C) + 1;
  return s;
}

// ------------------------------------------------------------- slab plan ---
// One forward slab: positions [pos0, pos0 + len) of every chunk (rows c * len + r).  w0 >= 0:
// every row of the slab attends keys [w0, j] (a refresh block, NEXT-4), else w(j) on L_max.
// The walk consumes the positions [out0, out1) of the slab (all of it under retained KV;
// the last C rows of a refresh block).
struct Slab { int pos0, len, w0, out0, out1; };

// Retained KV: full slabs of per_chunk positions while the remainder is large, then the
// remainder split frac / (1 - frac) (128-aligned); few chunks: a geometric plan (below).
// Refresh (NEXT-4): window block b = the rows whose window starts at w_b = b C (b = 0: rows
// [0, L_max); b >= 1: rows [L_max + (b-1) C, L_max + b C)) is evaluated FRESH over positions
// [w_b, block end) with every row's window start w_b, in sub-slabs of <= per_chunk positions
// (the K/V of a sub-slab stay in the ring for the next sub-slab of the same block).
static std::vector<Slab> slab_plan(const Params &p, int max_n, int n_chunks, int per_chunk) {
  std::vector<Slab> out;
  if (max_n <= 0) return out;
  if (p.refresh) {
    const int L = (int)p.lmax, C = (int)p.slide;
    for (int b = 0;; ++b) {
      const int w = b * C;
      const int o0 = b == 0 ? 0 : L + (b - 1) * C, o1 = std::min(max_n, b == 0 ? L : L + b * C);
      if (o0 >= max_n) break;
      for (int q0 = w; q0 < o1; q0 += per_chunk) {
        const int len = std::min(per_chunk, o1 - q0);
        out.push_back(Slab{q0, len, w, std::max(q0, o0), std::max(std::max(q0, o0), q0 + len)});
      }
    }
    return out;
  }
  std::vector<int> plan;
  if (const char *pl = std::getenv("NC_SLAB_PLAN")) {
    for (const char *q = pl; *q;) {
      plan.push_back(std::max(128, std::min(per_chunk, std::atoi(q) / 128 * 128)));
      while (*q && *q != ',') ++q;
      if (*q == ',') ++q;
    }
  } else if (n_chunks <= 2) {
    // Few chunks: the walk (~4 us per position, latency-bound, one cluster per chunk) and
    // the N-gram precompute feeding it (~4 us per token) outlast the forward (~2.8 us per
    // position per chunk at 4,096 rows), so start them early: a small first slab, then
    // doubling up to 4,096 positions -- the walk of a slab then never waits long for its
    // N-gram slab (config2 with 1 chunk: unbounded doubling 185 ms, capped at 2,048 207 ms
    // (the forward of small slabs is inefficient), at 4,096 145 ms).
    int len = 1024;
    for (int pos = 0; pos < max_n; pos += len, len = std::min({per_chunk, 2 * len, 4096})) plan.push_back(len);
  } else {
    const char *fs = std::getenv("NC_SLAB_FRAC");
    const double frac = fs ? std::min(0.95, std::max(0.05, std::atof(fs))) : 0.80;
    int rem = max_n;
    while (frac * rem > per_chunk) {   // full slabs until the last two fit the split
      plan.push_back(per_chunk);
      rem -= per_chunk;
    }
    const int first = ((int)(frac * rem) + 127) / 128 * 128;
    if (rem <= 256 || first >= rem) {
      plan.push_back(rem);
    } else {
      plan.push_back(first);
      plan.push_back(rem - first);
    }
  }
  int pos0 = 0;
  for (size_t k = 0; pos0 < max_n; ++k) {
    const int len = std::min(k < plan.size() ? plan[k] : per_chunk, max_n - pos0);
    out.push_back(Slab{pos0, len, -1, pos0, pos0 + len});
    pos0 += len;
  }
  return out;
}

// attention tiles of rows [a0, a1) of chunk c in a slab: <= 128 rows each, split where the
// window start changes (only happens off 128-row boundaries with L_max = L - 1)
static void push_tiles(std::vector<AttnTile> &tiles, int c, int a0, int a1, int pos0, int len, int w0,
                       const Params &p) {
  const int TR = nc_model::attn_tile_rows();
  for (int b0 = a0; b0 < a1;) {
    int e = std::min(a1, b0 + TR);
    if (w0 < 0)
      for (int j = b0 + 1; j < e; ++j)
        if (window_start_h(j, p.lmax, p.slide) != window_start_h(b0, p.lmax, p.slide)) { e = j; break; }
    tiles.push_back(AttnTile{c, b0, e - b0, c * len + (b0 - pos0), w0});
    b0 = e;
  }
}
// sum over rows [p0, p1) of n_ctx(j) = j - w + 1 (w = w0 of a refresh slab, else w(j))
static double ctx_sum_slab(int64_t p0, int64_t p1, int w0, const Params &p) {
  double s = 0;
  for (int64_t j = p0; j < p1; ++j) s += (double)j - (w0 >= 0 ? (double)w0 : window_start_h(j, p.lmax, p.slide)) + 1;
  return s;
}

// rows of a slab: chunk c's positions [pos0, pos0 + len) are rows c * len + r
__global__ void slab_rows_kernel(const uint32_t *tokens, const int64_t *tok_off, const uint32_t *ntok, int len,
                                 int pos0, int M, uint32_t bos, uint32_t *x, int32_t *chunk, int32_t *pos) {
  int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  int c = m / len, r = m % len, p = pos0 + r;
  bool valid = p < (int)ntok[c];
  x[m] = (!valid || p == 0) ? bos : tokens[tok_off[c] + p - 1];
  chunk[m] = c;
  pos[m] = valid ? p : -1;
}

__global__ void step_rows_kernel(const uint32_t *ntok, int n_chunks, int j, int32_t *chunk, int32_t *pos,
                                 AttnTile *tiles, int32_t *chunk_of, int32_t *row0, int32_t *count) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_chunks) return;
  bool act = j < (int)ntok[c];
  chunk[c] = c;
  pos[c] = act ? j : -1;
  tiles[c] = AttnTile{c, j, act ? 1 : 0, c, -1};
  chunk_of[c] = c;
  row0[c] = c;
  count[c] = act ? 1 : 0;
}

// decode step rows with the step index on the device (graph-replayable): reads j, then bumps it
__global__ void step_rows_dev_kernel(const uint32_t *ntok, int n_chunks, int *jctr, int32_t *chunk, int32_t *pos,
                                     AttnTile *tiles, int32_t *chunk_of, int32_t *row0, int32_t *count) {
  const int j = *jctr;
  for (int c = threadIdx.x; c < n_chunks; c += blockDim.x) {
    const bool act = j < (int)ntok[c];
    chunk[c] = c;
    pos[c] = act ? j : -1;
    tiles[c] = AttnTile{c, j, act ? 1 : 0, c, -1};
    chunk_of[c] = c;
    row0[c] = c;
    count[c] = act ? 1 : 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) *jctr = j + 1;
}

static uint32_t pow2_at_least(uint64_t x) {
  uint32_t p = 32;
  while (p < x) p <<= 1;
  return p;
}

struct WalkBufs {
  WalkState *st;
  double *b;
  uint32_t *cu;
  float *spadd;
  unsigned long long *keys;
  uint32_t *vals;
  NgRecord *recs;
  NgTok *ng_pre = nullptr;
  float *ng_spadd = nullptr;
  uint32_t hcap, rcap, ng_ring = 1;
  // ng_ring > 0: tokens per chunk kept in the precomputed N-gram ring (encode)
  void alloc(Bag &bag, int n_chunks, uint32_t V, uint32_t max_n, const Params &p, cudaStream_t s,
             uint32_t ring = 0) {
    rcap = std::max<uint32_t>(1, std::min<uint32_t>(p.cap, max_n));
    hcap = pow2_at_least(2ull * rcap);
    st = bag.get<WalkState>(n_chunks);
    b = bag.get<double>((size_t)n_chunks * V);
    cu = bag.get<uint32_t>((size_t)n_chunks * V);
    spadd = bag.get<float>((size_t)n_chunks * V);
    keys = bag.get<unsigned long long>((size_t)n_chunks * kMaxOrders * hcap);
    vals = bag.get<uint32_t>((size_t)n_chunks * kMaxOrders * hcap);
    recs = bag.get<NgRecord>((size_t)n_chunks * kMaxOrders * rcap);
    NC_CUDA(cudaMemsetAsync(b, 0, (size_t)n_chunks * V * sizeof(double), s));
    NC_CUDA(cudaMemsetAsync(cu, 0, (size_t)n_chunks * V * sizeof(uint32_t), s));
    NC_CUDA(cudaMemsetAsync(spadd, 0, (size_t)n_chunks * V * sizeof(float), s));
    NC_CUDA(cudaMemsetAsync(keys, 0, (size_t)n_chunks * kMaxOrders * hcap * 8, s));
    if (ring) {
      ng_ring = ring;
      ng_pre = bag.get<NgTok>((size_t)n_chunks * ring);
      ng_spadd = bag.get<float>((size_t)n_chunks * V);
      NC_CUDA(cudaMemsetAsync(ng_spadd, 0, (size_t)n_chunks * V * sizeof(float), s));
    }
    launch_walk_init(st, n_chunks, s);
  }
  void fill(WalkArgs &a, const Params &p, uint32_t V) const {
    a.st = st; a.b = b; a.cu = cu; a.spadd = spadd; a.ng_keys = keys; a.ng_vals = vals; a.ng_recs = recs;
    a.hcap = hcap; a.rcap = rcap; a.ng_pre = ng_pre; a.ng_ring = ng_ring; a.ng_spadd = ng_spadd;
    a.V = V; a.cdf_bits = p.cdf_bits; a.warmup = p.warmup; a.flags = p.flags; a.orders = p.orders; a.cap = p.cap;
    a.inv_tau = (float)p.inv_tau; a.alpha = p.alpha; a.eta = p.eta; a.coder = p.coder;
  }
};

// Refresh semantics in the decode direction (NEXT-4): when step j is the first row of window
// block b >= 1 (j = L_max + (b - 1) C), the surviving positions [w_b, j) (w_b = b C) of every
// chunk are re-evaluated from scratch -- one slab forward with window start w_b, no head --
// into the decode forward's KV ring, exactly the rows the compressor's refresh slab computed
// for them (per-row arithmetic is batch-invariant, D15), so decoding stays bit-identical.
struct Refill {
  Forward fw2{nullptr, nullptr};
  const uint32_t *toks = nullptr;   // token ids in chunk-major layout (tok_off), x_p = toks[p - 1]
  const int64_t *tok_off = nullptr;
  const uint32_t *ntok = nullptr;
  uint32_t *xs = nullptr;
  int32_t *rc = nullptr, *rp = nullptr;
  AttnTile *tiles_d = nullptr;
  int n_chunks = 0, len = 0;
  uint32_t bos = 0;
  std::vector<uint32_t> ntok_h;
  cudaStream_t s = nullptr;
  void init(nc_model *m, Bag &bag, Forward &fw, int n_ch, const Params &p, const uint32_t *toks_d,
            const int64_t *tok_off_d, const uint32_t *ntok_d, cudaStream_t st, const uint32_t *ntok_host = nullptr) {
    s = st;
    n_chunks = n_ch;
    len = (int)p.lmax - (int)p.slide;
    toks = toks_d; tok_off = tok_off_d; ntok = ntok_d;
    bos = m->s.bos;
    fw2 = Forward{m, st};
    const int Mr = n_chunks * ((len + 127) / 128 * 128);
    fw2.alloc(bag, Mr, n_chunks, fw.ring.ring, false, /*ring=*/&fw.ring, /*logits=*/false);
    xs = bag.get<uint32_t>(Mr);
    rc = bag.get<int32_t>(Mr);
    rp = bag.get<int32_t>(Mr);
    tiles_d = bag.get<AttnTile>((size_t)n_chunks * ((len + 127) / 128 + 8));
    if (ntok_host) ntok_h.assign(ntok_host, ntok_host + n_chunks);
  }
  // the re-prefill (if step j starts a refresh block); returns true if it ran
  bool before_step(uint32_t j, const Params &p) {
    const int L = (int)p.lmax, C = (int)p.slide;
    if ((int)j < L || ((int)j - L) % C != 0) return false;
    const int w = ((int)j - L) / C * C + C;
    std::vector<AttnTile> tiles;
    for (int c = 0; c < n_chunks; ++c) {
      const int e = ntok_h.empty() ? (int)j : std::min<int>((int)j, (int)ntok_h[c]);
      push_tiles(tiles, c, w, e, w, len, w, p);
    }
    if (tiles.empty()) return false;
    NC_CUDA(cudaMemcpyAsync(tiles_d, tiles.data(), tiles.size() * sizeof(AttnTile), cudaMemcpyHostToDevice, s));
    const int Ms = n_chunks * len;
    slab_rows_kernel<<<(Ms + 255) / 256, 256, 0, s>>>(toks, tok_off, ntok, len, w, Ms, bos, xs, rc, rp);
    NC_CUDA(cudaGetLastError());
    RowMeta rm{xs, rc, rp};
    fw2.run(Ms, 0, 0, rm, tiles_d, (int)tiles.size(), p, nullptr, /*head=*/false);
    stats().launches++;
    return true;
  }
};

// --------------------------------------------------------------- compress ---
void compress_device(nc_model *m, const uint32_t *tokens_dev, const std::vector<uint32_t> &ntok,
                     const Params &p, cudaStream_t s, CompressOut &out, int container_chunks) {
  const auto t_entry = std::chrono::steady_clock::now();
  Nvtx nv_all("nc.compress_device");
  NC_CUDA(cudaSetDevice(m->device));
  const Shape &S = m->s;
  const int n_chunks = (int)ntok.size();
  uint32_t max_n = 0;
  uint64_t total = 0;
  std::vector<int64_t> tok_off(n_chunks);
  for (int c = 0; c < n_chunks; ++c) {
    tok_off[c] = (int64_t)total;
    total += ntok[c];
    max_n = std::max(max_n, ntok[c]);
  }
  out.cum.assign(total, 0);
  out.freq.assign(total, 0);
  out.err.assign(n_chunks, 0);
  if (p.debug_dump) out.p_true.assign(total, 0.f);
  Stats &st = stats();
  if (n_chunks == 0 || max_n == 0) return;
  if (S.V >= (1u << p.cdf_bits)) fail(NC_ERR_INVALID, "T = 2^cdf_bits must exceed V");

  // Slab plan (slab_plan above).  The walk of slab s overlaps the forward of slab s+1 (own
  // stream, logits double-buffered); only the last slab's walk runs after the forward.
  // Bigger slabs run the GEMMs more efficiently (fewer tile waves), a smaller last slab
  // shortens that final walk.  Measured on config2 (3885 positions): 4 x 1024 -> 109 ms,
  // 2 x ~1940 -> 101.5 ms, 2944 + 941 (frac 0.75) -> 96.8 ms (early kernels); with the faster
  // walk of r01f, frac 0.70 / 0.75 / 0.80 / 0.85 -> 75.0 / 74.2 / 73.1 / 73.6 ms.  Slabs are
  // 128-aligned so no 128-row attention tile crosses a retained-window step (C | 128 k).
  // NC_SLAB_PLAN="a,b,..." (diagnostics) gives explicit lengths.
  const int per_chunk = std::max(128, (int)(p.max_slab_rows / n_chunks) / 128 * 128);
  const std::vector<Slab> slabs = slab_plan(p, (int)max_n, n_chunks, per_chunk);
  int R = 128;
  for (const Slab &sb : slabs) R = std::max(R, ((sb.len + 127) / 128) * 128);
  const int n_slabs = (int)slabs.size();
  const int ring_len = (int)p.window + R;
  const int M = n_chunks * R;   // buffer rows (the largest slab)
  ensure_rope(m, (int64_t)max_n + 1);

  Bag bag(s);
  bag.also(m->walk_stream);
  bag.also(m->ng_stream);
  Forward fw{m, s};
  fw.alloc(bag, M, n_chunks, ring_len, n_slabs > 1);
  std::vector<uint32_t> ntok_v(ntok);
  uint32_t *ntok_d = bag.upload(ntok_v);
  int64_t *tok_off_d = bag.upload(tok_off);
  uint32_t *xs = bag.get<uint32_t>(M);
  int32_t *rchunk = bag.get<int32_t>(M), *rpos = bag.get<int32_t>(M);
  // attention tiles and walk entries for every slab
  std::vector<AttnTile> tiles;
  std::vector<int> tile_off(n_slabs + 1, 0);
  std::vector<int32_t> w_chunk, w_row0, w_count;
  std::vector<int> w_off(n_slabs + 1, 0);
  for (int sl = 0; sl < n_slabs; ++sl) {
    tile_off[sl] = (int)tiles.size();
    w_off[sl] = (int)w_chunk.size();
    const Slab &sb = slabs[sl];
    for (int c = 0; c < n_chunks; ++c) {
      push_tiles(tiles, c, sb.pos0, std::min(sb.pos0 + sb.len, (int)ntok[c]), sb.pos0, sb.len, sb.w0, p);
      const int o1 = std::min(sb.out1, (int)ntok[c]);
      if (o1 > sb.out0) { w_chunk.push_back(c); w_row0.push_back(c * sb.len + (sb.out0 - sb.pos0)); w_count.push_back(o1 - sb.out0); }
    }
    // the persistent attention kernel claims tiles in list order: heaviest (latest positions,
    // most keys) first so the last claims are short
    std::stable_sort(tiles.begin() + tile_off[sl], tiles.end(),
                     [](const AttnTile &x, const AttnTile &y) { return x.p0 > y.p0; });
  }
  tile_off[n_slabs] = (int)tiles.size();
  w_off[n_slabs] = (int)w_chunk.size();
  AttnTile *tiles_d = bag.upload(tiles);
  int32_t *wc_d = bag.upload(w_chunk), *wr_d = bag.upload(w_row0), *wn_d = bag.upload(w_count);
  WalkBufs wb;
  const bool use_ng = p.flags & 1u;
  wb.alloc(bag, n_chunks, S.V, max_n, p, s, use_ng ? (uint32_t)(2 * R) : 0u);
  uint32_t *cum_d = bag.get<uint32_t>(total), *freq_d = bag.get<uint32_t>(total);
  float *p_d = p.debug_dump ? bag.get<float>(total) : nullptr;

  // streams: forward (s), N-gram precompute (ns, runs ahead; ring of 2 slabs), walk (ws)
  // events: per slab forward start/end, walk start/end, N-gram done
  cudaStream_t ws = m->walk_stream, ns = m->ng_stream;
  Events ev(5 * n_slabs + 1);
  cudaEvent_t ev_init = ev[5 * n_slabs];
  NC_CUDA(cudaEventRecord(ev_init, s));
  const auto t_setup = std::chrono::steady_clock::now();
  NC_CUDA(cudaStreamWaitEvent(ns, ev_init, 0));
  NC_CUDA(cudaStreamWaitEvent(ws, ev_init, 0));
  // the walk keeps one SM per chunk busy for a whole slab: leave those SMs out of
  // the persistent GEMM grids so every GEMM CTA is resident at once
  // GEMM tiles are claimed dynamically, so the persistent grids need no SM reservation
  set_reserved_sms(0);
  WalkArgs wbase{};
  wbase.logits = nullptr; wbase.ldl = S.V;
  wbase.tokens = tokens_dev; wbase.tok_off = tok_off_d;
  wbase.out_cum = cum_d; wbase.out_freq = freq_d; wbase.out_p = p_d;
  wbase.mode = 0;
  wbase.n_chunks_total = container_chunks >= 0 ? container_chunks : n_chunks;
  wb.fill(wbase, p, S.V);
  for (int sl = 0; sl < n_slabs; ++sl) {
    if (use_ng) {
      // ring slot i % ng_ring of this slab's walked tokens last held token i - ng_ring: wait
      // for the walk of the last slab holding such a token (none while within the ring)
      const int64_t need = (int64_t)slabs[sl].out1 - (int64_t)wb.ng_ring;
      int q = -1;
      for (int k2 = 0; k2 < sl; ++k2)
        if (slabs[k2].out0 < need && slabs[k2].out1 > slabs[k2].out0) q = k2;
      if (q >= 0) NC_CUDA(cudaStreamWaitEvent(ns, ev[4 * q + 3], 0));
      WalkArgs na = wbase;
      na.chunk_of = wc_d + w_off[sl]; na.row0 = wr_d + w_off[sl]; na.count = wn_d + w_off[sl];
      na.n_entries = w_off[sl + 1] - w_off[sl];
      launch_ngram_precompute(na, ns);
      NC_CUDA(cudaEventRecord(ev[4 * n_slabs + sl], ns));
      st.launches++;
    }
    Nvtx nv_slab("nc.slab (forward + walk launches)");
    if (sl >= 2) NC_CUDA(cudaStreamWaitEvent(s, ev[4 * (sl - 2) + 3], 0));   // logits buffer free again
    fw.logits = fw.lbuf[sl & 1];
    NC_CUDA(cudaEventRecord(ev[4 * sl], s));
    const int len = slabs[sl].len, q0 = slabs[sl].pos0, Ms = n_chunks * len;
    PROF(K_MISC, 0, (slab_rows_kernel<<<(Ms + 255) / 256, 256, 0, s>>>(tokens_dev, tok_off_d, ntok_d, len, q0, Ms,
                                                                       S.bos, xs, rchunk, rpos)));
    st.launches++;
    RowMeta rows{xs, rchunk, rpos};
    double valid = 0, ctx = 0;
    for (int c = 0; c < n_chunks; ++c) {
      int64_t a0 = q0, a1 = std::min<int64_t>((int64_t)q0 + len, ntok[c]);
      if (a1 > a0) { valid += (double)(a1 - a0); ctx += ctx_sum_slab(a0, a1, slabs[sl].w0, p); }
    }
    fw.run(Ms, valid, 4.0 * S.H * S.dh * ctx, rows, tiles_d + tile_off[sl], tile_off[sl + 1] - tile_off[sl], p,
           nullptr);
    NC_CUDA(cudaEventRecord(ev[4 * sl + 1], s));
    NC_CUDA(cudaStreamWaitEvent(ws, ev[4 * sl + 1], 0));
    if (use_ng) NC_CUDA(cudaStreamWaitEvent(ws, ev[4 * n_slabs + sl], 0));
    NC_CUDA(cudaEventRecord(ev[4 * sl + 2], ws));
    WalkArgs wa = wbase;
    wa.chunk_of = wc_d + w_off[sl]; wa.row0 = wr_d + w_off[sl]; wa.count = wn_d + w_off[sl];
    wa.n_entries = w_off[sl + 1] - w_off[sl];
    wa.logits = fw.logits;
    prof().begin(K_WALK, 4.0 * S.V * valid, ws);
    static const bool no_walk = std::getenv("NC_DIAG_NO_WALK") != nullptr;   // diagnostics only (output wrong)
    if (!no_walk) launch_walk(wa, ws);
    prof().end(ws);
    NC_CUDA(cudaEventRecord(ev[4 * sl + 3], ws));
    st.launches++;
    NC_CUDA(cudaGetLastError());
  }
  Nvtx nv_sync("nc.compress sync + D2H");
  NC_CUDA(cudaStreamWaitEvent(s, ev[4 * (n_slabs - 1) + 3], 0));
  set_reserved_sms(0);
  NC_CUDA(cudaMemcpyAsync(out.cum.data(), cum_d, total * 4, cudaMemcpyDeviceToHost, s));
  NC_CUDA(cudaMemcpyAsync(out.freq.data(), freq_d, total * 4, cudaMemcpyDeviceToHost, s));
  if (p_d) NC_CUDA(cudaMemcpyAsync(out.p_true.data(), p_d, total * 4, cudaMemcpyDeviceToHost, s));
  std::vector<WalkState> hs(n_chunks);
  NC_CUDA(cudaMemcpyAsync(hs.data(), wb.st, n_chunks * sizeof(WalkState), cudaMemcpyDeviceToHost, s));
  NC_CUDA(cudaStreamSynchronize(s));
  if (prof().on) prof().collect();
  if (std::getenv("NC_WALK_REPORT")) walk_timing_report();
  if (std::getenv("NC_GEMM_REPORT")) gemm_timing_report();
  if (std::getenv("NC_ATT_REPORT")) attn_timing_report();
  for (int c = 0; c < n_chunks; ++c) out.err[c] = hs[c].err;
  for (int sl = 0; sl < n_slabs; ++sl) {
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, ev[4 * sl], ev[4 * sl + 1]);
    cudaEventElapsedTime(&b, ev[4 * sl + 2], ev[4 * sl + 3]);
    st.forward_ms += a;
    st.walk_ms += b;
  }
  if (std::getenv("NC_TIMELINE")) {   // diagnostics: stream timeline of this compression (ms from the start)
    fprintf(stderr, "host: setup before the first launch %.2f ms, launch..sync %.2f ms\n",
            std::chrono::duration<double, std::milli>(t_setup - t_entry).count(),
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_setup).count());
    auto at = [&](cudaEvent_t e) {
      float t = 0;
      cudaEventElapsedTime(&t, ev_init, e);
      return t;
    };
    for (int sl = 0; sl < n_slabs; ++sl)
      fprintf(stderr, "slab %d (%d positions): forward %.2f-%.2f  ngram done %.2f  walk %.2f-%.2f\n", sl,
              slabs[sl].len, at(ev[4 * sl]), at(ev[4 * sl + 1]), use_ng ? at(ev[4 * n_slabs + sl]) : 0.f,
              at(ev[4 * sl + 2]), at(ev[4 * sl + 3]));
  }
}

// --------------------------------------------------------------- container ---
void encode_container(const Params &p, const std::vector<uint32_t> &ntok, const CompressOut &co,
                      std::vector<uint8_t> &out) {
  Nvtx nv("nc.range coder + NC05");
  const size_t n = ntok.size();
  std::vector<Nc05Chunk> chunks(n);
  std::vector<size_t> off(n + 1, 0);
  for (size_t c = 0; c < n; ++c) off[c + 1] = off[c] + ntok[c];
  for (size_t c = 0; c < n; ++c)
    if (co.err[c]) fail(NC_ERR_INTEGRITY, "quantizer residual would drop a count below 1 (D6)");
  auto work = [&](size_t c) {
    uint64_t bits;
    if (p.coder == NC_CODER_ANS) {
      ans_encode(co.cum.data() + off[c], co.freq.data() + off[c], off[c + 1] - off[c], p.cdf_bits,
                 chunks[c].stream, bits);
    } else {
      WncEncoder enc;
      for (size_t i = off[c]; i < off[c + 1]; ++i) enc.encode(co.cum[i], co.freq[i], p.cdf_bits);
      enc.finish(chunks[c].stream, bits);
    }
    if (bits > 0xFFFFFFFFull) fail(NC_ERR_INVALID, "chunk bitstream exceeds the u32 bit_count field");
    chunks[c].bits = (uint32_t)bits;
    chunks[c].tokens = ntok[c];
  };
  unsigned nt = std::max(1u, std::min<unsigned>((unsigned)n, std::thread::hardware_concurrency()));
  if (nt <= 1 || n <= 1) {
    for (size_t c = 0; c < n; ++c) work(c);
  } else {
    std::vector<std::thread> th;
    std::vector<std::string> errs(nt);
    for (unsigned t = 0; t < nt; ++t)
      th.emplace_back([&, t] {
        try {
          for (size_t c = t; c < n; c += nt) work(c);
        } catch (std::exception &e) { errs[t] = e.what(); }
      });
    for (auto &x : th) x.join();
    for (auto &e : errs)
      if (!e.empty()) fail(NC_ERR_INTEGRITY, e);
  }
  write_nc05((uint8_t)p.flags, (uint16_t)p.tau_milli, chunks, out);
}

// ------------------------------------------------------------- decompress ---
// A non-blocking stream owned by one decompression (a CUDA graph cannot be captured
// on the legacy default stream the caller may pass); ordered after the caller's work.
struct OwnStream {
  cudaStream_t s = nullptr;
  explicit OwnStream(cudaStream_t after) {
    NC_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t e;
    NC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    NC_CUDA(cudaEventRecord(e, after));
    NC_CUDA(cudaStreamWaitEvent(s, e, 0));
    cudaEventDestroy(e);
  }
  ~OwnStream() {
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  }
};

void decompress_device(nc_model *m, const uint8_t *blob, const Nc05View &view, const Params &p,
                       cudaStream_t s_caller, std::vector<std::vector<uint32_t>> &toks, int container_chunks) {
  NC_CUDA(cudaSetDevice(m->device));
  Nvtx nv_all("nc.decompress_device");
  OwnStream own(s_caller);
  cudaStream_t s = own.s;
  const Shape &S = m->s;
  const int n_chunks = (int)view.ents.size();
  toks.assign(n_chunks, {});
  uint32_t max_n = 0;
  uint64_t total = 0;
  std::vector<int64_t> tok_off(n_chunks), s_off(n_chunks);
  std::vector<uint64_t> s_bits(n_chunks);
  std::vector<uint32_t> ntok(n_chunks);
  uint64_t blob_len = 0;
  for (int c = 0; c < n_chunks; ++c) {
    ntok[c] = view.ents[c].tokens;
    tok_off[c] = (int64_t)total;
    total += ntok[c];
    max_n = std::max(max_n, ntok[c]);
    s_off[c] = (int64_t)view.ents[c].off;
    s_bits[c] = view.ents[c].bits;
    blob_len = std::max<uint64_t>(blob_len, view.ents[c].off + view.ents[c].len);
  }
  if (n_chunks == 0 || max_n == 0) return;
  if (S.V >= (1u << p.cdf_bits)) fail(NC_ERR_INVALID, "T = 2^cdf_bits must exceed V");
  // a token costs at least -log2(1 - (V - 1)/T) bits (the largest count is T - (V - 1)), and
  // the coder adds at most ~2 bits: reject token counts the stream cannot hold BEFORE
  // sizing any buffer from them (a crafted header could ask for 2^32 tokens in 0 bits)
  {
    const double min_bits = -std::log2(1.0 - (double)(S.V - 1) / (double)(1ull << p.cdf_bits));
    for (int c = 0; c < n_chunks; ++c)
      if ((double)ntok[c] * min_bits > (double)s_bits[c] + 64.0)
        fail(NC_ERR_INTEGRITY, "chunk " + std::to_string(c) + " claims more tokens than its bit_count can code");
  }
  Stats &st = stats();
  ensure_rope(m, (int64_t)max_n + 1);
  Bag bag(s);
  Forward fw{m, s};
  const int ring_len = (int)p.window + 128;   // 128-key attention blocks never wrap
  fw.alloc(bag, n_chunks, n_chunks, ring_len);
  std::vector<uint8_t> bl(blob, blob + blob_len);
  uint8_t *blob_d = bag.upload(bl);
  int64_t *s_off_d = bag.upload(s_off), *tok_off_d = bag.upload(tok_off);
  uint64_t *s_bits_d = bag.upload(s_bits);
  uint32_t *ntok_d = bag.upload(ntok);
  std::vector<uint32_t> bos(n_chunks, S.bos);
  uint32_t *x_cur = bag.upload(bos);
  int32_t *rchunk = bag.get<int32_t>(n_chunks), *rpos = bag.get<int32_t>(n_chunks);
  AttnTile *tiles = bag.get<AttnTile>(n_chunks);
  int32_t *wc = bag.get<int32_t>(n_chunks), *wr = bag.get<int32_t>(n_chunks), *wn = bag.get<int32_t>(n_chunks);
  WalkBufs wb;
  wb.alloc(bag, n_chunks, S.V, max_n, p, s);
  uint32_t *out_tok = bag.get<uint32_t>(total);
  WalkArgs wa{};
  wa.chunk_of = wc; wa.row0 = wr; wa.count = wn; wa.n_entries = n_chunks;
  wa.logits = fw.logits; wa.ldl = S.V;
  wa.tok_off = tok_off_d; wa.streams = blob_d; wa.stream_off = s_off_d; wa.stream_bits = s_bits_d;
  wa.out_tok = out_tok; wa.next_x = x_cur; wa.mode = 1;
  wa.n_chunks_total = container_chunks >= 0 ? container_chunks : n_chunks;
  wb.fill(wa, p, S.V);
  int *jctr = bag.get<int>(1);
  NC_CUDA(cudaMemsetAsync(jctr, 0, sizeof(int), s));
  cudaEvent_t e0, e1;
  NC_CUDA(cudaEventCreate(&e0));
  NC_CUDA(cudaEventCreate(&e1));
  NC_CUDA(cudaEventRecord(e0, s));
  // one decode step: rows of step j (j on the device), forward of one row per chunk, walk
  auto step = [&](uint32_t j) {
    double valid = 0;
    for (int c = 0; c < n_chunks; ++c) valid += j < ntok[c] ? 1 : 0;
    const double ctx = (double)j - window_start_h(j, p.lmax, p.slide) + 1;
    PROF(K_MISC, 0, (step_rows_dev_kernel<<<1, 256, 0, s>>>(ntok_d, n_chunks, jctr, rchunk, rpos, tiles, wc, wr, wn)));
    RowMeta rows{x_cur, rchunk, rpos};
    fw.run(n_chunks, valid, 4.0 * S.H * S.dh * ctx * valid, rows, tiles, n_chunks, p, nullptr, true, true);
    PROF(K_WALK, 4.0 * S.V * valid, launch_walk(wa, s));
    st.launches += 2;
  };
  // Every step launches the same kernels with the same arguments (the step index lives
  // on the device), so after one eager step (which also sizes every lazily allocated
  // launcher buffer) the step is captured once as a CUDA graph and replayed.  Per-launch
  // profiling (CUDA events around every kernel) runs eagerly instead.
  const bool graph = !prof().on && !std::getenv("NC_DECODE_NO_GRAPH");
  Refill rf;   // refresh semantics: re-evaluate the surviving window at every block start
  if (p.refresh) rf.init(m, bag, fw, n_chunks, p, out_tok, tok_off_d, ntok_d, s, ntok.data());
  step(0);
  if (graph && max_n > 1) {
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    const uint64_t l0 = st.launches;
    NC_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    step(1);
    NC_CUDA(cudaStreamEndCapture(s, &g));
    const uint64_t per_step = st.launches - l0;
    st.launches = l0;
    NC_CUDA(cudaGraphInstantiate(&ge, g, 0));
    for (uint32_t j = 1; j < max_n; ++j) {
      if (p.refresh) rf.before_step(j, p);
      NC_CUDA(cudaGraphLaunch(ge, s));
      st.launches += per_step;
      if ((j & 255) == 255) NC_CUDA(cudaGetLastError());
    }
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
  } else {
    for (uint32_t j = 1; j < max_n; ++j) {
      if (p.refresh) rf.before_step(j, p);
      step(j);
      if ((j & 255) == 255) {
        NC_CUDA(cudaGetLastError());
        if (prof().on) { NC_CUDA(cudaStreamSynchronize(s)); prof().collect(); }
      }
    }
  }
  NC_CUDA(cudaEventRecord(e1, s));
  if (std::getenv("NC_ATT_REPORT")) attn_timing_report();   // diagnostics builds (-DNC_ATT_TIMING)
  std::vector<uint32_t> all(total);
  NC_CUDA(cudaMemcpyAsync(all.data(), out_tok, total * 4, cudaMemcpyDeviceToHost, s));
  std::vector<WalkState> hs(n_chunks);
  NC_CUDA(cudaMemcpyAsync(hs.data(), wb.st, n_chunks * sizeof(WalkState), cudaMemcpyDeviceToHost, s));
  NC_CUDA(cudaStreamSynchronize(s));
  if (prof().on) prof().collect();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  st.forward_ms += ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  for (int c = 0; c < n_chunks; ++c) {
    if (hs[c].err) fail(NC_ERR_INTEGRITY, "decoder integrity failure in chunk " + std::to_string(c));
    if (p.coder == NC_CODER_ANS) {
      // rANS (D39): the decoder ends in the encoder's start state L = 2^31 having read every
      // word, and the stream is whole words with nothing after them
      if (ntok[c] && (hs[c].value != (1ull << 31) || hs[c].bitpos != s_bits[c] ||
                      (uint64_t)view.ents[c].len * 8 != s_bits[c]))
        fail(NC_ERR_INTEGRITY, "rANS end state of chunk " + std::to_string(c) + " is not the encoder's start state (wrong params or corrupt stream)");
      toks[c].assign(all.begin() + tok_off[c], all.begin() + tok_off[c] + ntok[c]);
      continue;
    }
    // every renormalisation shift of the decoder matches one encoder step;
    // bit_count = steps + 2 (finish emits 1 + (pending+1) bits)  (D8)
    if (ntok[c] && hs[c].bitpos - 32 + 2 != s_bits[c])
      fail(NC_ERR_INTEGRITY, "bit_count mismatch in chunk " + std::to_string(c) + " (wrong params or corrupt stream)");
    // and the stream must END exactly as the encoder's finish() leaves it from the decoder's
    // final state: bit b = [low >= QUARTER], then (pending + 1) copies of !b, then zero padding
    // (D8; "tampering ... never silent partial corruption past the integrity checks")
    if (ntok[c]) {
      const uint8_t *sp = blob + s_off[c];
      const uint64_t steps = hs[c].bitpos - 32, pend = hs[c].pend;
      auto bit_at = [&](uint64_t k) { return (uint32_t)(sp[k >> 3] >> (7 - (k & 7))) & 1u; };
      const uint32_t b = hs[c].low < (1ull << 30) ? 0u : 1u;
      bool ok = pend <= steps;
      for (uint64_t k = steps - std::min<uint64_t>(pend, steps); ok && k < steps + 2; ++k)
        ok = bit_at(k) == (k == steps - pend ? b : (b ^ 1u));
      for (uint64_t k = steps + 2; ok && k < (uint64_t)view.ents[c].len * 8; ++k) ok = bit_at(k) == 0u;
      if (!ok) fail(NC_ERR_INTEGRITY, "stream tail of chunk " + std::to_string(c) + " is not the coder's finish (corrupt stream)");
    }
    toks[c].assign(all.begin() + tok_off[c], all.begin() + tok_off[c] + ntok[c]);
  }
}

// ------------------------------------------------------------------ debug ---
void debug_forward(nc_model *m, const uint32_t *x, uint32_t rows, const Params &p, int mode, float *out) {
  NC_CUDA(cudaSetDevice(m->device));
  const Shape &S = m->s;
  cudaStream_t s = nullptr;
  if (rows == 0) return;
  ensure_rope(m, (int64_t)rows + 1);
  Bag bag(s);
  std::vector<uint32_t> xv(x, x + rows);
  uint32_t *x_d = bag.upload(xv);
  Forward fw{m, s};
  // the slab kernel maps x through "tokens[p-1]"; feed x shifted so that x_j = x[j]
  std::vector<uint32_t> shifted(rows);
  for (uint32_t j = 0; j + 1 < rows; ++j) shifted[j] = x[j + 1];
  uint32_t *t_d = bag.upload(shifted);
  std::vector<int64_t> off{0};
  int64_t *off_d = bag.upload(off);
  std::vector<uint32_t> nt{rows};
  uint32_t *nt_d = bag.upload(nt);
  if (mode == 0) {
    const int per = std::max(128, (int)p.max_slab_rows / 128 * 128);
    const std::vector<Slab> slabs = slab_plan(p, (int)rows, 1, per);
    int Rr = 128;
    for (const Slab &sb : slabs) Rr = std::max(Rr, (sb.len + 127) / 128 * 128);
    fw.alloc(bag, Rr, 1, (int)p.window + Rr);
    uint32_t *xs = bag.get<uint32_t>(Rr);
    int32_t *rc = bag.get<int32_t>(Rr), *rp = bag.get<int32_t>(Rr);
    for (const Slab &sb : slabs) {
      std::vector<AttnTile> tiles;
      push_tiles(tiles, 0, sb.pos0, sb.pos0 + sb.len, sb.pos0, sb.len, sb.w0, p);
      AttnTile *td = bag.upload(tiles);
      slab_rows_kernel<<<(sb.len + 255) / 256, 256, 0, s>>>(t_d, off_d, nt_d, sb.len, sb.pos0, sb.len, x[0], xs, rc, rp);
      RowMeta rm{xs, rc, rp};
      fw.run(sb.len, 0, 0, rm, td, (int)tiles.size(), p, nullptr);
      if (sb.out1 > sb.out0)
        NC_CUDA(cudaMemcpyAsync(out + (size_t)sb.out0 * S.V, fw.logits + (size_t)(sb.out0 - sb.pos0) * S.V,
                                (size_t)(sb.out1 - sb.out0) * S.V * 4, cudaMemcpyDeviceToHost, s));
    }
  } else {
    fw.alloc(bag, 1, 1, (int)p.window + 128);
    Refill rf;
    if (p.refresh) rf.init(m, bag, fw, 1, p, t_d, off_d, nt_d, s);
    int32_t *rc = bag.get<int32_t>(1), *rp = bag.get<int32_t>(1);
    AttnTile *tiles = bag.get<AttnTile>(1);
    int32_t *wc = bag.get<int32_t>(1), *wr = bag.get<int32_t>(1), *wn = bag.get<int32_t>(1);
    for (uint32_t j = 0; j < rows; ++j) {
      if (p.refresh) rf.before_step(j, p);
      step_rows_kernel<<<1, 32, 0, s>>>(nt_d, 1, (int)j, rc, rp, tiles, wc, wr, wn);
      RowMeta rm{x_d + j, rc, rp};
      fw.run(1, 0, 0, rm, tiles, 1, p, nullptr, true, true);
      NC_CUDA(cudaMemcpyAsync(out + (size_t)j * S.V, fw.logits, (size_t)S.V * 4, cudaMemcpyDeviceToHost, s));
    }
  }
  NC_CUDA(cudaStreamSynchronize(s));
}

void debug_gemm(int device, const float *A, const float *B, uint32_t M, uint32_t N, uint32_t K, int mode,
                float *out) {
  NC_CUDA(cudaSetDevice(device));
  if (K % 32 || N % 64) fail(NC_ERR_INVALID, "debug_gemm needs K % 32 == 0 and N % 64 == 0");
  if (mode != 0) fail(NC_ERR_INVALID, "debug_gemm: mode 0 (tcgen05 3xTF32) is the only GEMM");
  cudaStream_t s = nullptr;
  Bag bag(s);
  std::vector<float> a(A, A + (size_t)M * K), b(B, B + (size_t)N * K), ones(M, 1.f);
  float *a_d = bag.upload(a), *b_d = bag.upload(b), *r_d = bag.upload(ones);
  float *c_d = bag.get<float>((size_t)M * N);
  if (mode == 0) {
    float *ah = bag.get<float>((size_t)M * K), *al = bag.get<float>((size_t)M * K);
    float *bh = bag.get<float>((size_t)N * K), *bl = bag.get<float>((size_t)N * K);
    launch_split_planes(a_d, ah, al, (size_t)M * K, s);
    launch_split_planes(b_d, bh, bl, (size_t)N * K, s);
    TcGemmArgs g{};
    g.M = (int)M; g.N = (int)N; g.K = (int)K; g.rinv = r_d; g.C = c_d; g.ldc = (int)N;
    TcOperands op{ah, al, (uint64_t)M, bh, bl};
    launch_gemm_tc(EPI_HEAD, g, op, s);
    // diagnostics: NC_GEMM_REPS=n times n launches (NC_GEMM_EPI=resid: the residual
    // epilogue on a scratch h; NC_GEMM_NOSTORE=1: no epilogue writes) -> stderr
    if (const char *reps_s = getenv("NC_GEMM_REPS")) {
      const int reps = std::max(1, atoi(reps_s));
      if (const char *sp = getenv("NC_GEMM_SPLIT")) set_splitk_mode(atoi(sp));
      const char *epi_s = getenv("NC_GEMM_EPI");
      const bool resid = epi_s && std::string(epi_s) == "resid";
      TcGemmArgs t = g;
      t.no_store = getenv("NC_GEMM_NOSTORE") ? 1 : 0;
      float *h = nullptr;
      if (resid) {
        h = bag.get<float>((size_t)M * N * 3);
        NC_CUDA(cudaMemsetAsync(h, 0, (size_t)M * N * 12, s));
        t.C = h; t.C_hi = h + (size_t)M * N; t.C_lo = h + 2 * (size_t)M * N;
      }
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      for (int w = 0; w < 3; ++w) launch_gemm_tc(resid ? EPI_RESID : EPI_HEAD, t, op, s);
      cudaEventRecord(e0, s);
      for (int r = 0; r < reps; ++r) launch_gemm_tc(resid ? EPI_RESID : EPI_HEAD, t, op, s);
      cudaEventRecord(e1, s);
      NC_CUDA(cudaEventSynchronize(e1));
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      cudaEventDestroy(e0); cudaEventDestroy(e1);
      const double us = 1e3 * ms / reps;
      set_splitk_mode(1);
      fprintf(stderr, "gemm_tc M=%u N=%u K=%u epi=%s nostore=%d: %.1f us/launch, %.1f TFLOP/s (algorithmic)\n", M, N,
              K, resid ? "resid" : "head", t.no_store, us, 2.0 * M * N * K / (us * 1e-6) / 1e12);
      gemm_timing_report();
    }
  }
  NC_CUDA(cudaGetLastError());
  NC_CUDA(cudaMemcpyAsync(out, c_d, (size_t)M * N * 4, cudaMemcpyDeviceToHost, s));
  NC_CUDA(cudaStreamSynchronize(s));
}

void debug_attention(int device, const float *q, const float *k, const float *v, uint32_t n, uint32_t H, uint32_t KV,
                     uint32_t window, uint32_t slide, int mode, float *o) {
  NC_CUDA(cudaSetDevice(device));
  if (mode != 0) fail(NC_ERR_INVALID, "debug_attention: mode 0 (tcgen05 3xTF32) is the only attention");
  if (!n) return;
  cudaStream_t s = nullptr;
  Bag bag(s);
  const int ring = (int)(((n + 127) / 128) * 128);   // every position in its own slot
  const size_t qd = (size_t)H * 64, kvd = (size_t)KV * 64;
  std::vector<float> qv(q, q + n * qd), kv(k, k + n * kvd), vv(v, v + n * kvd);
  const int rows = ring;
  std::vector<float> qpad(rows * qd, 0.f), kpad((size_t)ring * kvd, 0.f), vpad((size_t)ring * kvd, 0.f);
  std::copy(qv.begin(), qv.end(), qpad.begin());
  std::copy(kv.begin(), kv.end(), kpad.begin());
  std::copy(vv.begin(), vv.end(), vpad.begin());
  float *q_d = bag.upload(qpad), *k_d = bag.upload(kpad), *v_d = bag.upload(vpad);
  float *oh = bag.get<float>((size_t)rows * qd), *ol = bag.get<float>((size_t)rows * qd);
  const int TR = 128;
  std::vector<AttnTile> tiles;
  for (uint32_t p0 = 0; p0 < n; p0 += TR) tiles.push_back(AttnTile{0, (int)p0, (int)std::min<uint32_t>(TR, n - p0), (int)p0, -1});
  AttnTile *t_d = bag.upload(tiles);
  if (mode == 0) {
    float *qh = bag.get<float>(rows * qd), *ql = bag.get<float>(rows * qd);
    float *kh = bag.get<float>(ring * kvd), *kl = bag.get<float>(ring * kvd);
    float *vh = bag.get<float>(ring * kvd), *vl = bag.get<float>(ring * kvd);
    launch_split_planes(q_d, qh, ql, rows * qd, s);
    launch_split_planes(k_d, kh, kl, ring * kvd, s);
    launch_split_planes(v_d, vh, vl, ring * kvd, s);
    AttnTcArgs at{};
    at.tiles = t_d; at.n_tiles = (int)tiles.size(); at.q_hi = qh; at.q_lo = ql; at.ldq = (int)qd; at.q_rows = rows;
    at.k_hi = kh; at.k_lo = kl; at.v_hi = vh; at.v_lo = vl; at.ring = ring; at.n_chunks = 1; at.n_layers = 1;
    at.layer = 0; at.o_hi = oh; at.o_lo = ol; at.ldo = (int)qd; at.H = (int)H; at.KV = (int)KV;
    at.window = (int)window; at.slide = (int)slide;
    const char *dbg = std::getenv("NC_ATTN_DEBUG");
    at.debug = dbg ? std::atoi(dbg) : 0;
    if (at.debug) {
      NC_CUDA(cudaMemsetAsync(oh, 0, rows * qd * 4, s));
      NC_CUDA(cudaMemsetAsync(ol, 0, rows * qd * 4, s));
    }
    const int reps = std::getenv("NC_ATTN_REPS") ? std::atoi(std::getenv("NC_ATTN_REPS")) : 1;
    for (int rep = 0; rep < reps; ++rep) {
      double fl = 0;
      for (uint32_t j = 0; j < n; ++j) fl += 4.0 * H * 64 * ((double)j - window_start_h(j, window, slide) + 1);
      PROF(K_ATTN, fl, launch_attention_tc(at, s));
    }
    if (prof().on) { NC_CUDA(cudaStreamSynchronize(s)); prof().collect(); }
    if (std::getenv("NC_ATTN_REPS")) attn_timing_report();
    std::vector<float> a(rows * qd), b(rows * qd);
    NC_CUDA(cudaMemcpyAsync(a.data(), oh, a.size() * 4, cudaMemcpyDeviceToHost, s));
    NC_CUDA(cudaMemcpyAsync(b.data(), ol, b.size() * 4, cudaMemcpyDeviceToHost, s));
    NC_CUDA(cudaStreamSynchronize(s));
    for (size_t i = 0; i < n * qd; ++i) o[i] = a[i] + b[i];
  }
  NC_CUDA(cudaGetLastError());
}

void debug_walk(int device, const float *logits, uint32_t n_lrows, const uint32_t *tok, uint32_t n, uint32_t V,
                const Params &p, uint32_t *cum, uint32_t *freq, float *p_true, float *pt_true, const uint32_t *rows,
                uint32_t n_rows, float *pt_rows, float *p_rows, uint32_t *c_rows) {
  NC_CUDA(cudaSetDevice(device));
  if (n == 0) return;
  if (V >= (1u << p.cdf_bits)) fail(NC_ERR_INVALID, "T = 2^cdf_bits must exceed V");
  for (uint32_t k = 0; k < n_rows; ++k)
    if (rows[k] >= n || (k && rows[k] <= rows[k - 1])) fail(NC_ERR_INVALID, "dump rows must be ascending and < n_tok");
  const uint32_t R = (n_lrows == 0 || n_lrows > n) ? n : n_lrows;   // token j uses logits row j % R
  cudaStream_t s = nullptr;
  Bag bag(s);
  std::vector<float> lg(logits, logits + (size_t)R * V);
  float *lg_d = bag.upload(lg);
  std::vector<uint32_t> tk(tok, tok + n);
  uint32_t *tk_d = bag.upload(tk);
  std::vector<int64_t> off{0};
  int64_t *off_d = bag.upload(off);
  std::vector<int32_t> zero{0};
  int32_t *c_d = bag.upload(zero), *r_d = bag.upload(zero);
  WalkBufs wb;
  wb.alloc(bag, 1, V, n, p, s, R);
  uint32_t *cum_d = bag.get<uint32_t>(n), *freq_d = bag.get<uint32_t>(n);
  float *p_d = bag.get<float>(n), *pt_d = bag.get<float>(n);
  WalkArgs wa{};
  wa.chunk_of = c_d; wa.row0 = r_d; wa.n_entries = 1;
  wa.logits = lg_d; wa.ldl = V; wa.tokens = tk_d; wa.tok_off = off_d;
  wa.out_cum = cum_d; wa.out_freq = freq_d; wa.out_p = p_d; wa.out_pt = pt_d; wa.mode = 0;
  wa.n_chunks_total = p.n_chunks ? (int)p.n_chunks : 1;   // the container this chunk belongs to (cluster size)
  const size_t dn = (size_t)n_rows * V;
  if (n_rows) {
    std::vector<uint32_t> rv(rows, rows + n_rows);
    wa.dump_rows = bag.upload(rv);
    wa.n_dump = n_rows;
    wa.dump_chunk = 0;
    wa.dump_pt = bag.get<float>(dn);
    wa.dump_p = bag.get<float>(dn);
    wa.dump_c = bag.get<uint32_t>(dn);
  }
  wb.fill(wa, p, V);
  // segments of R tokens over the same R logits rows (the walk state carries over, as between slabs)
  std::vector<int32_t> cnts;
  for (uint32_t j0 = 0; j0 < n; j0 += R) cnts.push_back((int32_t)std::min(R, n - j0));
  int32_t *n_d = bag.upload(cnts);
  for (size_t k = 0; k < cnts.size(); ++k) {
    wa.count = n_d + k;
    if (p.flags & 1u) launch_ngram_precompute(wa, s);
    launch_walk(wa, s);
    NC_CUDA(cudaGetLastError());
  }
  NC_CUDA(cudaMemcpyAsync(cum, cum_d, n * 4, cudaMemcpyDeviceToHost, s));
  NC_CUDA(cudaMemcpyAsync(freq, freq_d, n * 4, cudaMemcpyDeviceToHost, s));
  NC_CUDA(cudaMemcpyAsync(p_true, p_d, n * 4, cudaMemcpyDeviceToHost, s));
  if (pt_true) NC_CUDA(cudaMemcpyAsync(pt_true, pt_d, n * 4, cudaMemcpyDeviceToHost, s));
  if (n_rows) {
    if (pt_rows) NC_CUDA(cudaMemcpyAsync(pt_rows, wa.dump_pt, dn * 4, cudaMemcpyDeviceToHost, s));
    if (p_rows) NC_CUDA(cudaMemcpyAsync(p_rows, wa.dump_p, dn * 4, cudaMemcpyDeviceToHost, s));
    if (c_rows) NC_CUDA(cudaMemcpyAsync(c_rows, wa.dump_c, dn * 4, cudaMemcpyDeviceToHost, s));
  }
  WalkState hs;
  NC_CUDA(cudaMemcpyAsync(&hs, wb.st, sizeof(hs), cudaMemcpyDeviceToHost, s));
  NC_CUDA(cudaStreamSynchronize(s));
  if (hs.err) fail(NC_ERR_INTEGRITY, "walk integrity failure (D6)");
}

}  // namespace nc
