// Multi-GPU chunk sharding: one process per GPU, chunks are
// independent units, rank r owns a contiguous chunk range, and the
// only collective is one NCCL allgather of the per-chunk table (12 B/chunk).
//
// NCCL is dlopen'ed (preferring the copy torch already loaded) so libnc.so has
// no link-time NCCL dependency and never mixes two NCCL builds in a process.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <numeric>

#include "engine.hpp"
#include "walk.cuh"

struct nc_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1, device = 0;
};

namespace {

struct NcclApi {
  void *h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char *(*errStr)(ncclResult_t) = nullptr;
};

NcclApi &nccl() {
  static NcclApi api;
  if (api.h) return api;
  const char *names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char *n : names) {
    api.h = dlopen(n, RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (api.h) break;
  }
  if (!api.h)
    for (const char *n : names) {
      api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
  if (!api.h) nc::fail(NC_ERR_BACKEND, "NCCL library not found (libnccl.so.2)");
  api.getUniqueId = (decltype(api.getUniqueId))dlsym(api.h, "ncclGetUniqueId");
  api.commInitRank = (decltype(api.commInitRank))dlsym(api.h, "ncclCommInitRank");
  api.allGather = (decltype(api.allGather))dlsym(api.h, "ncclAllGather");
  api.commDestroy = (decltype(api.commDestroy))dlsym(api.h, "ncclCommDestroy");
  api.errStr = (decltype(api.errStr))dlsym(api.h, "ncclGetErrorString");
  if (!api.getUniqueId || !api.commInitRank || !api.allGather || !api.commDestroy)
    nc::fail(NC_ERR_BACKEND, "NCCL symbols missing");
  return api;
}

void nccl_check(ncclResult_t r, const char *what) {
  if (r != ncclSuccess)
    nc::fail(NC_ERR_BACKEND, std::string(what) + ": " + (nccl().errStr ? nccl().errStr(r) : "nccl error"));
}

template <class F>
nc_status guard(F &&f) {
  try {
    f();
    return NC_OK;
  } catch (nc::Error &e) {
    nc::set_last_error(e.what());
    return e.code;
  } catch (std::exception &e) {
    nc::set_last_error(e.what());
    return NC_ERR_BACKEND;
  }
}

}  // namespace

namespace nc {

// rank r owns chunks [r*k, min((r+1)*k, n)), k = ceil(n / world)
void shard_range(uint32_t n, int world, int rank, uint32_t &c0, uint32_t &c1) {
  uint32_t k = (n + world - 1) / world;
  c0 = std::min<uint32_t>(n, (uint32_t)rank * k);
  c1 = std::min<uint32_t>(n, c0 + k);
}

// Build rank r's byte range of the final NC05 container from the full chunk
// table (3 u32 per chunk: tokens, bits, stream_len) and its own streams.
void shard_part(const uint32_t *table, uint32_t n, uint8_t flags, uint16_t tau_milli, int world, int rank,
                const uint8_t *my_streams, size_t my_len, std::vector<uint8_t> &part, uint64_t &part_offset,
                uint64_t &total_n) {
  uint32_t c0, c1;
  shard_range(n, world, rank, c0, c1);
  uint64_t before = 0, mine = 0, all = 0;
  for (uint32_t c = 0; c < n; ++c) {
    if (table[3 * c + 2] != (table[3 * c + 1] + 7ull) / 8) fail(NC_ERR_INTEGRITY, "chunk table inconsistent");
    all += table[3 * c + 2];
    if (c < c0) before += table[3 * c + 2];
    else if (c < c1) mine += table[3 * c + 2];
  }
  if (mine != my_len) fail(NC_ERR_INTEGRITY, "own stream bytes do not match the gathered table");
  if (n > 0xFFFFu) fail(NC_ERR_INVALID, "too many chunks for NC05 (u16 chunk_count)");
  const uint64_t hdr = 9 + 12ull * n;
  total_n = hdr + all;
  part.clear();
  if (rank == 0) {
    std::vector<Nc05Chunk> none;
    std::vector<uint8_t> h;
    write_nc05(flags, tau_milli, none, h);
    h[7] = n & 255;
    h[8] = (n >> 8) & 255;
    for (uint32_t c = 0; c < n; ++c)
      for (int f = 0; f < 3; ++f)
        for (int by = 0; by < 4; ++by) h.push_back((table[3 * c + f] >> (8 * by)) & 255);
    part = h;
    part_offset = 0;
  } else {
    part_offset = hdr + before;
  }
  part.insert(part.end(), my_streams, my_streams + my_len);
}

}  // namespace nc

extern "C" {

nc_status nc_comm_unique_id(uint8_t id[128]) {
  if (!id) return NC_ERR_INVALID;
  return guard([&] {
    ncclUniqueId u;
    nccl_check(nccl().getUniqueId(&u), "ncclGetUniqueId");
    static_assert(sizeof(u) == 128, "ncclUniqueId size");
    std::memcpy(id, &u, 128);
  });
}

nc_status nc_comm_init(int rank, int world, const uint8_t id[128], int device, nc_comm **out) {
  if (!id || !out || world < 1 || rank < 0 || rank >= world) return NC_ERR_INVALID;
  *out = nullptr;
  return guard([&] {
    NC_CUDA(cudaSetDevice(device));
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    nc_comm *c = new nc_comm();
    c->rank = rank; c->world = world; c->device = device;
    ncclResult_t r = nccl().commInitRank(&c->comm, world, u, rank);
    if (r != ncclSuccess) { delete c; nccl_check(r, "ncclCommInitRank"); }
    *out = c;
  });
}

void nc_comm_free(nc_comm *c) {
  if (!c) return;
  if (c->comm) nccl().commDestroy(c->comm);
  delete c;
}

static void gather_u32(nc_comm *c, const std::vector<uint32_t> &mine, std::vector<uint32_t> &all, cudaStream_t s) {
  const size_t k = mine.size();
  all.assign(k * c->world, 0);
  uint32_t *d_in = static_cast<uint32_t *>(nc::dev_alloc(k * 4 + 4, s));
  uint32_t *d_out = static_cast<uint32_t *>(nc::dev_alloc(k * 4 * c->world + 4, s));
  NC_CUDA(cudaMemcpyAsync(d_in, mine.data(), k * 4, cudaMemcpyHostToDevice, s));
  nccl_check(nccl().allGather(d_in, d_out, k, ncclUint32, c->comm, s), "ncclAllGather");
  NC_CUDA(cudaMemcpyAsync(all.data(), d_out, k * 4 * c->world, cudaMemcpyDeviceToHost, s));
  NC_CUDA(cudaStreamSynchronize(s));
  nc::dev_free(d_in, s);
  nc::dev_free(d_out, s);
}

nc_status nc_compress_shard(nc_model *m, nc_comm *c, const uint8_t *in, size_t n, const nc_params *p,
                            void *cuda_stream, uint8_t **part, size_t *part_n, uint64_t *part_offset,
                            uint64_t *total_n) {
  if (!m || !c || (!in && n) || !part || !part_n || !part_offset || !total_n) return NC_ERR_INVALID;
  *part = nullptr; *part_n = 0;
  nc::stats() = nc::Stats{};
  return guard([&] {
    nc::Params q = nc::validate(p);
    cudaStream_t s = (cudaStream_t)cuda_stream;
    NC_CUDA(cudaSetDevice(m->device));
    const uint32_t want = q.n_chunks ? q.n_chunks : (uint32_t)c->world * q.chunks_per_gpu;
    if (want > 0xFFFFu) nc::fail(NC_ERR_INVALID, "too many chunks for NC05 (u16 chunk_count)");
    std::vector<uint64_t> cuts = nc::split_chunks(in, n, want);
    const uint32_t nch = (uint32_t)cuts.size() - 1;
    uint32_t c0, c1;
    nc::shard_range(nch, c->world, c->rank, c0, c1);
    std::vector<uint32_t> tokens, ntok;
    for (uint32_t k = c0; k < c1; ++k) {
      size_t before = tokens.size();
      m->encode(in + cuts[k], cuts[k + 1] - cuts[k], tokens);
      ntok.push_back((uint32_t)(tokens.size() - before));
    }
    std::vector<uint8_t> mine_blob;
    std::vector<uint32_t> mine_tab;
    std::vector<uint8_t> my_streams;
    if (c1 > c0) {
      uint32_t *tok_d = static_cast<uint32_t *>(nc::dev_alloc(tokens.size() * 4 + 4, s));
      if (!tokens.empty()) NC_CUDA(cudaMemcpyAsync(tok_d, tokens.data(), tokens.size() * 4, cudaMemcpyHostToDevice, s));
      nc::CompressOut co;
      nc::compress_device(m, tok_d, ntok, q, s, co, (int)nch);
      nc::dev_free(tok_d, s);
      nc::encode_container(q, ntok, co, mine_blob);
      nc::Nc05View v = nc::read_nc05(mine_blob.data(), mine_blob.size());
      for (auto &e : v.ents) {
        mine_tab.insert(mine_tab.end(), {e.tokens, e.bits, e.len});
        my_streams.insert(my_streams.end(), mine_blob.begin() + e.off, mine_blob.begin() + e.off + e.len);
      }
    }
    const uint32_t k = (nch + c->world - 1) / c->world;
    mine_tab.resize(3 * (size_t)k, 0);
    std::vector<uint32_t> all;
    gather_u32(c, mine_tab, all, s);
    std::vector<uint32_t> table(3 * (size_t)nch);
    for (uint32_t ch = 0; ch < nch; ++ch) {
      uint32_t r = ch / k, j = ch % k;
      for (int f = 0; f < 3; ++f) table[3 * ch + f] = all[(size_t)r * 3 * k + 3 * j + f];
    }
    std::vector<uint8_t> out;
    uint64_t off, tot;
    nc::shard_part(table.data(), nch, (uint8_t)q.flags, (uint16_t)q.tau_milli, c->world, c->rank,
                   my_streams.data(), my_streams.size(), out, off, tot);
    uint8_t *o = static_cast<uint8_t *>(std::malloc(out.size() + 1));
    if (!o) nc::fail(NC_ERR_NOMEM, "malloc");
    std::memcpy(o, out.data(), out.size());
    *part = o; *part_n = out.size(); *part_offset = off; *total_n = tot;
  });
}

nc_status nc_decompress_shard(nc_model *m, nc_comm *c, const uint8_t *in, size_t n, const nc_params *p,
                              void *cuda_stream, uint8_t **part, size_t *part_n, uint64_t *part_offset,
                              uint64_t *total_n) {
  if (!m || !c || (!in && n) || !part || !part_n || !part_offset || !total_n) return NC_ERR_INVALID;
  *part = nullptr; *part_n = 0;
  nc::stats() = nc::Stats{};
  return guard([&] {
    nc::Params q = nc::validate(p);
    cudaStream_t s = (cudaStream_t)cuda_stream;
    NC_CUDA(cudaSetDevice(m->device));
    nc::Nc05View v = nc::read_nc05(in, n);
    q.flags = v.flags;
    q.tau_milli = v.tau_milli;
    q.inv_tau = 1000.0 / v.tau_milli;
    const uint32_t nch = (uint32_t)v.ents.size();
    uint32_t c0, c1;
    nc::shard_range(nch, c->world, c->rank, c0, c1);
    nc::Nc05View mine = v;
    mine.ents.assign(v.ents.begin() + c0, v.ents.begin() + c1);
    std::vector<std::vector<uint32_t>> toks;
    if (c1 > c0) nc::decompress_device(m, in, mine, q, s, toks, (int)nch);
    std::string text;
    for (auto &t : toks) m->tok.decode(t.data(), t.size(), text);
    // one allgather of decoded byte lengths (split into two u32 halves)
    std::vector<uint32_t> len{(uint32_t)(text.size() & 0xFFFFFFFFu), (uint32_t)(text.size() >> 32)}, all;
    gather_u32(c, len, all, s);
    uint64_t before = 0, tot = 0;
    for (int r = 0; r < c->world; ++r) {
      uint64_t l = all[2 * r] | ((uint64_t)all[2 * r + 1] << 32);
      if (r < c->rank) before += l;
      tot += l;
    }
    uint8_t *o = static_cast<uint8_t *>(std::malloc(text.size() + 1));
    if (!o) nc::fail(NC_ERR_NOMEM, "malloc");
    std::memcpy(o, text.data(), text.size());
    *part = o; *part_n = text.size(); *part_offset = before; *total_n = tot;
  });
}

// host-only pieces of the shard plan, exported for the gloo multi-process tests
nc_status nc_host_walk_ctas(uint32_t V, uint32_t n_chunks, uint32_t *ctas) {
  if (!ctas) return NC_ERR_INVALID;
  *ctas = (uint32_t)nc::walk_ctas_per_chunk(V, (int)n_chunks);
  return NC_OK;
}

nc_status nc_host_shard_range(uint32_t n_chunks, int world, int rank, uint32_t *c0, uint32_t *c1) {
  if (!c0 || !c1 || world < 1 || rank < 0 || rank >= world) return NC_ERR_INVALID;
  nc::shard_range(n_chunks, world, rank, *c0, *c1);
  return NC_OK;
}

nc_status nc_host_shard_part(const uint32_t *table, uint32_t n_chunks, uint8_t flags, uint16_t tau_milli, int world,
                             int rank, const uint8_t *my_streams, size_t my_len, uint8_t **part, size_t *part_n,
                             uint64_t *part_offset, uint64_t *total_n) {
  if ((!table && n_chunks) || !part || !part_n || !part_offset || !total_n) return NC_ERR_INVALID;
  *part = nullptr; *part_n = 0;
  return guard([&] {
    std::vector<uint8_t> out;
    nc::shard_part(table, n_chunks, flags, tau_milli, world, rank, my_streams, my_len, out, *part_offset, *total_n);
    uint8_t *o = static_cast<uint8_t *>(std::malloc(out.size() + 1));
    if (!o) nc::fail(NC_ERR_NOMEM, "malloc");
    std::memcpy(o, out.data(), out.size());
    *part = o; *part_n = out.size();
  });
}

}  // extern "C"
