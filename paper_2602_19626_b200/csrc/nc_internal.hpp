// Internal declarations shared by the C++ host runtime and the CUDA engine.
#pragma once
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>
#include <stdexcept>

#include "../../include/nc.h"

namespace nc {

// ---------------------------------------------------------------- errors ---
struct Error : std::runtime_error {
  nc_status code;
  Error(nc_status c, const std::string &m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(nc_status c, const std::string &m) { throw Error(c, m); }
void set_last_error(const std::string &m);  // thread-local, read by nc_last_error()

// ------------------------------------------------------------ model shape --
struct Shape {
  uint32_t n_layers, d, H, KV, dh, d_ff, V, bos, n_special;
  double rope_theta, eps;
};

// ------------------------------------------------------------- host side ---
struct NcwFile {  // parsed NCW1 (synth/weights.py documents the layout)
  Shape s;
  std::vector<char> raw;            // whole file
  size_t tensor_off = 64;           // fp32 tensors start
  std::vector<std::string> vocab;   // token id -> bytes
  const float *tensor(size_t off_floats) const {
    return reinterpret_cast<const float *>(raw.data() + tensor_off) + off_floats;
  }
};
NcwFile read_ncw(const std::string &path);

// Greedy longest-match tokenizer over the vocabulary (D30); specials skipped.
class Tokenizer {
 public:
  void build(const std::vector<std::string> &vocab, uint32_t n_special);
  void encode(const uint8_t *data, size_t n, std::vector<uint32_t> &out) const;
  void decode(const uint32_t *ids, size_t n, std::string &out) const;
  bool empty() const { return nodes_.empty(); }

 private:
  struct Node {
    int32_t tok = -1;
    uint32_t first = 0, count = 0;  // children in edges_[first, first+count), sorted by byte
  };
  struct Edge {
    uint8_t byte;
    uint32_t child;
  };
  std::vector<Node> nodes_;
  std::vector<Edge> edges_;
  std::vector<std::string> vocab_;
  uint32_t root_children_[256];
};

// Chunk split (D28): returns cut offsets, chunk i = [cuts[i], cuts[i+1]).
std::vector<uint64_t> split_chunks(const uint8_t *in, size_t n, uint32_t n_chunks);

// 32-bit WNC arithmetic coder (D7-D8).
class WncEncoder {
 public:
  void encode(uint32_t cum_lo, uint32_t freq, uint32_t cdf_bits);
  void finish(std::vector<uint8_t> &out, uint64_t &bit_count);

 private:
  void put(uint32_t bit);
  void emit(uint32_t bit);
  uint64_t low_ = 0, high_ = 0xFFFFFFFFull, pending_ = 0;
  std::vector<uint8_t> bytes_;
  uint32_t acc_ = 0, nacc_ = 0;
  uint64_t nbits_ = 0;
};

// rANS coder (the paper's future-work ANS; reading D39): 64-bit state, L = 2^31,
// 32-bit renormalisation words, symbols encoded in reverse; the stream holds the words in the
// decoder's order, big-endian; bit_count = 32 x words.
void ans_encode(const uint32_t *cum, const uint32_t *freq, size_t n, uint32_t cdf_bits,
                std::vector<uint8_t> &out, uint64_t &bit_count);

// NC05 container.
struct Nc05Chunk {
  uint32_t tokens, bits;
  std::vector<uint8_t> stream;
};
void write_nc05(uint8_t flags, uint16_t tau_milli, const std::vector<Nc05Chunk> &chunks,
                std::vector<uint8_t> &out);
struct Nc05View {
  uint8_t flags;
  uint16_t tau_milli;
  struct Ent {
    uint32_t tokens, bits, len;
    uint64_t off;
  };
  std::vector<Ent> ents;
};
Nc05View read_nc05(const uint8_t *in, size_t n);

// validated parameter set
struct Params {
  uint32_t cdf_bits, flags, tau_milli, window, slide, warmup, orders, cap, n_chunks,
      chunks_per_gpu, max_slab_rows, debug_dump;
  double eta, alpha, inv_tau;
  bool refresh;     // NEXT-4: refresh window semantics (NC_WINDOW_REFRESH)
  uint32_t lmax;    // D10: L_max = window, or window - 1 (NC_WINDOW_LMAX_M1)
  uint32_t coder;   // NC_CODER_WNC (0) or NC_CODER_ANS (1)
};
Params validate(const nc_params *p);

}  // namespace nc
