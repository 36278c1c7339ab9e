// HF-format checkpoints (config.json + model.safetensors + tokenizer.json) and the byte-level
// BPE tokenizer (hf_loader.cpp).
#pragma once
#include <cstdint>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "nc_internal.hpp"

namespace nc {

class BpeTokenizer {
 public:
  // parse tokenizer.json; fills the id -> bytes table (size V) and the special-token count
  void build(const std::string &tokenizer_json, uint32_t V, std::vector<std::string> &vocab_bytes,
             uint32_t &n_special);
  void encode(const uint8_t *data, size_t n, std::vector<uint32_t> &out) const;

 private:
  struct Merge { uint32_t rank, id; };
  void bpe_word(const uint8_t *w, size_t n, std::vector<uint32_t> &out) const;
  std::unordered_map<uint64_t, Merge> merges_;   // (left id, right id) -> rank, merged id
  uint32_t byte_id_[256] = {};
  bool digits_ = false;
};

// config.json + model.safetensors (HF Llama names, F32/F16/BF16) -> the NCW1 tensor order in
// memory; tokenizer.json -> bpe and the vocabulary bytes
NcwFile read_hf(const std::string &dir, std::unique_ptr<BpeTokenizer> &bpe);

}  // namespace nc
