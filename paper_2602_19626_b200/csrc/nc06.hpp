// NC06 hybrid binary format, host side (host_nc06.cpp).
#pragma once
#include <cstddef>
#include <cstdint>
#include <vector>

#include "nc_internal.hpp"

namespace nc {

constexpr uint8_t kBinary = 0, kText = 1;             // entry kinds
constexpr uint8_t kRaw = 0, kDeflate = 1, kLzma = 2;  // binary section methods

struct Region {
  uint8_t kind;
  uint64_t len;
};

// segmentation of arbitrary bytes into alternating text / binary regions
std::vector<Region> segment(const uint8_t *in, size_t n);
// binary blob codec: returns the method, payload in out
uint8_t blob_encode(const uint8_t *in, size_t n, std::vector<uint8_t> &out);
void blob_decode(uint8_t method, const uint8_t *in, size_t n, size_t expect, std::vector<uint8_t> &out);

// container: the text section is taken from a full NC05 container of the text document
void write_nc06(uint8_t flags, uint16_t tau_milli, const std::vector<Region> &regs, uint8_t method,
                const std::vector<uint8_t> &payload, const uint8_t *nc05, size_t nc05_n, std::vector<uint8_t> &out);
struct Nc06View {
  uint8_t flags = 0, method = 0;
  uint16_t tau_milli = 0;
  std::vector<Region> regs;
  uint64_t text_len = 0, bin_len = 0;
  size_t payload_off = 0, payload_len = 0, text_off = 0;
};
Nc06View read_nc06(const uint8_t *in, size_t n);

}  // namespace nc
