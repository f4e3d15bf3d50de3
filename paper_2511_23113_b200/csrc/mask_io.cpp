// DBSPMSK1 mask files (reference proj/include/dbsp/mask_io.hpp:17-207):
// 28-byte little-endian header -- magic "DBSPMSK1", u32 version 1, heads,
// q_blocks, kv_blocks, block_size -- then heads*q_blocks rows of
// ceil(kv_blocks/8) bytes, bit k at byte k/8, position k%8.  Writes are
// atomic (temp file + rename); parse errors name the byte offset.  Lets real
// PAROAttention / SpargeAttn mask dumps feed the planner and the kernel.
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "../../include/dbsp_b200.h"
#include "capi_util.hpp"
#include "core.hpp"

using namespace dbsp_core;

namespace {

constexpr char kMagic[8] = {'D', 'B', 'S', 'P', 'M', 'S', 'K', '1'};
constexpr uint32_t kVersion = 1;
constexpr size_t kHeader = 28;
constexpr uint64_t kMaxDim = 1u << 20;

void put32(std::string& s, uint32_t v) {
  for (int i = 0; i < 4; ++i) s.push_back(char((v >> (8 * i)) & 0xff));
}
uint32_t get32(const std::string& s, size_t at) {
  uint32_t v = 0;
  for (int i = 0; i < 4; ++i) v |= uint32_t(uint8_t(s[at + i])) << (8 * i);
  return v;
}

std::string slurp(const char* path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) fail(kIo, std::string("cannot open '") + path + "'");
  return std::string(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
}

struct Header {
  uint32_t heads, nq, nk, block_size;
};

Header parse_header(const std::string& d, const std::string& origin) {
  if (d.size() < 8 || std::memcmp(d.data(), kMagic, 8) != 0)
    fail(kParse, origin + ": bad magic at byte 0");
  if (d.size() < kHeader)
    fail(kParse, origin + ": truncated header at byte " + std::to_string(d.size()));
  const uint32_t version = get32(d, 8);
  if (version != kVersion)
    fail(kParse, origin + ": unsupported version " + std::to_string(version) + " at byte 8");
  Header h{get32(d, 12), get32(d, 16), get32(d, 20), get32(d, 24)};
  if (!h.heads || !h.nq || !h.nk || !h.block_size || h.heads > kMaxDim || h.nq > kMaxDim ||
      h.nk > kMaxDim)
    fail(kParse, origin + ": dimension out of range at byte 12");
  const uint64_t expected = kHeader + uint64_t(h.heads) * h.nq * ((h.nk + 7) / 8);
  if (d.size() != expected)
    fail(kParse, origin + ": payload size mismatch: expected " + std::to_string(expected) +
                     " bytes, got " + std::to_string(d.size()) + " (payload starts at byte " +
                     std::to_string(kHeader) + ")");
  return h;
}

}  // namespace

using dbsp_capi::guard;

extern "C" {

int dbsp_save_mask_set(const dbsp_mask_set* set, const char* path) {
  return guard([&] {
    if (!set || !path) fail(kContract, "null argument");
    const MaskView m = make_view(set->heads, set->num_heads, set->num_q_blocks, set->num_kv_blocks,
                                 set->block_size);
    const size_t row_bytes = (size_t(m.nk) + 7) / 8;
    std::string out;
    out.reserve(kHeader + size_t(m.H) * m.nq * row_bytes);
    out.append(kMagic, 8);
    put32(out, kVersion);
    put32(out, m.H);
    put32(out, m.nq);
    put32(out, m.nk);
    put32(out, m.block_size);
    for (uint32_t h = 0; h < m.H; ++h)
      for (uint32_t q = 0; q < m.nq; ++q) {
        const uint64_t* r = m.row(h, q);
        for (size_t b = 0; b < row_bytes; ++b) out.push_back(char((r[b / 8] >> (8 * (b % 8))) & 0xff));
      }
    namespace fs = std::filesystem;
    const fs::path dst(path), tmp = std::string(path) + ".tmp";
    {
      std::ofstream f(tmp, std::ios::binary | std::ios::trunc);
      if (!f) fail(kIo, "cannot open '" + tmp.string() + "' for writing");
      f.write(out.data(), std::streamsize(out.size()));
      if (!f) fail(kIo, "write failed for '" + tmp.string() + "'");
    }
    std::error_code ec;
    fs::rename(tmp, dst, ec);
    if (ec) fail(kIo, "cannot rename '" + tmp.string() + "' to '" + dst.string() + "'");
  });
}

int dbsp_load_mask_set_header(const char* path, uint32_t* heads, uint32_t* q_blocks,
                              uint32_t* kv_blocks, uint32_t* block_size) {
  return guard([&] {
    if (!path) fail(kContract, "null path");
    const Header h = parse_header(slurp(path), path);
    if (heads) *heads = h.heads;
    if (q_blocks) *q_blocks = h.nq;
    if (kv_blocks) *kv_blocks = h.nk;
    if (block_size) *block_size = h.block_size;
  });
}

int dbsp_load_mask_set(const char* path, uint64_t* words_out) {
  return guard([&] {
    if (!path || !words_out) fail(kContract, "null argument");
    const std::string d = slurp(path);
    const Header h = parse_header(d, path);
    const size_t row_bytes = (size_t(h.nk) + 7) / 8, wpr = (size_t(h.nk) + 63) / 64;
    std::fill(words_out, words_out + size_t(h.heads) * h.nq * wpr, 0ull);
    size_t off = kHeader;
    for (uint64_t r = 0; r < uint64_t(h.heads) * h.nq; ++r, off += row_bytes) {
      uint64_t* w = words_out + r * wpr;
      for (size_t b = 0; b < row_bytes; ++b) {
        const uint64_t byte = uint8_t(d[off + b]);
        if (!byte) continue;
        const size_t k0 = b * 8;
        if (k0 + 8 > h.nk && (byte >> (h.nk - k0)) != 0)
          fail(kParse, std::string(path) + ": padding bit set at byte " + std::to_string(off + b));
        w[k0 / 64] |= byte << (k0 % 64);
      }
    }
  });
}

}  // extern "C"
