// DBSPMSK1 mask files — the drop-in counterpart of the reference's
// proj/include/dbsp/mask_io.hpp (save_mask_set :131-147, load_mask_set
// :149-207, JSON fixture sidecars :80-127).  Binary files are written and
// parsed in libdbsp_b200.so (dbsp_save_mask_set / dbsp_load_mask_set: atomic
// temp-file + rename writes, parse errors that name the byte offset), so a
// file written here is byte-identical to one the reference writes
// (tests/test_mask_io.py).  Failures throw the reference's classes: io_error
// for the filesystem, parse_error for contents.
#pragma once

#include <cstdint>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "../dbsp_b200.h"
#include "error.hpp"
#include "mask.hpp"
#include "metrics.hpp"  // json.hpp when the include path has it (DBSP_HAVE_JSON)

namespace dbsp {

inline void save_mask_set(const AttentionMaskSet& set, const std::filesystem::path& path) {
  const detail::MaskView v(set);
  detail::check(dbsp_save_mask_set(v.get(), path.string().c_str()));
}

namespace detail {

inline std::string slurp_file(const std::filesystem::path& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw io_error("cannot open '" + path.string() + "'");
  return std::string(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
}

#ifdef DBSP_HAVE_JSON
// Fixture sidecar: {"heads", "q_blocks", "kv_blocks", "block_size", "rows"}
// with heads*q_blocks rows of ceil(kv_blocks/8) bytes as hex, byte b holding
// keys 8b..8b+7 least-significant bit first (the DBSPMSK1 row bytes).
inline AttentionMaskSet sidecar_mask_set(const std::string& text, const std::string& origin) {
  nlohmann::json j;
  try {
    j = nlohmann::json::parse(text);
  } catch (const nlohmann::json::exception& e) {
    throw parse_error(origin + ": invalid JSON sidecar: " + e.what());
  }
  try {
    const uint32_t H = j.at("heads").get<uint32_t>(), nq = j.at("q_blocks").get<uint32_t>();
    const uint32_t nk = j.at("kv_blocks").get<uint32_t>(), bs = j.at("block_size").get<uint32_t>();
    if (!H || !nq || !nk || !bs) throw parse_error(origin + ": sidecar dimensions must be positive");
    const auto& rows = j.at("rows");
    if (rows.size() != size_t(H) * nq)
      throw parse_error(origin + ": sidecar needs heads*q_blocks row strings, got " +
                        std::to_string(rows.size()));
    const size_t row_bytes = (size_t(nk) + 7) / 8, wpr = (size_t(nk) + 63) / 64;
    auto hexval = [&](char c, size_t r) -> uint64_t {
      if (c >= '0' && c <= '9') return uint64_t(c - '0');
      if (c >= 'a' && c <= 'f') return uint64_t(c - 'a' + 10);
      if (c >= 'A' && c <= 'F') return uint64_t(c - 'A' + 10);
      throw parse_error(origin + ": row " + std::to_string(r) + " has a non-hex character");
    };
    // keys past nk in the last byte are ignored, as the reference does
    const uint64_t tail = (nk % 64) ? ((uint64_t(1) << (nk % 64)) - 1) : ~uint64_t(0);
    std::vector<uint64_t> words(size_t(H) * nq * wpr, 0);
    for (size_t r = 0; r < rows.size(); ++r) {
      const std::string hex = rows[r].get<std::string>();
      if (hex.size() != 2 * row_bytes)
        throw parse_error(origin + ": row " + std::to_string(r) + " needs " + std::to_string(2 * row_bytes) +
                          " hex chars");
      uint64_t* w = words.data() + r * wpr;
      for (size_t b = 0; b < row_bytes; ++b)
        w[b / 8] |= ((hexval(hex[2 * b], r) << 4) | hexval(hex[2 * b + 1], r)) << (8 * (b % 8));
      w[wpr - 1] &= tail;
    }
    return from_words(words, H, nq, nk, bs);
  } catch (const nlohmann::json::exception& e) {
    throw parse_error(origin + ": sidecar is missing a required key: " + e.what());
  }
}
#endif

}  // namespace detail

inline AttentionMaskSet load_mask_set(const std::filesystem::path& path) {
  const std::string p = path.string();
  {
    // Not a DBSPMSK1 file but a JSON object: a fixture sidecar.
    const std::string data = detail::slurp_file(path);
    if (data.size() < 8 || std::memcmp(data.data(), "DBSPMSK1", 8) != 0) {
      const size_t first = data.find_first_not_of(" \t\r\n");
      if (first != std::string::npos && data[first] == '{') {
#ifdef DBSP_HAVE_JSON
        return detail::sidecar_mask_set(data, p);
#else
        throw parse_error(p + ": JSON sidecars need json.hpp on the include path");
#endif
      }
    }
  }
  uint32_t H = 0, nq = 0, nk = 0, bs = 0;
  detail::check(dbsp_load_mask_set_header(p.c_str(), &H, &nq, &nk, &bs));
  std::vector<uint64_t> words(size_t(H) * nq * ((size_t(nk) + 63) / 64));
  detail::check(dbsp_load_mask_set(p.c_str(), words.data()));
  return detail::from_words(words, H, nq, nk, bs);
}

}  // namespace dbsp
