// Per-head block masks of one attention call — the drop-in counterpart of the
// reference's proj/include/dbsp/mask.hpp (BlockMask :22-78, AttentionMaskSet
// :83-113, GeneratorSpec :137-162, generate/perturb :233-273, popcounts
// :275-292).  Storage is the same Q-major u64 row layout; the generators and
// counts run in libdbsp_b200.so through the C ABI (bit-identical output,
// pinned by tests/test_planner_golden.py).
#pragma once

#include <bit>
#include <cmath>
#include <cstdint>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "../dbsp_b200.h"
#include "error.hpp"
#include "rng.hpp"

namespace dbsp {

// Bit (q, k) set: the 64x64 tile between Q block q and KV block k is computed.
class BlockMask {
 public:
  BlockMask(uint32_t num_q_blocks, uint32_t num_kv_blocks)
      : nq_(num_q_blocks), nk_(num_kv_blocks), wpr_((size_t(num_kv_blocks) + 63) / 64),
        words_(size_t(num_q_blocks) * wpr_, 0) {
    if (nq_ == 0 || nk_ == 0) throw config_error("BlockMask dimensions must be positive");
  }

  uint32_t num_q_blocks() const { return nq_; }
  uint32_t num_kv_blocks() const { return nk_; }
  size_t words_per_row() const { return wpr_; }

  bool get(uint32_t q, uint32_t k) const { return (words_[at(q, k)] >> (k & 63)) & 1u; }
  void set(uint32_t q, uint32_t k, bool v) {
    const uint64_t bit = uint64_t(1) << (k & 63);
    if (v)
      words_[at(q, k)] |= bit;
    else
      words_[at(q, k)] &= ~bit;
  }
  void flip(uint32_t q, uint32_t k) { words_[at(q, k)] ^= uint64_t(1) << (k & 63); }
  uint64_t row_word(uint32_t q, size_t w) const { return words_[size_t(q) * wpr_ + w]; }
  uint64_t row_popcount(uint32_t q) const {
    uint64_t c = 0;
    for (size_t w = 0; w < wpr_; ++w) c += uint64_t(std::popcount(row_word(q, w)));
    return c;
  }
  uint64_t popcount() const {
    uint64_t c = 0;
    for (uint64_t w : words_) c += uint64_t(std::popcount(w));
    return c;
  }

  // Extension: raw rows for the C ABI (Nq * words_per_row words).
  const uint64_t* data() const { return words_.data(); }
  uint64_t* data() { return words_.data(); }

  bool operator==(const BlockMask&) const = default;

 private:
  size_t at(uint32_t q, uint32_t k) const { return size_t(q) * wpr_ + (k >> 6); }
  uint32_t nq_, nk_;
  size_t wpr_;
  std::vector<uint64_t> words_;
};

class AttentionMaskSet {
 public:
  AttentionMaskSet(std::vector<BlockMask> masks, uint32_t block_size)
      : masks_(std::move(masks)), block_size_(block_size) {
    if (masks_.empty()) throw config_error("mask set needs at least one head");
    if (block_size_ == 0) throw config_error("block_size must be positive");
    for (const BlockMask& m : masks_)
      if (m.num_q_blocks() != masks_[0].num_q_blocks() ||
          m.num_kv_blocks() != masks_[0].num_kv_blocks())
        throw config_error("all heads must share identical grid dimensions");
  }

  uint32_t num_heads() const { return uint32_t(masks_.size()); }
  uint32_t num_q_blocks() const { return masks_[0].num_q_blocks(); }
  uint32_t num_kv_blocks() const { return masks_[0].num_kv_blocks(); }
  uint32_t block_size() const { return block_size_; }
  const BlockMask& head(uint32_t j) const { return masks_[j]; }
  const std::vector<BlockMask>& masks() const { return masks_; }
  uint64_t grid_cells() const { return uint64_t(num_heads()) * num_q_blocks() * num_kv_blocks(); }

  bool operator==(const AttentionMaskSet& o) const {
    return block_size_ == o.block_size_ && masks_ == o.masks_;
  }

 private:
  std::vector<BlockMask> masks_;
  uint32_t block_size_;
};

namespace detail {

// C-ABI view of a mask set: one row pointer per head, no copy.
struct MaskView {
  explicit MaskView(const AttentionMaskSet& s) {
    ptrs.reserve(s.num_heads());
    for (const BlockMask& m : s.masks()) ptrs.push_back(m.data());
    c.heads = ptrs.data();
    c.num_heads = s.num_heads();
    c.num_q_blocks = s.num_q_blocks();
    c.num_kv_blocks = s.num_kv_blocks();
    c.block_size = s.block_size();
  }
  MaskView(const MaskView&) = delete;
  MaskView& operator=(const MaskView&) = delete;
  const dbsp_mask_set* get() const { return &c; }
  std::vector<const uint64_t*> ptrs;
  dbsp_mask_set c{};
};

inline AttentionMaskSet from_words(const std::vector<uint64_t>& words, uint32_t H, uint32_t nq,
                                   uint32_t nk, uint32_t block_size) {
  std::vector<BlockMask> masks;
  masks.reserve(H);
  const size_t per = size_t(nq) * ((size_t(nk) + 63) / 64);
  for (uint32_t h = 0; h < H; ++h) {
    BlockMask m(nq, nk);
    std::copy(words.begin() + per * h, words.begin() + per * (h + 1), m.data());
    masks.push_back(std::move(m));
  }
  return AttentionMaskSet(std::move(masks), block_size);
}

}  // namespace detail

enum class MaskPattern { uniform_random, banded_diagonal, clustered };

inline const char* to_string(MaskPattern p) {
  switch (p) {
    case MaskPattern::uniform_random: return "random";
    case MaskPattern::banded_diagonal: return "banded";
    case MaskPattern::clustered: return "clustered";
  }
  return "?";
}

inline MaskPattern parse_pattern(std::string_view s) {
  if (s == "random" || s == "uniform-random") return MaskPattern::uniform_random;
  if (s == "banded" || s == "banded-diagonal") return MaskPattern::banded_diagonal;
  if (s == "clustered") return MaskPattern::clustered;
  throw config_error("unknown mask pattern '" + std::string(s) +
                     "' (expected random|banded|clustered)");
}

struct GeneratorSpec {
  uint32_t num_heads = 1;
  uint32_t num_q_blocks = 1;
  uint32_t num_kv_blocks = 1;
  uint32_t block_size = 64;
  MaskPattern pattern = MaskPattern::uniform_random;
  double min_density = 0.5;
  double max_density = 0.5;
  double skew = 1.0;
  uint64_t seed = 0;

  void validate() const {
    if (num_heads == 0 || num_q_blocks == 0 || num_kv_blocks == 0 || block_size == 0)
      throw config_error("generator dimensions must be positive");
    if (!(min_density >= 0.0) || !(max_density <= 1.0) || !(min_density <= max_density))
      throw config_error("density law requires 0 <= min_density <= max_density <= 1");
    if (!(skew > 0.0)) throw config_error("skew exponent must be > 0");
  }
  // Head h's target density: min + (max - min) * (h / (H-1))^skew.
  double head_density(uint32_t h) const {
    const double t = num_heads > 1 ? std::pow(double(h) / (num_heads - 1), skew) : 0.0;
    return min_density + (max_density - min_density) * t;
  }
};

inline AttentionMaskSet generate_mask_set(const GeneratorSpec& spec) {
  spec.validate();
  dbsp_generator_spec c{spec.num_heads, spec.num_q_blocks, spec.num_kv_blocks, spec.block_size,
                        uint32_t(spec.pattern), spec.min_density, spec.max_density, spec.skew,
                        spec.seed};
  std::vector<uint64_t> words(size_t(spec.num_heads) * spec.num_q_blocks *
                              ((size_t(spec.num_kv_blocks) + 63) / 64));
  detail::check(dbsp_generate_mask_set(&c, words.data()));
  return detail::from_words(words, spec.num_heads, spec.num_q_blocks, spec.num_kv_blocks,
                            spec.block_size);
}

inline AttentionMaskSet perturb_mask_set(const AttentionMaskSet& set, double flip_rate,
                                         uint64_t seed) {
  detail::MaskView v(set);
  std::vector<uint64_t> words(size_t(set.num_heads()) * set.num_q_blocks() *
                              set.head(0).words_per_row());
  detail::check(dbsp_perturb_mask_set(v.get(),flip_rate, seed, words.data()));
  return detail::from_words(words, set.num_heads(), set.num_q_blocks(), set.num_kv_blocks(),
                            set.block_size());
}

inline uint64_t total_blocks(const AttentionMaskSet& set) {
  detail::MaskView v(set);
  uint64_t out = 0;
  detail::check(dbsp_total_blocks(v.get(),&out));
  return out;
}

inline double density(const AttentionMaskSet& set) {
  detail::MaskView v(set);
  double out = 0;
  detail::check(dbsp_density(v.get(),&out));
  return out;
}

inline std::vector<uint64_t> blocks_per_head(const AttentionMaskSet& set) {
  detail::MaskView v(set);
  std::vector<uint64_t> out(set.num_heads());
  detail::check(dbsp_blocks_per_head(v.get(),out.data()));
  return out;
}

}  // namespace dbsp
