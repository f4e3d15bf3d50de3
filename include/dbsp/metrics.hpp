// Strategies, partition plans, workload tables and the sparse imbalance ratio
// rho_s — drop-in counterpart of the reference's proj/include/dbsp/metrics.hpp
// (ParallelStrategy :20-51, enumerate_strategies :56-66, PartitionPlan /
// validate_plan / default_plan :70-113, WorkloadTable / workload_table
// :117-168, imbalance_ratio :173-186, ExchangeVolume :190-211, JSON :213-246).
// Computation runs in libdbsp_b200.so (bit-identical results).
#pragma once

#include <cstdint>
#include <string>
#include <string_view>
#include <vector>

#include "../dbsp_b200.h"
#include "error.hpp"
#include "mask.hpp"

#if __has_include(<json.hpp>)
#include <json.hpp>
#define DBSP_HAVE_JSON 1
#endif

namespace dbsp {

// UxRy: x-way Ulysses (heads) times y-way ring (sequence); x*y GPUs.
struct ParallelStrategy {
  uint32_t ulysses = 1;  // x
  uint32_t ring = 1;     // y
  uint32_t gpus() const { return ulysses * ring; }
  auto operator<=>(const ParallelStrategy&) const = default;
};

inline std::string to_string(ParallelStrategy s) {
  return "U" + std::to_string(s.ulysses) + "R" + std::to_string(s.ring);
}

inline ParallelStrategy parse_strategy(std::string_view text) {
  auto bad = [&]() -> ParallelStrategy {
    throw config_error("invalid strategy '" + std::string(text) + "' (expected UxRy)");
  };
  if (text.size() < 4 || text[0] != 'U') return bad();
  const size_t r = text.find('R', 1);
  if (r == std::string_view::npos || r == 1 || r + 1 >= text.size()) return bad();
  auto number = [&](std::string_view digits, uint32_t& out) {
    uint64_t v = 0;
    for (char c : digits) {
      if (c < '0' || c > '9') return false;
      v = v * 10 + uint64_t(c - '0');
      if (v > 0xffffffffu) return false;
    }
    out = uint32_t(v);
    return true;
  };
  ParallelStrategy s;
  if (!number(text.substr(1, r - 1), s.ulysses) || !number(text.substr(r + 1), s.ring)) return bad();
  if (s.ulysses < 1 || s.ring < 1) return bad();
  return s;
}

inline std::vector<ParallelStrategy> enumerate_strategies(uint32_t total_gpus) {
  dbsp_strategy buf[33];
  uint32_t n = 0;
  detail::check(dbsp_enumerate_strategies(total_gpus, buf, &n));
  std::vector<ParallelStrategy> out;
  for (uint32_t i = 0; i < n; ++i) out.push_back({buf[i].ulysses, buf[i].ring});
  return out;
}

struct PartitionPlan {
  std::vector<uint32_t> head_assignment;  // head -> Ulysses rank in [0, x)
  std::vector<uint32_t> q_assignment;     // Q block -> ring rank in [0, y)
  std::vector<uint32_t> kv_assignment;    // KV block -> ring group in [0, y)
  bool operator==(const PartitionPlan&) const = default;
};

namespace detail {

inline dbsp_strategy cs(ParallelStrategy s) { return dbsp_strategy{s.ulysses, s.ring}; }

// Mutable C view of a plan (the C ABI takes non-const arrays for outputs).
inline dbsp_plan cplan(PartitionPlan& p) {
  return dbsp_plan{p.head_assignment.data(), p.q_assignment.data(), p.kv_assignment.data()};
}
inline dbsp_plan cplan(const PartitionPlan& p) { return cplan(const_cast<PartitionPlan&>(p)); }

inline PartitionPlan sized_plan(const AttentionMaskSet& set) {
  PartitionPlan p;
  p.head_assignment.resize(set.num_heads());
  p.q_assignment.resize(set.num_q_blocks());
  p.kv_assignment.resize(set.num_kv_blocks());
  return p;
}

inline void check_dims(const AttentionMaskSet& set, const PartitionPlan& p) {
  if (p.head_assignment.size() != set.num_heads() || p.q_assignment.size() != set.num_q_blocks() ||
      p.kv_assignment.size() != set.num_kv_blocks())
    throw contract_error("plan dimensions do not match the mask set");
}

}  // namespace detail

inline void validate_plan(const AttentionMaskSet& set, ParallelStrategy strategy,
                          const PartitionPlan& plan) {
  detail::check_dims(set, plan);
  detail::MaskView v(set);
  const dbsp_plan c = detail::cplan(plan);
  detail::check(dbsp_validate_plan(v.get(), detail::cs(strategy), &c));
}

inline PartitionPlan default_plan(const AttentionMaskSet& set, ParallelStrategy strategy) {
  detail::MaskView v(set);
  PartitionPlan p = detail::sized_plan(set);
  dbsp_plan c = detail::cplan(p);
  detail::check(dbsp_default_plan(v.get(), detail::cs(strategy), &c));
  return p;
}

// Dense-block counts per synchronisation period (rows) and GPU u*y + r (columns).
struct WorkloadTable {
  uint32_t gpus = 1;
  std::vector<std::vector<uint64_t>> counts;
  uint32_t periods() const { return uint32_t(counts.size()); }
  uint64_t total() const {
    uint64_t t = 0;
    for (const auto& row : counts)
      for (uint64_t c : row) t += c;
    return t;
  }
};

inline WorkloadTable workload_table(const AttentionMaskSet& set, ParallelStrategy strategy,
                                    const PartitionPlan& plan) {
  detail::check_dims(set, plan);
  detail::MaskView v(set);
  const dbsp_plan c = detail::cplan(plan);
  const uint32_t G = strategy.gpus(), rows = strategy.ring > 1 ? strategy.ring : 1;
  std::vector<uint64_t> flat(size_t(rows) * G);
  uint32_t periods = 0;
  detail::check(dbsp_workload_table(v.get(), detail::cs(strategy), &c, flat.data(), &periods));
  WorkloadTable t;
  t.gpus = G;
  for (uint32_t p = 0; p < periods; ++p)
    t.counts.emplace_back(flat.begin() + size_t(p) * G, flat.begin() + size_t(p + 1) * G);
  return t;
}

inline double imbalance_ratio(const WorkloadTable& table) {
  std::vector<uint64_t> flat;
  for (const auto& row : table.counts) {
    if (row.size() != table.gpus) throw contract_error("workload row width differs from gpus");
    flat.insert(flat.end(), row.begin(), row.end());
  }
  double out = 1.0;
  detail::check(dbsp_imbalance_ratio(flat.data(), table.periods(), table.gpus, &out));
  return out;
}

struct ExchangeVolume {
  uint64_t q_blocks_moved = 0;
  uint64_t kv_blocks_moved = 0;
  uint64_t token_payload = 0;
  bool operator==(const ExchangeVolume&) const = default;
};

inline ExchangeVolume exchange_volume(const AttentionMaskSet& set, ParallelStrategy strategy,
                                      const PartitionPlan& plan) {
  detail::check_dims(set, plan);
  detail::MaskView v(set);
  const dbsp_plan c = detail::cplan(plan);
  dbsp_exchange e{};
  detail::check(dbsp_exchange_volume(v.get(), detail::cs(strategy), &c, &e));
  return {e.q_blocks_moved, e.kv_blocks_moved, e.token_payload};
}

#ifdef DBSP_HAVE_JSON
inline nlohmann::json workload_to_json(const WorkloadTable& table) {
  return {{"periods", table.periods()}, {"gpus", table.gpus}, {"counts", table.counts},
          {"rho_s", imbalance_ratio(table)}};
}

inline nlohmann::json plan_to_json(ParallelStrategy strategy, const PartitionPlan& plan) {
  return {{"strategy", {{"x", strategy.ulysses}, {"y", strategy.ring}}},
          {"head_assignment", plan.head_assignment},
          {"q_assignment", plan.q_assignment},
          {"kv_assignment", plan.kv_assignment}};
}

inline PartitionPlan plan_from_json(const nlohmann::json& j,
                                    ParallelStrategy* strategy_out = nullptr) {
  try {
    if (strategy_out) {
      strategy_out->ulysses = j.at("strategy").at("x").get<uint32_t>();
      strategy_out->ring = j.at("strategy").at("y").get<uint32_t>();
    }
    PartitionPlan p;
    p.head_assignment = j.at("head_assignment").get<std::vector<uint32_t>>();
    p.q_assignment = j.at("q_assignment").get<std::vector<uint32_t>>();
    p.kv_assignment = j.at("kv_assignment").get<std::vector<uint32_t>>();
    return p;
  } catch (const nlohmann::json::exception& e) {
    throw parse_error(std::string("invalid plan JSON: ") + e.what());
  }
}
#endif

}  // namespace dbsp
