// Dual-balanced partitioner — drop-in counterpart of the reference's
// proj/include/dbsp/planner.hpp (PlannerConfig :21-35, PlanOutcome :37-42,
// summed_grid :47-61, head_level_imbalance :65-76, partition_heads :96-112,
// biased greedy :119-145, partition_blocks :151-170, plan_dual :175-217,
// brute-force oracles :249-338).  The planning runs in libdbsp_b200.so (host
// C++, assignments and doubles bit-identical to the reference).
#pragma once

#include <cmath>
#include <cstdint>
#include <limits>
#include <utility>
#include <vector>

#include "../dbsp_b200.h"
#include "error.hpp"
#include "mask.hpp"
#include "metrics.hpp"

namespace dbsp {

inline constexpr double kInfiniteReward = std::numeric_limits<double>::infinity();

struct PlannerConfig {
  double reuse_threshold = 1.10;  // P_s: keep the previous head plan while its rho <= P_s
  double exchange_reward = 0.0;   // R_b: home-rank bias of the block greedy (inf = never move)
  void validate() const {
    if (!(reuse_threshold >= 1.0)) throw config_error("reuse threshold must be >= 1");
    if (std::isnan(exchange_reward) || exchange_reward < 0.0)
      throw config_error("exchange reward must be >= 0 or infinite");
  }
};

struct PlanOutcome {
  PartitionPlan plan;
  bool head_replanned = false;
  double rho_pre = 1.0;
  double rho_post = 1.0;
};

inline std::vector<uint64_t> summed_grid(const AttentionMaskSet& set) {
  detail::MaskView v(set);
  std::vector<uint64_t> g(size_t(set.num_q_blocks()) * set.num_kv_blocks());
  detail::check(dbsp_summed_grid(v.get(), g.data()));
  return g;
}

inline double head_level_imbalance(const std::vector<uint64_t>& weights,
                                   const std::vector<uint32_t>& assignment, uint32_t x) {
  if (assignment.size() != weights.size())
    throw contract_error("assignment size differs from weights");
  double out = 1.0;
  detail::check(dbsp_head_level_imbalance(weights.data(), assignment.data(),
                                          uint32_t(weights.size()), x, &out));
  return out;
}

inline std::vector<uint32_t> partition_heads(const AttentionMaskSet& set, uint32_t x) {
  detail::MaskView v(set);
  std::vector<uint32_t> a(set.num_heads());
  detail::check(dbsp_partition_heads(v.get(), x, a.data()));
  return a;
}

namespace detail {

inline std::vector<uint32_t> biased_greedy(const std::vector<uint64_t>& weights, uint32_t y,
                                           double reward) {
  std::vector<uint32_t> a(weights.size());
  check(dbsp_biased_greedy(weights.data(), uint32_t(weights.size()), y, reward, a.data()));
  return a;
}

}  // namespace detail

inline std::pair<std::vector<uint32_t>, std::vector<uint32_t>> partition_blocks(
    const AttentionMaskSet& set, uint32_t y, double reward) {
  detail::MaskView v(set);
  std::vector<uint32_t> q(set.num_q_blocks()), kv(set.num_kv_blocks());
  detail::check(dbsp_partition_blocks(v.get(), y, reward, q.data(), kv.data()));
  return {std::move(q), std::move(kv)};
}

inline PlanOutcome plan_dual(const AttentionMaskSet& set, ParallelStrategy strategy,
                             const PlannerConfig& config, const PartitionPlan* prev = nullptr) {
  config.validate();  // same check order as the reference: config, then prev
  if (prev) detail::check_dims(set, *prev);
  detail::MaskView v(set);
  PlanOutcome out;
  out.plan = detail::sized_plan(set);
  dbsp_plan c = detail::cplan(out.plan);
  const dbsp_planner_config cfg{config.reuse_threshold, config.exchange_reward};
  dbsp_plan prev_c{};
  if (prev) prev_c = detail::cplan(*prev);
  dbsp_plan_outcome oc{};
  detail::check(dbsp_plan_dual(v.get(), detail::cs(strategy), &cfg, prev ? &prev_c : nullptr, &c, &oc));
  out.head_replanned = oc.head_replanned != 0;
  out.rho_pre = oc.rho_pre;
  out.rho_post = oc.rho_post;
  return out;
}

inline std::vector<uint32_t> brute_force_heads(const AttentionMaskSet& set, uint32_t x) {
  detail::MaskView v(set);
  std::vector<uint32_t> a(set.num_heads());
  detail::check(dbsp_brute_force_heads(v.get(), x, a.data()));
  return a;
}

struct BlockOracleResult {
  std::vector<uint32_t> q_assignment;
  std::vector<uint32_t> kv_assignment;
  double rho = 1.0;
};

inline BlockOracleResult brute_force_blocks(const std::vector<uint64_t>& grid, uint32_t nq,
                                            uint32_t nk, uint32_t y) {
  if (grid.size() != size_t(nq) * nk)
    throw contract_error("summed grid size does not match its dimensions");
  BlockOracleResult r;
  r.q_assignment.resize(nq);
  r.kv_assignment.resize(nk);
  detail::check(dbsp_brute_force_blocks(grid.data(), nq, nk, y, r.q_assignment.data(),
                                        r.kv_assignment.data(), &r.rho));
  return r;
}

}  // namespace dbsp
