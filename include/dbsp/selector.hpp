// Per-call U x R strategy selector — drop-in counterpart of the reference's
// proj/include/dbsp/selector.hpp (SelectorState :18-43, Selection :45-49,
// select :55-75).  The state lives in libdbsp_b200.so (internally locked),
// so C, Python and C++ callers can share one per process.
#pragma once

#include <cstdint>
#include <optional>
#include <utility>
#include <vector>

#include "../dbsp_b200.h"
#include "error.hpp"
#include "latency.hpp"
#include "metrics.hpp"
#include "planner.hpp"

namespace dbsp {

class SelectorState {
 public:
  explicit SelectorState(uint32_t total_gpus) : total_gpus_(total_gpus) {
    detail::check(dbsp_selector_create(total_gpus, &h_));
    prebuilt_ = enumerate_strategies(total_gpus);
  }
  ~SelectorState() { dbsp_selector_destroy(h_); }
  SelectorState(const SelectorState&) = delete;
  SelectorState& operator=(const SelectorState&) = delete;

  uint32_t total_gpus() const { return total_gpus_; }
  const std::vector<ParallelStrategy>& prebuilt_groups() const { return prebuilt_; }

  std::optional<std::pair<ParallelStrategy, PartitionPlan>> stored(int64_t layer) const {
    int32_t found = 0;
    dbsp_strategy s{};
    uint32_t sizes[3] = {0, 0, 0};
    detail::check(dbsp_selector_stored(h_, layer, &found, &s, sizes, nullptr));
    if (!found) return std::nullopt;
    PartitionPlan p;
    p.head_assignment.resize(sizes[0]);
    p.q_assignment.resize(sizes[1]);
    p.kv_assignment.resize(sizes[2]);
    dbsp_plan c = detail::cplan(p);
    detail::check(dbsp_selector_stored(h_, layer, &found, &s, sizes, &c));
    return std::make_pair(ParallelStrategy{s.ulysses, s.ring}, std::move(p));
  }

  void store(int64_t layer, ParallelStrategy strategy, PartitionPlan plan) {
    const uint32_t sizes[3] = {uint32_t(plan.head_assignment.size()),
                               uint32_t(plan.q_assignment.size()),
                               uint32_t(plan.kv_assignment.size())};
    const dbsp_plan c = detail::cplan(plan);
    detail::check(dbsp_selector_store(h_, layer, detail::cs(strategy), &c, sizes));
  }

  dbsp_selector* handle() const { return h_; }

 private:
  uint32_t total_gpus_;
  dbsp_selector* h_ = nullptr;
  std::vector<ParallelStrategy> prebuilt_;
};

struct Selection {
  ParallelStrategy strategy;
  PlanOutcome outcome;
  LatencyBreakdown latency;
};

inline Selection select(int64_t layer_id, const AttentionMaskSet& set,
                        const MachineProfile& profile, const PlannerConfig& config,
                        SelectorState& state) {
  detail::MaskView v(set);
  detail::ProfileView pv(profile);
  Selection out;
  out.outcome.plan = detail::sized_plan(set);
  dbsp_plan c = detail::cplan(out.outcome.plan);
  const dbsp_planner_config cfg{config.reuse_threshold, config.exchange_reward};
  dbsp_strategy s{};
  dbsp_plan_outcome oc{};
  dbsp_latency lat{};
  detail::check(dbsp_select(state.handle(), layer_id, v.get(), pv.get(), &cfg, &s, &c, &oc, &lat));
  out.strategy = {s.ulysses, s.ring};
  out.outcome.head_replanned = oc.head_replanned != 0;
  out.outcome.rho_pre = oc.rho_pre;
  out.outcome.rho_post = oc.rho_post;
  out.latency = detail::from_c(lat);
  return out;
}

// select() from device-resident mask words (u64 [H][Nq][ceil(Nk/64)], the
// BlockMask row layout): the mask integers are computed on the GPU, the
// result equals select() on the same masks bit for bit (dbsp_select_device).
inline Selection select_device(int64_t layer_id, const uint64_t* d_words, uint32_t heads, uint32_t q_blocks,
                               uint32_t kv_blocks, uint32_t block_size, const MachineProfile& profile,
                               const PlannerConfig& config, SelectorState& state, void* stream = nullptr) {
  detail::ProfileView pv(profile);
  Selection out;
  out.outcome.plan.head_assignment.assign(heads, 0);
  out.outcome.plan.q_assignment.assign(q_blocks, 0);
  out.outcome.plan.kv_assignment.assign(kv_blocks, 0);
  dbsp_plan c = detail::cplan(out.outcome.plan);
  const dbsp_planner_config cfg{config.reuse_threshold, config.exchange_reward};
  dbsp_strategy s{};
  dbsp_plan_outcome oc{};
  dbsp_latency lat{};
  detail::check(dbsp_select_device(state.handle(), layer_id, d_words, heads, q_blocks, kv_blocks, block_size,
                                   pv.get(), &cfg, &s, &c, &oc, &lat, stream));
  out.strategy = {s.ulysses, s.ring};
  out.outcome.head_replanned = oc.head_replanned != 0;
  out.outcome.rho_pre = oc.rho_pre;
  out.outcome.rho_post = oc.rho_post;
  out.latency = detail::from_c(lat);
  return out;
}

}  // namespace dbsp
