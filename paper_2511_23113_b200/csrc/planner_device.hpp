// GPU inputs of the U x R selector: the integers
// select() needs from the masks, computed from device-resident mask words.
//   - MaskStats: per-head counts and Q/KV marginals of the head-summed grid
//     (planner.hpp:47-61,160-167), by K1;
//   - workload tables b_{i,g} (metrics.hpp:133-168) for a batch of
//     (strategy, plan) jobs, by one popcount kernel.
// Both are exact integers, so select_batched over them returns the host
// select()'s plan and doubles bit for bit.
#pragma once

#include <vector>

#include "core.hpp"

namespace dbsp_device_planner {

// Synchronous on `stream` (the integers are read back).
dbsp_core::MaskStats mask_stats(const uint64_t* d_words, uint32_t H, uint32_t nq, uint32_t nk,
                                void* stream);

// One table per job; y=1 jobs come from st.head_counts on the host.
std::vector<dbsp_core::Table> workload_tables(const uint64_t* d_words, const dbsp_core::MaskView& dims,
                                              const dbsp_core::MaskStats& st,
                                              const std::vector<dbsp_core::TableJob>& jobs, void* stream);

}  // namespace dbsp_device_planner
