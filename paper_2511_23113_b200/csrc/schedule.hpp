// Work schedule of the block-sparse attention kernel.
//
// One work item = one local head x one 128-row Q tile (two 64-row Q blocks of
// the same head, or one block padded to 128 rows).  Its entries are the KV
// blocks in the union of the two rows' dense sets, each tagged with which
// half actually needs it.  tcgen05 runs M=128 tiles at the same issue cost as
// M=64 (B300_MICROARCH.md: floor = max(M,128)*N/256 cycles), so pairing two
// 64-row Q blocks is never slower than one M=64 tile per block and is twice
// as fast when their KV sets coincide.
#pragma once

#include <cstdint>
#include <vector>

#include "core.hpp"

namespace dbsp_core {

// Device layout: 32 bytes, read once per CTA.
struct alignas(16) WorkItem {
  uint32_t head;    // local head index in the Q/K/V buffers
  uint32_t qa;      // local Q block of rows 0..63
  uint32_t qb;      // local Q block of rows 64..127 (== qa when single)
  uint32_t begin;   // first entry
  uint32_t count;   // entries (KV tiles visited)
  uint32_t single;  // 1: rows 64..127 are padding
  uint32_t pad0, pad1;
};

// Entry bit layout.
constexpr uint32_t kEntryKvMask = (1u << 22) - 1;  // local KV block index
constexpr uint32_t kEntryDenseA = 1u << 22;        // tile dense for rows 0..63
constexpr uint32_t kEntryDenseB = 1u << 23;        // tile dense for rows 64..127
constexpr uint32_t kEntryValidShift = 24;          // (valid keys - 1), 6 bits

struct LocalView {
  uint32_t heads = 0, q_blocks = 0, kv_blocks = 0;
  const uint32_t* head_ids = nullptr;  // null = identity
  const uint32_t* q_ids = nullptr;
  const uint32_t* kv_ids = nullptr;
  uint32_t kv_tokens_global = 0;  // 0 = every block full
};

struct Schedule {
  std::vector<WorkItem> items;
  std::vector<uint32_t> entries;
  uint64_t tile_visits = 0;  // sum of counts (MMA tiles issued)
  uint64_t dense_tiles = 0;  // 64x64 tiles actually dense (softmax work)
  uint32_t max_head = 0, max_q_block = 0, max_kv_block = 0;  // bounds checked at launch
  uint32_t flags = 0;  // build flags (kSchedQuad selects a two-stage kernel)
};

// Schedule flags (dbsp_schedule_build's `flags`).
constexpr uint32_t kSchedPairQ = 1;      // two Q blocks per 128-row tile
constexpr uint32_t kSchedGlobalLpt = 2;  // heaviest items first across all heads
constexpr uint32_t kSchedHeadOrder = 4;  // heaviest first within each head, heads in order
// Neither bit set: heads in groups of max(1, kLptGroupKvBlocks / local KV
// blocks) -- a group's K/V (at d=128: 2048 blocks x 64 keys x 128 x 2 B x
// (K, V) = 64 MB) fits the 126 MB L2 -- heaviest-first within each group,
// groups in head order.  Measured on one B200 (tests/ab_probe.py --sustained,
// 30 back-to-back launches per variant; tests/variant_cycles.py for DRAM):
//   CogVideoX (48 heads x 278 blocks, groups of 7): 1.72 ms vs 1.76 global
//     LPT (1.94 GB DRAM per launch) vs 1.91 per-head (0.42 GB); 0.42 GB;
//   Wan (40 x 512, groups of 4): 6.006 vs 6.004 ms per-head vs 6.42 global
//     (6.4 GB DRAM: power-capped, it costs clock);
//   HunyuanVideo (24 x 1857): groups of 1 = per-head.
// Global order starts every head's heaviest items first; a group keeps that
// across the group's heads while its K/V stays in L2.
constexpr uint32_t kLptGroupKvBlocks = 2048;
// Small views (a few waves of CTAs, e.g. one SP rank's share) stay one group:
// a last head group would otherwise run as a serial tail (the G=8 Wan
// per-rank kernels -- 5 heads x 512 blocks -- measured 1.26x instead of 1.41x
// db-SP over uniform when split into groups of 4 + 1).
constexpr uint64_t kLptGroupMinHeadBlocks = 4096;
// Heads per ordering group for a local view (0 = one group: global LPT).
inline uint32_t lpt_head_group(uint32_t flags, uint32_t heads, uint32_t kv_blocks) {
  if (flags & kSchedGlobalLpt) return 0;
  if (flags & kSchedHeadOrder) return 1;
  if (uint64_t(heads) * kv_blocks <= kLptGroupMinHeadBlocks) return 0;
  const uint32_t g = kLptGroupKvBlocks / (kv_blocks ? kv_blocks : 1u);
  return g >= heads ? 0u : (g ? g : 1u);
}
constexpr uint32_t kSchedQuad = 8;       // layout: four Q blocks per item
constexpr uint32_t kSchedKey128 = 16;    // layout: 128-key steps
constexpr uint32_t kSchedCtaPair = 128;  // d=128 CTA-pair kernel (attn_kernel_pd3.cuh); implies 1|8|16
// For head_dim 128: the automatic layout choice.  Round 1 picked the CTA-pair
// quad schedule where its dense fraction stayed within 0.95x of the pair
// schedule's (then 4-8% faster there).  Since the one-CTA kernel issues its
// MMAs warp-uniformly (round 2) it takes fewer cycles than the CTA-pair kernel
// on every measured mask family -- Wan 8.20 M vs 8.89 M, HunyuanVideo 60.1 M
// vs 62.2 M cycles per launch (profiles/r02_kernel_choice.md) -- and the quad
// union can only be sparser than the pair union, so AUTO now resolves to the
// pair layout.  The CTA-pair kernel stays available through kSchedCtaPair.
constexpr uint32_t kSchedAutoD128 = 256;
constexpr uint32_t kSchedKnown = kSchedPairQ | kSchedGlobalLpt | kSchedHeadOrder | kSchedQuad | kSchedKey128 |
                                 kSchedCtaPair | kSchedAutoD128;
// Flags as built: CTA_PAIR implies the quad layout bits; QUAD / KEY128 alone
// (the retired two-stage one-CTA kernels) and unknown bits are config errors.
uint32_t normalize_sched_flags(uint32_t flags);
// Quad items: WorkItem{head, q0, q1, begin, count, pad_mask, q2, q3}; entries
// carry one dense bit per row at 22..25 and (valid keys - 1) at 26..31.
constexpr uint32_t kQuadValidShift = 26;

// Builds the work items in LPT launch order (see schedule.cpp).
void build_schedule(const MaskView& m, const LocalView& v, uint32_t flags, Schedule& out);

}  // namespace dbsp_core
