// Host builder of the attention work list (see schedule.hpp).
#include "schedule.hpp"

#include <algorithm>
#include <bit>
#include <numeric>

namespace dbsp_core {

uint32_t normalize_sched_flags(uint32_t flags) {
  if (flags & ~kSchedKnown) fail(kConfig, "unknown schedule flag bits");
  if (flags & kSchedCtaPair) flags |= kSchedPairQ | kSchedQuad | kSchedKey128;
  else if (flags & (kSchedQuad | kSchedKey128))
    fail(kConfig, "quad / 128-key layouts run only the CTA-pair kernel: pass DBSP_SCHED_CTA_PAIR");
  if ((flags & kSchedAutoD128) && (flags & kSchedCtaPair))
    fail(kConfig, "DBSP_SCHED_AUTO_D128 chooses the layout itself; do not combine it with CTA_PAIR");
  if (flags & kSchedAutoD128) flags = (flags & ~kSchedAutoD128) | kSchedPairQ;  // see schedule.hpp
  return flags;
}

void build_schedule(const MaskView& m, const LocalView& v, uint32_t flags, Schedule& out) {
  flags = normalize_sched_flags(flags);
  const bool pair_q = (flags & kSchedPairQ) != 0;
  const uint32_t head_group = lpt_head_group(flags, v.heads, v.kv_blocks);  // 0 = global LPT
  if (v.heads == 0 || v.q_blocks == 0 || v.kv_blocks == 0)
    fail(kConfig, "local view dimensions must be positive");
  if (v.kv_blocks > kEntryKvMask) fail(kConfig, "too many local KV blocks");
  auto gh = [&](uint32_t i) { return v.head_ids ? v.head_ids[i] : i; };
  auto gq = [&](uint32_t i) { return v.q_ids ? v.q_ids[i] : i; };
  auto gk = [&](uint32_t i) { return v.kv_ids ? v.kv_ids[i] : i; };
  for (uint32_t i = 0; i < v.heads; ++i)
    if (gh(i) >= m.H) fail(kContract, "local head maps past the mask set");
  for (uint32_t i = 0; i < v.q_blocks; ++i)
    if (gq(i) >= m.nq) fail(kContract, "local Q block maps past the mask grid");

  // Global KV block -> local index, and the set of locally present blocks.
  const size_t wpr = m.wpr;
  std::vector<uint32_t> local_of(m.nk, UINT32_MAX);
  std::vector<uint64_t> present(wpr, 0);
  for (uint32_t i = 0; i < v.kv_blocks; ++i) {
    const uint32_t k = gk(i);
    if (k >= m.nk) fail(kContract, "local KV block maps past the mask grid");
    if (local_of[k] != UINT32_MAX) fail(kContract, "KV block listed twice in the local view");
    local_of[k] = i;
    present[k / 64] |= 1ull << (k % 64);
  }
  auto valid_keys = [&](uint32_t k) -> uint32_t {
    if (v.kv_tokens_global == 0) return 64;
    const uint64_t start = uint64_t(k) * 64;
    if (start >= v.kv_tokens_global) return 1;  // fully padded block: keep one key slot
    return uint32_t(std::min<uint64_t>(64, v.kv_tokens_global - start));
  };

  struct Raw {
    WorkItem it;
    std::vector<uint32_t> e;
  };
  std::vector<Raw> raw;
  raw.reserve(size_t(v.heads) * ((v.q_blocks + 1) / 2));
  out.tile_visits = 0;
  out.dense_tiles = 0;
  const bool quad = (flags & kSchedQuad) != 0;
  const uint32_t step = quad ? 4 : pair_q ? 2 : 1;
  std::vector<uint64_t> uni(wpr);
  for (uint32_t hl = 0; hl < v.heads && quad; ++hl) {
    // Four Q blocks per item (two 128-row tiles of a CTA pair), one KV list:
    // the union of the four rows; entry bit 22+i marks row i dense.
    const uint32_t h = gh(hl);
    for (uint32_t a = 0; a < v.q_blocks; a += 4) {
      uint32_t q[4];
      const uint64_t* rows[4];
      uint32_t pad = 0;
      for (uint32_t i = 0; i < 4; ++i) {
        const bool in = a + i < v.q_blocks;
        q[i] = in ? a + i : a;
        rows[i] = in ? m.row(h, gq(q[i])) : nullptr;
        pad |= in ? 0u : (1u << i);
      }
      Raw r;
      r.it = WorkItem{hl, q[0], q[1], 0, 0, pad, q[2], q[3]};
      for (size_t w = 0; w < wpr; ++w) {
        uint64_t x = 0;
        for (int i = 0; i < 4; ++i) x |= rows[i] ? rows[i][w] : 0ull;
        uni[w] = x & present[w];
      }
      for (size_t w = 0; w < wpr; ++w)
        for (uint64_t word = uni[w]; word; word &= word - 1) {
          const uint32_t k = uint32_t(w * 64 + std::countr_zero(word));
          const uint64_t bit = 1ull << (k % 64);
          uint32_t e = local_of[k] | ((valid_keys(k) - 1) << kQuadValidShift);
          for (uint32_t i = 0; i < 4; ++i)
            if (rows[i] && (rows[i][w] & bit)) {
              e |= 1u << (22 + i);
              ++out.dense_tiles;
            }
          r.e.push_back(e);
        }
      r.it.count = uint32_t(r.e.size());
      out.tile_visits += r.it.count;
      raw.push_back(std::move(r));
    }
  }
  for (uint32_t hl = 0; hl < v.heads && !quad; ++hl) {
    const uint32_t h = gh(hl);
    for (uint32_t a = 0; a < v.q_blocks; a += step) {
      const bool single = !pair_q || a + 1 >= v.q_blocks;
      const uint32_t b = single ? a : a + 1;
      const uint64_t* ra = m.row(h, gq(a));
      const uint64_t* rb = single ? nullptr : m.row(h, gq(b));
      Raw r;
      r.it = WorkItem{hl, a, b, 0, 0, single ? 1u : 0u, 0, 0};
      for (size_t w = 0; w < wpr; ++w) uni[w] = (ra[w] | (rb ? rb[w] : 0)) & present[w];
      for (size_t w = 0; w < wpr; ++w)
        for (uint64_t word = uni[w]; word; word &= word - 1) {
          const uint32_t k = uint32_t(w * 64 + std::countr_zero(word));
          const uint64_t bit = 1ull << (k % 64);
          const bool da = (ra[w] & bit) != 0;
          const bool db = rb && (rb[w] & bit) != 0;
          r.e.push_back(local_of[k] | (da ? kEntryDenseA : 0u) | (db ? kEntryDenseB : 0u) |
                        ((valid_keys(k) - 1) << kEntryValidShift));
          out.dense_tiles += uint64_t(da) + uint64_t(db);
        }
      r.it.count = uint32_t(r.e.size());
      out.tile_visits += r.it.count;
      raw.push_back(std::move(r));
    }
  }
  std::vector<uint32_t> order(raw.size());
  std::iota(order.begin(), order.end(), 0u);
  // Heaviest-first (LPT) launch order.  The hardware hands CTAs to free SM
  // slots in blockIdx order, so this is a dynamic LPT schedule, within head
  // groups whose K/V fits the L2 (schedule.hpp lpt_head_group).
  std::stable_sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) {
    if (head_group) {
      const uint32_t gx = raw[x].it.head / head_group, gy = raw[y].it.head / head_group;
      if (gx != gy) return gx < gy;
    }
    return raw[x].it.count > raw[y].it.count;
  });
  out.items.clear();
  out.entries.clear();
  out.flags = flags;
  out.max_head = v.heads - 1;
  out.max_q_block = v.q_blocks - 1;
  out.max_kv_block = v.kv_blocks - 1;
  out.items.reserve(raw.size());
  out.entries.reserve(out.tile_visits);
  for (uint32_t i : order) {
    WorkItem it = raw[i].it;
    it.begin = uint32_t(out.entries.size());
    out.entries.insert(out.entries.end(), raw[i].e.begin(), raw[i].e.end());
    out.items.push_back(it);
  }
}

}  // namespace dbsp_core
