// Host implementation of the db-SP planner: mask model, rho_s metrics,
// dual-balanced partitioner, Eq.4 latency model and U x R selector.
// Reference semantics are cited per function (paths under the reference
// proj/include/dbsp/).  See core.hpp for the bit-exactness contract.
#include "core.hpp"

#include <algorithm>
#include <bit>
#include <cmath>
#include <exception>
#include <limits>
#include <numeric>
#include <thread>
#include <utility>

namespace dbsp_core {

namespace {

std::string str(uint64_t v) { return std::to_string(v); }

// Splits [0, n) into contiguous chunks over up to `threads` std::threads; the
// body gets (chunk index, begin, end).  Integer partial results are merged by
// the caller in chunk order, so results never depend on the thread count.
template <class F>
void parallel_chunks(size_t n, size_t threads, F&& body) {
  threads = std::max<size_t>(1, std::min(threads, n));
  if (threads == 1) {
    body(size_t(0), size_t(0), n);
    return;
  }
  std::vector<std::thread> pool;
  for (size_t t = 1; t < threads; ++t)
    pool.emplace_back([&, t] { body(t, n * t / threads, n * (t + 1) / threads); });
  body(size_t(0), size_t(0), n / threads);
  for (std::thread& th : pool) th.join();
}

size_t planner_threads(uint64_t work_words) {
  if (work_words < (uint64_t(1) << 16)) return 1;  // small sets: threads cost more than they save
  const unsigned hw = std::thread::hardware_concurrency();
  return std::min<size_t>(hw ? hw : 1, 8);
}

}  // namespace

MaskView make_view(const uint64_t* const* heads, uint32_t H, uint32_t nq, uint32_t nk,
                   uint32_t block_size) {
  // AttentionMaskSet / BlockMask constructor checks (mask.hpp:24-31, 85-94).
  if (nq == 0 || nk == 0) fail(kConfig, "BlockMask dimensions must be positive");
  if (H == 0) fail(kConfig, "mask set needs at least one head");
  if (block_size == 0) fail(kConfig, "block_size must be positive");
  if (!heads) fail(kContract, "mask set has no head pointers");
  for (uint32_t h = 0; h < H; ++h)
    if (!heads[h]) fail(kContract, "mask head " + str(h) + " is null");
  MaskView v;
  v.heads = heads;
  v.H = H;
  v.nq = nq;
  v.nk = nk;
  v.block_size = block_size;
  v.wpr = (size_t(nk) + 63) / 64;
  return v;
}

// ---------------------------------------------------------------------------
// mask.hpp

uint64_t popcount_words(const uint64_t* w, size_t n) {
  uint64_t c = 0;
  for (size_t i = 0; i < n; ++i) c += uint64_t(std::popcount(w[i]));
  return c;
}

std::vector<uint64_t> head_counts(const MaskView& m) {
  std::vector<uint64_t> out(m.H);
  const size_t n = size_t(m.nq) * m.wpr;
  for (uint32_t h = 0; h < m.H; ++h) out[h] = popcount_words(m.heads[h], n);
  return out;
}

uint64_t total_blocks(const MaskView& m) {
  uint64_t t = 0;
  for (uint64_t c : head_counts(m)) t += c;
  return t;
}

// mask.hpp:282-284: total / (H * Nq * Nk) in double.
double density(const MaskView& m) {
  return static_cast<double>(total_blocks(m)) / static_cast<double>(m.cells());
}

// Strategy-independent integers of one mask set.  Column weights use a
// bit-sliced vertical counter per word position (carry-save increments), so
// the cost is O(rows * words) instead of a walk over every set bit.
MaskStats mask_stats(const MaskView& m, bool marginals) {
  MaskStats st;
  st.head_counts = head_counts(m);
  for (uint64_t c : st.head_counts) st.total += c;
  if (!marginals) return st;
  st.have_marginals = true;
  st.row_weights.assign(m.nq, 0);
  st.col_weights.assign(m.nk, 0);
  const size_t wpr = m.wpr;
  const size_t T = planner_threads(uint64_t(m.H) * m.nq * wpr);
  std::vector<std::vector<uint64_t>> rows_part(T, std::vector<uint64_t>(m.nq, 0));
  std::vector<std::vector<uint64_t>> cols_part(T, std::vector<uint64_t>(m.nk, 0));
  parallel_chunks(m.H, T, [&](size_t t, size_t h0, size_t h1) {
    const uint64_t rows = uint64_t(h1 - h0) * m.nq;
    const int planes = std::max(1, int(std::bit_width(rows)));
    std::vector<uint64_t> plane(size_t(planes) * wpr, 0);
    std::vector<uint64_t>& rw = rows_part[t];
    for (size_t h = h0; h < h1; ++h) {
      for (uint32_t q = 0; q < m.nq; ++q) {
        const uint64_t* r = m.row(uint32_t(h), q);
        uint64_t rc = 0;
        for (size_t w = 0; w < wpr; ++w) {
          const uint64_t word = r[w];
          rc += uint64_t(std::popcount(word));
          uint64_t carry = word;  // bit-sliced vertical counter, carry-save increment
          for (int p = 0; carry; ++p) {
            uint64_t& cell = plane[size_t(p) * wpr + w];
            const uint64_t c = cell & carry;
            cell ^= carry;
            carry = c;
          }
        }
        rw[q] += rc;
      }
    }
    std::vector<uint64_t>& cw = cols_part[t];
    for (uint32_t k = 0; k < m.nk; ++k) {
      const size_t w = k / 64;
      const unsigned b = k % 64;
      uint64_t v = 0;
      for (int p = 0; p < planes; ++p) v |= ((plane[size_t(p) * wpr + w] >> b) & 1ull) << p;
      cw[k] = v;
    }
  });
  for (size_t t = 0; t < T; ++t) {
    for (uint32_t q = 0; q < m.nq; ++q) st.row_weights[q] += rows_part[t][q];
    for (uint32_t k = 0; k < m.nk; ++k) st.col_weights[k] += cols_part[t][k];
  }
  return st;
}

namespace {

inline void set_bit(uint64_t* rows, size_t wpr, uint32_t q, uint32_t k) {
  rows[size_t(q) * wpr + k / 64] |= 1ull << (k % 64);
}
inline bool get_bit(const uint64_t* rows, size_t wpr, uint32_t q, uint32_t k) {
  return (rows[size_t(q) * wpr + k / 64] >> (k % 64)) & 1ull;
}

// mask.hpp:166-172: one Bernoulli draw per cell in row-major order.
void gen_uniform(uint64_t* rows, size_t wpr, uint32_t nq, uint32_t nk, double p, SplitMix& rng) {
  for (uint32_t q = 0; q < nq; ++q)
    for (uint32_t k = 0; k < nk; ++k)
      if (rng.coin(p)) set_bit(rows, wpr, q, k);
}

// mask.hpp:176-195: the `target` cells closest to the q = k*Nq/Nk diagonal,
// ordered by (distance, linear index).  The order is total, so selecting the
// first `target` with nth_element gives exactly the reference's set.
void gen_banded(uint64_t* rows, size_t wpr, uint32_t nq, uint32_t nk, double p) {
  const uint64_t cells = uint64_t(nq) * nk;
  const uint64_t target = static_cast<uint64_t>(std::llround(p * static_cast<double>(cells)));
  if (target == 0) return;
  std::vector<std::pair<double, uint64_t>> key;
  key.reserve(cells);
  for (uint32_t q = 0; q < nq; ++q)
    for (uint32_t k = 0; k < nk; ++k) {
      const double diag = static_cast<double>(k) * nq / nk;
      key.emplace_back(std::abs(static_cast<double>(q) - diag), uint64_t(q) * nk + k);
    }
  if (target < cells) std::nth_element(key.begin(), key.begin() + target, key.end());
  for (uint64_t i = 0; i < std::min(target, cells); ++i) {
    const uint64_t c = key[i].second;
    set_bit(rows, wpr, uint32_t(c / nk), uint32_t(c % nk));
  }
}

// mask.hpp:200-228: random rectangles (h, w, q0, k0 drawn in that order),
// clipped in row-major order at the target; 256 rectangles in a row adding
// nothing end the loop and a row-major scan fills the remainder.
void gen_clustered(uint64_t* rows, size_t wpr, uint32_t nq, uint32_t nk, double p,
                   SplitMix& rng) {
  const uint64_t cells = uint64_t(nq) * nk;
  const uint64_t target = static_cast<uint64_t>(std::llround(p * static_cast<double>(cells)));
  uint64_t have = 0;
  int idle = 0;
  while (have < target && idle < 256) {
    const uint32_t rh = 1 + uint32_t(rng.below(std::max(1u, nq / 4)));
    const uint32_t rw = 1 + uint32_t(rng.below(std::max(1u, nk / 4)));
    const uint32_t q0 = uint32_t(rng.below(nq - rh + 1));
    const uint32_t k0 = uint32_t(rng.below(nk - rw + 1));
    uint64_t fresh = 0;
    for (uint32_t q = q0; q < q0 + rh && have < target; ++q)
      for (uint32_t k = k0; k < k0 + rw && have < target; ++k)
        if (!get_bit(rows, wpr, q, k)) {
          set_bit(rows, wpr, q, k);
          ++have;
          ++fresh;
        }
    idle = fresh ? 0 : idle + 1;
  }
  for (uint32_t q = 0; q < nq && have < target; ++q)
    for (uint32_t k = 0; k < nk && have < target; ++k)
      if (!get_bit(rows, wpr, q, k)) {
        set_bit(rows, wpr, q, k);
        ++have;
      }
}

}  // namespace

// mask.hpp:137-162 (validation, density ramp) and 233-256 (per-head substreams).
void generate_masks(const GenSpec& sp, uint64_t* out) {
  if (sp.H == 0 || sp.nq == 0 || sp.nk == 0 || sp.block_size == 0)
    fail(kConfig, "generator dimensions must be positive");
  if (!(sp.dmin >= 0.0) || !(sp.dmax <= 1.0) || !(sp.dmin <= sp.dmax))
    fail(kConfig, "density law requires 0 <= min_density <= max_density <= 1");
  if (!(sp.skew > 0.0)) fail(kConfig, "skew exponent must be > 0");
  if (sp.pattern > 2) fail(kConfig, "unknown mask pattern " + str(sp.pattern));
  const size_t wpr = (size_t(sp.nk) + 63) / 64;
  const size_t per_head = size_t(sp.nq) * wpr;
  std::fill(out, out + per_head * sp.H, 0ull);
  for (uint32_t h = 0; h < sp.H; ++h) {
    const double t =
        sp.H > 1 ? std::pow(static_cast<double>(h) / (sp.H - 1), sp.skew) : 0.0;
    const double p = sp.dmin + (sp.dmax - sp.dmin) * t;
    SplitMix rng(mix_seed(sp.seed, h, 0));
    uint64_t* rows = out + per_head * h;
    switch (sp.pattern) {
      case 0: gen_uniform(rows, wpr, sp.nq, sp.nk, p, rng); break;
      case 1: gen_banded(rows, wpr, sp.nq, sp.nk, p); break;
      default: gen_clustered(rows, wpr, sp.nq, sp.nk, p, rng); break;
    }
  }
}

// mask.hpp:260-273.
void perturb_masks(const MaskView& m, double flip_rate, uint64_t seed, uint64_t* out) {
  if (!(flip_rate >= 0.0) || !(flip_rate <= 1.0)) fail(kConfig, "flip_rate must be in [0, 1]");
  const size_t per_head = size_t(m.nq) * m.wpr;
  for (uint32_t h = 0; h < m.H; ++h)
    if (out + per_head * h != m.heads[h])
      std::copy(m.heads[h], m.heads[h] + per_head, out + per_head * h);
  if (flip_rate == 0.0) return;
  for (uint32_t h = 0; h < m.H; ++h) {
    SplitMix rng(mix_seed(seed, h, 0));
    uint64_t* rows = out + per_head * h;
    for (uint32_t q = 0; q < m.nq; ++q)
      for (uint32_t k = 0; k < m.nk; ++k)
        if (rng.coin(flip_rate)) rows[size_t(q) * m.wpr + k / 64] ^= 1ull << (k % 64);
  }
}

// ---------------------------------------------------------------------------
// metrics.hpp

// metrics.hpp:56-66.
std::vector<Strategy> enumerate_strategies(uint32_t gpus) {
  if (gpus < 1 || !std::has_single_bit(gpus))
    fail(kConfig, "GPU count must be a power of two >= 1, got " + str(gpus));
  std::vector<Strategy> out;
  for (uint32_t x = gpus;; x /= 2) {
    out.push_back({x, gpus / x});
    if (x == 1) break;
  }
  return out;
}

// metrics.hpp:78-90.
void validate_plan(const MaskView& m, Strategy s, const uint32_t* head, const uint32_t* q,
                   const uint32_t* kv) {
  if (!head || !q || !kv) fail(kContract, "plan dimensions do not match the mask set");
  for (uint32_t i = 0; i < m.H; ++i)
    if (head[i] >= s.x) fail(kContract, "head assigned past the Ulysses degree");
  for (uint32_t i = 0; i < m.nq; ++i)
    if (q[i] >= s.y) fail(kContract, "Q block assigned past the ring degree");
  for (uint32_t i = 0; i < m.nk; ++i)
    if (kv[i] >= s.y) fail(kContract, "KV block assigned past the ring degree");
}

// metrics.hpp:94-113: contiguous floor(i * degree / n).
Plan default_plan(const MaskView& m, Strategy s) {
  if (s.x < 1 || s.y < 1) fail(kConfig, "parallel degrees must be >= 1");
  if (s.x > m.H)
    fail(kConfig, "Ulysses degree " + str(s.x) + " exceeds head count " + str(m.H));
  auto split = [](uint64_t n, uint64_t deg) {
    std::vector<uint32_t> a(n);
    for (uint64_t i = 0; i < n; ++i) a[i] = uint32_t(i * deg / n);
    return a;
  };
  return Plan{split(m.H, s.x), split(m.nq, s.y), split(m.nk, s.y)};
}

// metrics.hpp:133-168.  Ring rank r processes KV group (r + i) mod y in
// period i, so a dense block of group g lands in period (g - r) mod y on GPU
// u*y + r.
Table workload_table(const MaskView& m, Strategy s, const uint32_t* head, const uint32_t* q,
                     const uint32_t* kv, const MaskStats* st) {
  validate_plan(m, s, head, q, kv);
  const uint32_t x = s.x, y = s.y;
  Table t;
  t.gpus = x * y;
  if (y == 1) {
    t.periods = 1;
    t.counts.assign(t.gpus, 0);
    const std::vector<uint64_t> local = st ? std::vector<uint64_t>() : head_counts(m);
    const std::vector<uint64_t>& hc = st ? st->head_counts : local;
    for (uint32_t h = 0; h < m.H; ++h) t.counts[head[h]] += hc[h];
    return t;
  }
  t.periods = y;
  t.counts.assign(size_t(y) * t.gpus, 0);
  const size_t wpr = m.wpr;
  std::vector<uint64_t> group(size_t(y) * wpr, 0);
  for (uint32_t k = 0; k < m.nk; ++k) group[size_t(kv[k]) * wpr + k / 64] |= 1ull << (k % 64);
  const size_t T = planner_threads(uint64_t(m.H) * m.nq * wpr * y / 4);
  std::vector<std::vector<uint64_t>> part(T, std::vector<uint64_t>(t.counts.size(), 0));
  parallel_chunks(m.H, T, [&](size_t ti, size_t h0, size_t h1) {
    std::vector<uint64_t>& cnt = part[ti];
    for (size_t h = h0; h < h1; ++h) {
      const uint32_t u = head[h];
      for (uint32_t qb = 0; qb < m.nq; ++qb) {
        const uint64_t* r = m.row(uint32_t(h), qb);
        const uint32_t rr = q[qb];
        const uint32_t gpu = u * y + rr;
        for (uint32_t g = 0; g < y; ++g) {
          const uint64_t* gb = group.data() + size_t(g) * wpr;
          uint64_t c = 0;
          for (size_t w = 0; w < wpr; ++w) c += uint64_t(std::popcount(r[w] & gb[w]));
          cnt[size_t((g + y - rr) % y) * t.gpus + gpu] += c;
        }
      }
    }
  });
  for (const auto& cnt : part)
    for (size_t i = 0; i < cnt.size(); ++i) t.counts[i] += cnt[i];
  return t;
}

// metrics.hpp:173-186: sum of per-period maxima over the balanced share.
double imbalance_ratio(const uint64_t* counts, uint32_t periods, uint32_t gpus) {
  uint64_t total = 0, sum_max = 0;
  for (uint32_t p = 0; p < periods; ++p) {
    uint64_t mx = 0;
    for (uint32_t g = 0; g < gpus; ++g) {
      const uint64_t c = counts[size_t(p) * gpus + g];
      mx = std::max(mx, c);
      total += c;
    }
    sum_max += mx;
  }
  if (total == 0) return 1.0;
  return static_cast<double>(sum_max) * static_cast<double>(gpus) /
         static_cast<double>(total);
}

// metrics.hpp:198-211.
Exchange exchange_volume(const MaskView& m, Strategy s, const uint32_t* q, const uint32_t* kv) {
  Exchange e;
  const uint64_t y = s.y, nq = m.nq, nk = m.nk;
  for (uint64_t i = 0; i < nq; ++i)
    if (q[i] != uint32_t(i * y / nq)) ++e.q_moved;
  for (uint64_t i = 0; i < nk; ++i)
    if (kv[i] != uint32_t(i * y / nk)) ++e.kv_moved;
  e.payload = (e.q_moved + 2 * e.kv_moved) * m.block_size;
  return e;
}

// ---------------------------------------------------------------------------
// planner.hpp

void PlannerConfig::validate() const {
  // planner.hpp:29-34.
  if (!(reuse_threshold >= 1.0)) fail(kConfig, "reuse threshold must be >= 1");
  if (std::isnan(exchange_reward) || exchange_reward < 0.0)
    fail(kConfig, "exchange reward must be >= 0 or infinite");
}

// planner.hpp:47-61: S[q*Nk + k] = #heads with bit (q, k).
std::vector<uint64_t> summed_grid(const MaskView& m) {
  std::vector<uint64_t> g(size_t(m.nq) * m.nk, 0);
  for (uint32_t h = 0; h < m.H; ++h)
    for (uint32_t q = 0; q < m.nq; ++q) {
      const uint64_t* r = m.row(h, q);
      uint64_t* out = g.data() + size_t(q) * m.nk;
      for (size_t w = 0; w < m.wpr; ++w)
        for (uint64_t word = r[w]; word; word &= word - 1)
          ++out[w * 64 + size_t(std::countr_zero(word))];
    }
  return g;
}

// planner.hpp:65-76.
double head_level_imbalance(const uint64_t* w, const uint32_t* a, size_t n, uint32_t x) {
  std::vector<uint64_t> load(x, 0);
  uint64_t total = 0;
  for (size_t i = 0; i < n; ++i) {
    if (a[i] >= x) fail(kContract, "head assigned past the Ulysses degree");
    load[a[i]] += w[i];
    total += w[i];
  }
  if (total == 0) return 1.0;
  const uint64_t mx = *std::max_element(load.begin(), load.end());
  return static_cast<double>(mx) * x / static_cast<double>(total);
}

namespace {

// planner.hpp:82-90: descending weight, ties by ascending index.
std::vector<uint32_t> heavy_first(const uint64_t* w, size_t n) {
  std::vector<uint32_t> idx(n);
  std::iota(idx.begin(), idx.end(), 0u);
  std::stable_sort(idx.begin(), idx.end(), [w](uint32_t a, uint32_t b) { return w[a] > w[b]; });
  return idx;
}

}  // namespace

// planner.hpp:96-112 (LPT; strict < keeps ties on the lowest rank).
std::vector<uint32_t> lpt_heads(const std::vector<uint64_t>& w, uint32_t x) {
  std::vector<uint32_t> a(w.size(), 0);
  std::vector<uint64_t> load(x, 0);
  for (uint32_t h : heavy_first(w.data(), w.size())) {
    uint32_t best = 0;
    for (uint32_t r = 1; r < x; ++r)
      if (load[r] < load[best]) best = r;
    a[h] = best;
    load[best] += w[h];
  }
  return a;
}

std::vector<uint32_t> partition_heads(const MaskView& m, uint32_t x, const MaskStats* st) {
  if (x < 1 || x > m.H)
    fail(kConfig, "Ulysses degree " + str(x) + " must be in [1, " + str(m.H) + "]");
  return st ? lpt_heads(st->head_counts, x) : lpt_heads(head_counts(m), x);
}

// planner.hpp:119-145.  The home-rank bias only steers the choice; loads
// grow by the unbiased weight.
std::vector<uint32_t> biased_greedy(const uint64_t* w, size_t n, uint32_t y, double reward) {
  std::vector<uint32_t> a(n, 0);
  if (std::isinf(reward)) {
    for (size_t i = 0; i < n; ++i) a[i] = uint32_t(i * y / n);
    return a;
  }
  std::vector<uint64_t> load(y, 0);
  for (uint32_t i : heavy_first(w, n)) {
    const uint32_t home = uint32_t(uint64_t(i) * y / n);
    const double bias = reward * static_cast<double>(w[i]);
    uint32_t best = 0;
    double best_load = static_cast<double>(load[0]) - (home == 0 ? bias : 0.0);
    for (uint32_t r = 1; r < y; ++r) {
      const double l = static_cast<double>(load[r]) - (home == r ? bias : 0.0);
      if (l < best_load) {
        best = r;
        best_load = l;
      }
    }
    a[i] = best;
    load[best] += w[i];
  }
  return a;
}

// planner.hpp:151-170: Q rows / KV columns of the head-summed grid.
void partition_blocks(const MaskView& m, uint32_t y, double reward, const MaskStats* st,
                      std::vector<uint32_t>& q_out, std::vector<uint32_t>& kv_out) {
  const uint32_t lim = std::min(m.nq, m.nk);
  if (y < 1 || y > lim)
    fail(kConfig, "ring degree " + str(y) + " must be in [1, " + str(lim) + "]");
  if (std::isnan(reward) || reward < 0.0)
    fail(kConfig, "exchange reward must be >= 0 or infinite");
  MaskStats local;
  if (!st || !st->have_marginals) {
    local = mask_stats(m, true);
    st = &local;
  }
  q_out = biased_greedy(st->row_weights.data(), m.nq, y, reward);
  kv_out = biased_greedy(st->col_weights.data(), m.nk, y, reward);
}

// Alg. 1's assignment steps (planner.hpp:195-214) without the two workload
// tables: head plan reused or re-packed, block plan always recomputed.  Only
// head counts and grid marginals are read, so a caller that evaluates the
// tables elsewhere (on the GPU, select_batched) gets the same plan.
void plan_assign(const MaskView& m, Strategy s, const PlannerConfig& cfg, const Plan* prev,
                 const MaskStats* st, Outcome& out) {
  const uint32_t x = s.x, y = s.y;
  if (x > 1) {
    bool reuse = false;
    if (prev) {
      const std::vector<uint64_t> local = st ? std::vector<uint64_t>() : head_counts(m);
      const std::vector<uint64_t>& w = st ? st->head_counts : local;
      reuse = head_level_imbalance(w.data(), prev->head.data(), m.H, x) <= cfg.reuse_threshold;
    }
    if (reuse) {
      out.plan.head = prev->head;
    } else {
      out.plan.head = partition_heads(m, x, st);
      out.head_replanned = true;
    }
  } else {
    out.plan.head.assign(m.H, 0);
  }
  if (y > 1) {
    partition_blocks(m, y, cfg.exchange_reward, st, out.plan.q, out.plan.kv);
  } else {
    out.plan.q.assign(m.nq, 0);
    out.plan.kv.assign(m.nk, 0);
  }
}

namespace {
void check_prev(const MaskView& m, Strategy s, const Plan* prev) {
  if (prev) {
    if (prev->head.size() != m.H || prev->q.size() != m.nq || prev->kv.size() != m.nk)
      fail(kContract, "plan dimensions do not match the mask set");
    validate_plan(m, s, prev->head.data(), prev->q.data(), prev->kv.data());
  }
}
}  // namespace

// planner.hpp:175-217 (Alg. 1).
Outcome plan_dual(const MaskView& m, Strategy s, const PlannerConfig& cfg, const Plan* prev,
                  const MaskStats* st, Table* post_table) {
  cfg.validate();
  check_prev(m, s, prev);
  Outcome out;
  {
    Plan dflt;
    const Plan* pre = prev;
    if (!pre) {
      dflt = default_plan(m, s);
      pre = &dflt;
    }
    out.rho_pre = imbalance_ratio(
        workload_table(m, s, pre->head.data(), pre->q.data(), pre->kv.data(), st));
  }
  plan_assign(m, s, cfg, prev, st, out);
  Table post = workload_table(m, s, out.plan.head.data(), out.plan.q.data(),
                              out.plan.kv.data(), st);
  out.rho_post = imbalance_ratio(post);
  if (post_table) *post_table = std::move(post);
  return out;
}

namespace {

constexpr uint64_t kGuard = 10'000'000;

uint64_t capped_pow(uint64_t base, uint64_t e, uint64_t cap) {
  uint64_t v = 1;
  for (uint64_t i = 0; i < e; ++i) {
    if (v > cap / base) return cap + 1;
    v *= base;
  }
  return v;
}

bool odometer(std::vector<uint32_t>& a, uint32_t radix) {
  for (size_t i = a.size(); i-- > 0;) {
    if (++a[i] < radix) return true;
    a[i] = 0;
  }
  return false;
}

}  // namespace

// planner.hpp:249-272: first optimum in lexicographic order.
std::vector<uint32_t> brute_force_heads(const MaskView& m, uint32_t x) {
  if (x < 1 || x > m.H)
    fail(kConfig, "Ulysses degree " + str(x) + " must be in [1, " + str(m.H) + "]");
  if (capped_pow(x, m.H, kGuard) > kGuard)
    fail(kSearchSpace, "head search space exceeds " + str(kGuard) + " assignments");
  const std::vector<uint64_t> w = head_counts(m);
  std::vector<uint32_t> a(m.H, 0), best(m.H, 0);
  uint64_t best_max = std::numeric_limits<uint64_t>::max();
  std::vector<uint64_t> load(x);
  do {
    std::fill(load.begin(), load.end(), 0);
    for (uint32_t h = 0; h < m.H; ++h) load[a[h]] += w[h];
    const uint64_t mx = *std::max_element(load.begin(), load.end());
    if (mx < best_max) {
      best_max = mx;
      best = a;
    }
  } while (odometer(a, x));
  return best;
}

// planner.hpp:282-338: joint enumeration minimising the ring rho.
void brute_force_blocks(const uint64_t* grid, uint32_t nq, uint32_t nk, uint32_t y,
                        std::vector<uint32_t>& q_out, std::vector<uint32_t>& kv_out,
                        double& rho) {
  if (y < 1 || y > std::min(nq, nk)) fail(kConfig, "ring degree out of range for the grid");
  const uint64_t qs = capped_pow(y, nq, kGuard), ks = capped_pow(y, nk, kGuard);
  if (qs > kGuard || ks > kGuard || qs > kGuard / ks)
    fail(kSearchSpace, "block search space exceeds " + str(kGuard) + " assignments");
  uint64_t total = 0;
  for (size_t i = 0; i < size_t(nq) * nk; ++i) total += grid[i];
  q_out.assign(nq, 0);
  kv_out.assign(nk, 0);
  rho = std::numeric_limits<double>::infinity();
  if (total == 0) {
    rho = 1.0;
    return;
  }
  std::vector<uint32_t> qa(nq, 0);
  std::vector<uint64_t> cell(size_t(y) * y);
  do {
    std::vector<uint32_t> ka(nk, 0);
    do {
      std::fill(cell.begin(), cell.end(), 0);
      for (uint32_t q = 0; q < nq; ++q)
        for (uint32_t k = 0; k < nk; ++k) {
          const uint64_t s = grid[size_t(q) * nk + k];
          if (s) cell[size_t((ka[k] + y - qa[q]) % y) * y + qa[q]] += s;
        }
      uint64_t sum_max = 0;
      for (uint32_t i = 0; i < y; ++i) {
        uint64_t mx = 0;
        for (uint32_t r = 0; r < y; ++r) mx = std::max(mx, cell[size_t(i) * y + r]);
        sum_max += mx;
      }
      const double r = static_cast<double>(sum_max) * y / static_cast<double>(total);
      if (r < rho) {
        rho = r;
        q_out = qa;
        kv_out = ka;
      }
    } while (odometer(ka, y));
  } while (odometer(qa, y));
}

// ---------------------------------------------------------------------------
// latency.hpp

// latency.hpp:27-40.
double Curve::eval(double x) const {
  if (xs.empty()) fail(kContract, "empty latency curve");
  if (xs.size() == 1) return ys[0];
  size_t hi = size_t(std::upper_bound(xs.begin(), xs.end(), x) - xs.begin());
  if (hi == 0) hi = 1;
  if (hi == xs.size()) hi = xs.size() - 1;
  const size_t lo = hi - 1;
  if (x == xs[lo]) return ys[lo];
  if (x == xs[hi]) return ys[hi];
  if (ys[lo] == ys[hi]) return ys[lo];
  const double t = (x - xs[lo]) / (xs[hi] - xs[lo]);
  return std::max(0.0, ys[lo] + t * (ys[hi] - ys[lo]));
}

double Profile::all2all_at(uint32_t d, double bytes) const {
  const auto it = all2all.find(d);
  if (it == all2all.end()) fail(kConfig, "profile missing all2all degree " + str(d));
  return it->second.eval(bytes);
}

double Profile::p2p_at(uint32_t d, double bytes) const {
  const auto it = p2p.find(d);
  if (it == p2p.end()) fail(kConfig, "profile missing p2p degree " + str(d));
  return it->second.eval(bytes);
}

namespace {

// latency.hpp:86-110: sorted knots; repeated payloads fold pairwise into
// their running mean; monotone non-negative.
Curve knots(std::vector<std::pair<double, double>> pts, const std::string& what) {
  std::sort(pts.begin(), pts.end());
  Curve c;
  for (const auto& [x, y] : pts) {
    if (!c.xs.empty() && x == c.xs.back()) {
      c.ys.back() = (c.ys.back() + y) / 2.0;
      continue;
    }
    c.xs.push_back(x);
    c.ys.push_back(y);
  }
  if (c.xs.size() < 2) fail(kConfig, what + " needs at least 2 samples at distinct payloads");
  for (size_t i = 0; i < c.ys.size(); ++i) {
    if (c.ys[i] < 0.0) fail(kConfig, what + " has a negative latency sample");
    if (i > 0 && c.ys[i] < c.ys[i - 1])
      fail(kConfig, what + " is not monotone non-decreasing in payload");
  }
  return c;
}

}  // namespace

// latency.hpp:114-169.
Profile fit_profile(const std::vector<Sample>& samples, const FitOptions& o) {
  if (!(o.exchange_overlap >= 0.0 && o.exchange_overlap <= 1.0))
    fail(kConfig, "exchange_overlap must be in [0, 1]");
  if (o.replan_seconds < 0.0 || o.bytes_per_token_per_head <= 0.0)
    fail(kConfig, "replan_seconds must be >= 0 and bytes_per_token_per_head > 0");
  std::map<uint32_t, std::vector<std::pair<double, double>>> a2a, p2p;
  std::vector<std::pair<double, double>> dense;
  for (const Sample& s : samples) {
    if (s.primitive == 0)
      a2a[s.degree].emplace_back(s.x, s.seconds);
    else if (s.primitive == 1)
      p2p[s.degree].emplace_back(s.x, s.seconds);
    else if (s.primitive == 2)
      dense.emplace_back(s.x, s.seconds);
    else
      fail(kConfig, "unknown profile primitive '" + str(s.primitive) + "'");
  }
  Profile p;
  for (auto& [d, pts] : a2a) p.all2all[d] = knots(std::move(pts), "all2all degree " + str(d));
  for (auto& [d, pts] : p2p) p.p2p[d] = knots(std::move(pts), "p2p degree " + str(d));
  std::sort(dense.begin(), dense.end());
  double distinct = 0;
  for (size_t i = 0; i < dense.size(); ++i)
    if (i == 0 || dense[i].first != dense[i - 1].first) ++distinct;
  if (distinct < 2) fail(kConfig, "dense needs at least 2 samples at distinct densities");
  double sx = 0, sy = 0, sxx = 0, sxy = 0;
  const double n = static_cast<double>(dense.size());
  for (const auto& [d, s] : dense) {
    sx += d;
    sy += s;
    sxx += d * d;
    sxy += d * s;
  }
  const double slope = (n * sxy - sx * sy) / (n * sxx - sx * sx);
  if (!(slope >= 0.0)) fail(kConfig, "dense samples imply a negative cost slope");
  p.dense_attn_seconds = slope;
  p.launch_seconds = std::max(0.0, (sy - slope * sx) / n);
  p.exchange_overlap = o.exchange_overlap;
  p.replan_seconds = o.replan_seconds;
  p.bytes_per_token_per_head = o.bytes_per_token_per_head;
  return p;
}

// latency.hpp:225-268.  Expression order matches the reference term by term.
Latency predict_from_inputs(const CallInputs& in, const Profile& p) {
  const uint32_t x = in.strategy.x, y = in.strategy.y;
  if (x < 1 || y < 1) fail(kConfig, "parallel degrees must be >= 1");
  if (!(in.rho >= 1.0)) fail(kContract, "imbalance ratio must be >= 1");
  if (!(in.density >= 0.0 && in.density <= 1.0)) fail(kContract, "density must be in [0, 1]");
  const double gpus = static_cast<double>(x) * y;
  const double q_tok = static_cast<double>(in.q_blocks) * in.block_size;
  const double kv_tok = static_cast<double>(in.kv_blocks) * in.block_size;
  const double heads = static_cast<double>(in.heads);
  const double bpt = p.bytes_per_token_per_head;

  Latency out;
  const double iter = p.dense_attn_seconds * in.density / (gpus * y) + p.launch_seconds;
  if (x > 1) {
    const double qkv = (q_tok + 2.0 * kv_tok) * heads * bpt;
    out.all2all = p.all2all_at(x, qkv / gpus);
  }
  double exposed_iter = 0.0;
  if (y > 1) {
    const double kv_bytes = 2.0 * (kv_tok / y) * (heads / x) * bpt;
    exposed_iter = std::max(0.0, p.p2p_at(y, kv_bytes) - iter);
  }
  out.compute = iter * y;
  out.exposed = exposed_iter * (y - 1);
  const double body = out.compute + out.exposed;
  out.imbalance = in.rho > 1.0 ? body * (in.rho - 1.0) : 0.0;
  if (in.exchange.payload > 0 && p.exchange_overlap < 1.0) {
    const double bytes = static_cast<double>(in.exchange.payload) *
                         (static_cast<double>(in.heads) / x) * p.bytes_per_token_per_head;
    out.exchange = (1.0 - p.exchange_overlap) * p.all2all_at(y, bytes / y);
  }
  if (in.charge_replan) out.replan = p.replan_seconds;
  out.total = out.all2all + out.compute + out.exposed + out.imbalance + out.exchange + out.replan;
  return out;
}

// latency.hpp:270-283.  `known_rho` lets the selector pass rho_post, which
// is the same workload_table/imbalance_ratio evaluation on the same plan.
Latency predict_latency(const MaskView& m, Strategy s, const Plan& plan, const Profile& p,
                        bool charge_replan, const MaskStats* st, const double* known_rho) {
  if (plan.head.size() != m.H || plan.q.size() != m.nq || plan.kv.size() != m.nk)
    fail(kContract, "plan dimensions do not match the mask set");
  CallInputs in;
  in.heads = m.H;
  in.q_blocks = m.nq;
  in.kv_blocks = m.nk;
  in.block_size = m.block_size;
  in.strategy = s;
  in.density = st ? static_cast<double>(st->total) / static_cast<double>(m.cells()) : density(m);
  in.rho = known_rho ? *known_rho
                     : imbalance_ratio(workload_table(m, s, plan.head.data(), plan.q.data(),
                                                      plan.kv.data(), st));
  validate_plan(m, s, plan.head.data(), plan.q.data(), plan.kv.data());
  in.exchange = exchange_volume(m, s, plan.q.data(), plan.kv.data());
  in.charge_replan = charge_replan;
  return predict_from_inputs(in, p);
}

// latency.hpp:295-315.
std::vector<Prediction> predict_all(const MaskView& m, const Profile& p, uint32_t gpus,
                                    const PlannerConfig& cfg,
                                    const std::map<Strategy, Plan>& prev) {
  const std::vector<Strategy> all = enumerate_strategies(gpus);
  bool ring = false;
  for (Strategy s : all)
    if (s.x <= m.H && s.y > 1 && s.y <= std::min(m.nq, m.nk)) ring = true;
  const MaskStats st = mask_stats(m, ring);
  std::vector<Strategy> feasible;
  for (Strategy s : all)
    if (s.x <= m.H && s.y <= std::min(m.nq, m.nk)) feasible.push_back(s);
  if (feasible.empty())
    fail(kConfig, "no feasible strategy for " + str(gpus) + " GPUs on this mask shape");
  // Strategies are independent (each reads the shared, immutable MaskStats),
  // so they are planned on parallel threads; results land in enumeration
  // order, so the outcome is identical to the sequential loop.
  std::vector<Prediction> out(feasible.size());
  std::vector<std::exception_ptr> errs(feasible.size());
  auto work = [&](size_t i) {
    try {
      const Strategy s = feasible[i];
      const auto it = prev.find(s);
      Prediction pr;
      pr.strategy = s;
      pr.outcome = plan_dual(m, s, cfg, it != prev.end() ? &it->second : nullptr, &st);
      pr.latency = predict_latency(m, s, pr.outcome.plan, p, false, &st, &pr.outcome.rho_post);
      out[i] = std::move(pr);
    } catch (...) {
      errs[i] = std::current_exception();
    }
  };
  const bool threaded = feasible.size() > 1 && uint64_t(m.H) * m.nq * m.wpr >= 4096 &&
                        std::thread::hardware_concurrency() > 1;
  if (threaded) {
    std::vector<std::thread> pool;
    for (size_t i = 1; i < feasible.size(); ++i) pool.emplace_back(work, i);
    work(0);
    for (std::thread& t : pool) t.join();
  } else {
    for (size_t i = 0; i < feasible.size(); ++i) work(i);
  }
  for (const std::exception_ptr& e : errs)  // first error in enumeration order wins
    if (e) std::rethrow_exception(e);
  return out;
}

// ---------------------------------------------------------------------------
// selector.hpp

Selector::Selector(uint32_t gpus) : gpus_(gpus) { (void)enumerate_strategies(gpus); }

bool Selector::stored(int64_t layer, Strategy& s, Plan& p) const {
  std::lock_guard<std::mutex> lock(mu_);
  const auto it = prev_.find(layer);
  if (it == prev_.end()) return false;
  s = it->second.first;
  p = it->second.second;
  return true;
}

void Selector::store(int64_t layer, Strategy s, Plan p) {
  std::lock_guard<std::mutex> lock(mu_);
  prev_[layer] = {s, std::move(p)};
}

// selector.hpp:55-75: first strict minimum in enumeration order (descending
// x), so exact ties go to the larger Ulysses degree.
Prediction select(Selector& state, int64_t layer, const MaskView& m, const Profile& p,
                  const PlannerConfig& cfg) {
  std::map<Strategy, Plan> prev;
  Strategy s;
  Plan plan;
  if (state.stored(layer, s, plan)) prev.emplace(s, std::move(plan));
  std::vector<Prediction> all = predict_all(m, p, state.gpus(), cfg, prev);
  size_t best = 0;
  for (size_t i = 1; i < all.size(); ++i)
    if (all[i].latency.total < all[best].latency.total) best = i;
  state.store(layer, all[best].strategy, all[best].outcome.plan);
  return std::move(all[best]);
}

// select() with the mask-dependent integers supplied from outside: `st`
// (head counts, grid marginals) and the workload tables (`tables`, one call
// for every (strategy, plan) pair of the selection).  Used by the device path
// (dbsp_select_device), where K1 and a table kernel produce them on the GPU;
// `m` then carries dimensions only.  Plans, doubles and the argmin follow the
// same code as select(), so the result is identical to the host path.
Prediction select_batched(Selector& state, int64_t layer, const MaskView& m, const MaskStats& st,
                          const Profile& p, const PlannerConfig& cfg, const BatchTables& tables) {
  cfg.validate();
  std::map<Strategy, Plan> prev;
  {
    Strategy s;
    Plan plan;
    if (state.stored(layer, s, plan)) prev.emplace(s, std::move(plan));
  }
  std::vector<Strategy> feasible;
  for (Strategy s : enumerate_strategies(state.gpus()))
    if (s.x <= m.H && s.y <= std::min(m.nq, m.nk)) feasible.push_back(s);
  if (feasible.empty())
    fail(kConfig, "no feasible strategy for " + str(state.gpus()) + " GPUs on this mask shape");
  std::vector<Prediction> all(feasible.size());
  std::vector<Plan> pre(feasible.size());
  std::vector<TableJob> jobs;
  for (size_t i = 0; i < feasible.size(); ++i) {
    const Strategy s = feasible[i];
    const auto it = prev.find(s);
    const Plan* pv = it != prev.end() ? &it->second : nullptr;
    check_prev(m, s, pv);
    pre[i] = pv ? *pv : default_plan(m, s);
    all[i].strategy = s;
    plan_assign(m, s, cfg, pv, &st, all[i].outcome);
    validate_plan(m, s, all[i].outcome.plan.head.data(), all[i].outcome.plan.q.data(),
                  all[i].outcome.plan.kv.data());
  }
  for (size_t i = 0; i < feasible.size(); ++i) {
    jobs.push_back({feasible[i], &pre[i]});
    jobs.push_back({feasible[i], &all[i].outcome.plan});
  }
  const std::vector<Table> t = tables(jobs);
  if (t.size() != jobs.size()) fail(kInternal, "table provider returned the wrong count");
  for (size_t i = 0; i < feasible.size(); ++i) {
    all[i].outcome.rho_pre = imbalance_ratio(t[2 * i]);
    all[i].outcome.rho_post = imbalance_ratio(t[2 * i + 1]);
    all[i].latency = predict_latency(m, feasible[i], all[i].outcome.plan, p, false, &st,
                                     &all[i].outcome.rho_post);
  }
  size_t best = 0;
  for (size_t i = 1; i < all.size(); ++i)
    if (all[i].latency.total < all[best].latency.total) best = i;
  state.store(layer, all[best].strategy, all[best].outcome.plan);
  return std::move(all[best]);
}

}  // namespace dbsp_core
