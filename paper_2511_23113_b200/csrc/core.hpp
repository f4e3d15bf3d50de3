// Internal host core of the db-SP planner (C++20).  Everything here is plain
// integer / double arithmetic over flat views; the C ABI (capi.cpp) wraps it,
// the C++ drop-in API (include/dbsp/*.hpp) and the Python package sit on top.
//
// Bit-exactness contract: every function reproduces the reference result for
// the same inputs (assignment vectors exactly, doubles to the last bit).  The
// planner is compiled with -ffp-contract=off so no FMA contraction changes a
// double expression.  Where this file is faster than the reference it is by
// computing the same integers differently (bit-sliced column counts instead
// of a per-bit walk, marginals computed once per call instead of once per
// ring degree), never by changing an expression that produces a double.
#pragma once

#include <cstddef>
#include <atomic>
#include <cstdint>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <functional>
#include <vector>

namespace dbsp_core {

// Kernel launches issued by this library (dbsp_launch_count): every launch
// site of our kernels bumps it (CUB's own kernels inside K2 are not counted).
inline std::atomic<uint64_t> g_launches{0};
inline void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }


// Status codes shared with the C ABI (include/dbsp_b200.h).
enum Code : int {
  kOk = 0,
  kInternal = 1,
  kConfig = 2,
  kIo = 3,
  kContract = 4,
  kParse = 5,
  kSearchSpace = 6,
  kCuda = 7,
};

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& what) : std::runtime_error(what), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& what) { throw Error(code, what); }

// splitmix64 (reference rng.hpp:10-35).
struct SplitMix {
  uint64_t s;
  explicit SplitMix(uint64_t seed) : s(seed) {}
  uint64_t u64() {
    s += 0x9e3779b97f4a7c15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double unit() { return static_cast<double>(u64() >> 11) * 0x1.0p-53; }
  bool coin(double p) { return unit() < p; }
  uint64_t below(uint64_t n) {
    return static_cast<uint64_t>((static_cast<unsigned __int128>(u64()) * n) >> 64);
  }
};

// rng.hpp:37-40.
inline uint64_t mix_seed(uint64_t base, uint64_t a, uint64_t b) {
  SplitMix r(base ^ (a * 0x9e3779b97f4a7c15ull) ^ (b * 0xc2b2ae3d27d4eb4full));
  return r.u64();
}

// Read-only view of a mask set: H pointers to Q-major rows of `wpr` words.
struct MaskView {
  const uint64_t* const* heads = nullptr;
  uint32_t H = 0, nq = 0, nk = 0, block_size = 0;
  size_t wpr = 0;

  const uint64_t* row(uint32_t h, uint32_t q) const { return heads[h] + size_t(q) * wpr; }
  uint64_t cells() const { return uint64_t(H) * nq * nk; }
};

MaskView make_view(const uint64_t* const* heads, uint32_t H, uint32_t nq, uint32_t nk,
                   uint32_t block_size);

struct Strategy {
  uint32_t x = 1, y = 1;
  uint32_t gpus() const { return x * y; }
  bool operator<(const Strategy& o) const { return x != o.x ? x < o.x : y < o.y; }
  bool operator==(const Strategy& o) const { return x == o.x && y == o.y; }
};

struct Plan {
  std::vector<uint32_t> head, q, kv;
};

struct Table {
  uint32_t gpus = 1, periods = 1;
  std::vector<uint64_t> counts;  // periods x gpus, row-major
  uint64_t total() const {
    uint64_t t = 0;
    for (uint64_t c : counts) t += c;
    return t;
  }
};

struct Exchange {
  uint64_t q_moved = 0, kv_moved = 0, payload = 0;
};

struct PlannerConfig {
  double reuse_threshold = 1.10;
  double exchange_reward = 0.0;
  void validate() const;
};

struct Outcome {
  Plan plan;
  bool head_replanned = false;
  double rho_pre = 1.0, rho_post = 1.0;
};

// Strategy-independent integers derived from one mask set.  Computed once per
// selector call and shared by every strategy's planning (the reference
// recomputes them per strategy; the integers are identical).
struct MaskStats {
  std::vector<uint64_t> head_counts;  // blocks_per_head
  std::vector<uint64_t> row_weights;  // Q marginals of summed_grid
  std::vector<uint64_t> col_weights;  // KV marginals of summed_grid
  uint64_t total = 0;
  bool have_marginals = false;
};

// --- mask.hpp ---------------------------------------------------------------
struct GenSpec {
  uint32_t H = 1, nq = 1, nk = 1, block_size = 64, pattern = 0;
  double dmin = 0.5, dmax = 0.5, skew = 1.0;
  uint64_t seed = 0;
};
void generate_masks(const GenSpec& spec, uint64_t* out);
void perturb_masks(const MaskView& in, double flip_rate, uint64_t seed, uint64_t* out);
uint64_t popcount_words(const uint64_t* w, size_t n);
std::vector<uint64_t> head_counts(const MaskView& m);
uint64_t total_blocks(const MaskView& m);
double density(const MaskView& m);
MaskStats mask_stats(const MaskView& m, bool marginals);

// --- metrics.hpp ------------------------------------------------------------
std::vector<Strategy> enumerate_strategies(uint32_t gpus);
void validate_plan(const MaskView& m, Strategy s, const uint32_t* head, const uint32_t* q,
                   const uint32_t* kv);
Plan default_plan(const MaskView& m, Strategy s);
Table workload_table(const MaskView& m, Strategy s, const uint32_t* head, const uint32_t* q,
                     const uint32_t* kv, const MaskStats* stats = nullptr);
double imbalance_ratio(const uint64_t* counts, uint32_t periods, uint32_t gpus);
inline double imbalance_ratio(const Table& t) {
  return imbalance_ratio(t.counts.data(), t.periods, t.gpus);
}
Exchange exchange_volume(const MaskView& m, Strategy s, const uint32_t* q, const uint32_t* kv);

// --- planner.hpp ------------------------------------------------------------
std::vector<uint64_t> summed_grid(const MaskView& m);
double head_level_imbalance(const uint64_t* w, const uint32_t* a, size_t n, uint32_t x);
std::vector<uint32_t> lpt_heads(const std::vector<uint64_t>& weights, uint32_t x);
std::vector<uint32_t> partition_heads(const MaskView& m, uint32_t x, const MaskStats* st);
std::vector<uint32_t> biased_greedy(const uint64_t* w, size_t n, uint32_t y, double reward);
void partition_blocks(const MaskView& m, uint32_t y, double reward, const MaskStats* st,
                      std::vector<uint32_t>& q_out, std::vector<uint32_t>& kv_out);
Outcome plan_dual(const MaskView& m, Strategy s, const PlannerConfig& cfg, const Plan* prev,
                  const MaskStats* st = nullptr, Table* post_table = nullptr);
std::vector<uint32_t> brute_force_heads(const MaskView& m, uint32_t x);
void brute_force_blocks(const uint64_t* grid, uint32_t nq, uint32_t nk, uint32_t y,
                        std::vector<uint32_t>& q_out, std::vector<uint32_t>& kv_out,
                        double& rho);

// --- latency.hpp ------------------------------------------------------------
struct Curve {
  std::vector<double> xs, ys;
  double eval(double x) const;
};
struct Profile {
  std::map<uint32_t, Curve> all2all, p2p;
  double dense_attn_seconds = 0, launch_seconds = 0, exchange_overlap = 1.0;
  double replan_seconds = 0, bytes_per_token_per_head = 256.0;
  double all2all_at(uint32_t degree, double bytes) const;
  double p2p_at(uint32_t degree, double bytes) const;
};
struct Sample {
  uint32_t primitive;  // 0 all2all, 1 p2p, 2 dense
  uint32_t degree;
  double x, seconds;
};
struct FitOptions {
  double exchange_overlap = 1.0, replan_seconds = 0.0, bytes_per_token_per_head = 256.0;
};
Profile fit_profile(const std::vector<Sample>& samples, const FitOptions& opt);
struct Latency {
  double all2all = 0, compute = 0, exposed = 0, imbalance = 0, exchange = 0, replan = 0,
         total = 0;
};
struct CallInputs {
  uint32_t heads = 1, q_blocks = 1, kv_blocks = 1, block_size = 1;
  Strategy strategy;
  double density = 0, rho = 1;
  Exchange exchange;
  bool charge_replan = false;
};
Latency predict_from_inputs(const CallInputs& in, const Profile& p);
Latency predict_latency(const MaskView& m, Strategy s, const Plan& plan, const Profile& p,
                        bool charge_replan, const MaskStats* st = nullptr,
                        const double* known_rho = nullptr);
struct Prediction {
  Strategy strategy;
  Outcome outcome;
  Latency latency;
};
std::vector<Prediction> predict_all(const MaskView& m, const Profile& p, uint32_t gpus,
                                    const PlannerConfig& cfg,
                                    const std::map<Strategy, Plan>& prev);

// --- selector.hpp -----------------------------------------------------------
class Selector {
 public:
  explicit Selector(uint32_t gpus);
  uint32_t gpus() const { return gpus_; }
  bool stored(int64_t layer, Strategy& s, Plan& p) const;
  void store(int64_t layer, Strategy s, Plan p);

 private:
  uint32_t gpus_;
  mutable std::mutex mu_;
  std::map<int64_t, std::pair<Strategy, Plan>> prev_;
};
// One workload table per (strategy, plan) job; see select_batched.
struct TableJob {
  Strategy s;
  const Plan* plan;
};
using BatchTables = std::function<std::vector<Table>(const std::vector<TableJob>&)>;
void plan_assign(const MaskView& m, Strategy s, const PlannerConfig& cfg, const Plan* prev,
                 const MaskStats* st, Outcome& out);
Prediction select_batched(Selector& state, int64_t layer, const MaskView& m, const MaskStats& st,
                          const Profile& p, const PlannerConfig& cfg, const BatchTables& tables);
Prediction select(Selector& state, int64_t layer, const MaskView& m, const Profile& p,
                  const PlannerConfig& cfg);

}  // namespace dbsp_core
