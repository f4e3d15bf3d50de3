// C++ drop-in API check: code written against the reference's `dbsp` headers
// (names, signatures, exception classes) compiles against include/dbsp/*.hpp
// and links libdbsp_b200.so.  The checks restate the reference acceptance
// criteria that need no simulator (proj/tests/acceptance.cpp c1-c6, c8, c9)
// plus the error behaviour of the reference unit tests.  Prints one line per
// check; exit code = number of failures.
#include "dbsp/attention.hpp"  // SpContext / sparse_attention: compiled and linked, not run (no GPU)
#include <algorithm>
#include <cmath>
#include <filesystem>
#include <fstream>
#include <unistd.h>
#include <cstdio>
#include <functional>
#include <limits>
#include <numeric>
#include <string>
#include <vector>

#include "dbsp/latency.hpp"
#include "dbsp/mask.hpp"
#include "dbsp/mask_io.hpp"
#include "dbsp/metrics.hpp"
#include "dbsp/planner.hpp"
#include "dbsp/selector.hpp"

using namespace dbsp;

static int failures = 0;

static void expect(bool ok, const std::string& what) {
  std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what.c_str());
  if (!ok) ++failures;
}

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static AttentionMaskSet bernoulli_set(Rng& rng, uint32_t H, uint32_t nq, uint32_t nk, double p) {
  std::vector<BlockMask> heads;
  for (uint32_t h = 0; h < H; ++h) {
    BlockMask m(nq, nk);
    for (uint32_t q = 0; q < nq; ++q)
      for (uint32_t k = 0; k < nk; ++k)
        if (rng.bernoulli(p)) m.set(q, k, true);
    heads.push_back(std::move(m));
  }
  return AttentionMaskSet(std::move(heads), 64);
}

static AttentionMaskSet weights_set(const std::vector<uint64_t>& w, uint32_t cap) {
  std::vector<BlockMask> heads;
  for (uint64_t x : w) {
    BlockMask m(1, cap);
    for (uint32_t k = 0; k < x; ++k) m.set(0, k, true);
    heads.push_back(std::move(m));
  }
  return AttentionMaskSet(std::move(heads), 64);
}

static uint64_t peak(const std::vector<uint64_t>& w, const std::vector<uint32_t>& a, uint32_t x) {
  std::vector<uint64_t> l(x, 0);
  for (size_t i = 0; i < w.size(); ++i) l[a[i]] += w[i];
  return *std::max_element(l.begin(), l.end());
}

static MachineProfile node() {
  MachineProfile p;
  const std::vector<double> x = {1e6, 1.6e7, 2.56e8, 1.07e9};
  p.all2all[2] = {x, {3e-5, 1.2e-4, 1.5e-3, 5.5e-3}};
  p.all2all[4] = {x, {4e-5, 1.8e-4, 2.2e-3, 8e-3}};
  p.all2all[8] = {x, {5e-5, 2.4e-4, 3e-3, 1.1e-2}};
  p.p2p[2] = {x, {2e-5, 9e-5, 1.2e-3, 4.6e-3}};
  p.p2p[4] = {x, {2.2e-5, 9.5e-5, 1.25e-3, 4.8e-3}};
  p.p2p[8] = {x, {2.4e-5, 1e-4, 1.3e-3, 5e-3}};
  p.dense_attn_seconds = 0.65;
  p.launch_seconds = 1e-4;
  p.exchange_overlap = 0.95;
  p.replan_seconds = 2e-4;
  return p;
}

int main() {
  {  // the attention faces link (their calls need a GPU and are exercised from Python)
    volatile auto uid = &dbsp::SpContext::unique_id;
    void (*sp)(dbsp::SpContext&, const dbsp::AttentionMaskSet&, dbsp::ParallelStrategy, const dbsp::PartitionPlan&,
               const void*, const void*, const void*, void*, uint32_t, void*) = &dbsp::sparse_attention;
    (void)uid;
    (void)sp;
    auto* sd = &dbsp::select_device;
    auto* qp = &dbsp::qkv_project;
    (void)sd;
    (void)qp;
  }
  // c1: rho fixtures.
  {
    WorkloadTable a{2, {{3, 1}, {2, 2}}}, b{2, {{4, 0}}}, c{2, {{5, 5}, {7, 7}}};
    expect(imbalance_ratio(a) == 1.25 && imbalance_ratio(b) == 2.0 && imbalance_ratio(c) == 1.0,
           "c1 rho fixtures [[3,1],[2,2]]=1.25 [[4,0]]=2 uniform=1");
  }
  // c2: workload tables conserve the block total.
  {
    Rng rng(20001);
    bool ok = true;
    for (int i = 0; i < 300 && ok; ++i) {
      const uint32_t H = 1 + uint32_t(rng.next_below(16)), nq = 1 + uint32_t(rng.next_below(32)),
                     nk = 1 + uint32_t(rng.next_below(32)), G = 1u << (1 + rng.next_below(3));
      const auto all = enumerate_strategies(G);
      const ParallelStrategy s = all[rng.next_below(all.size())];
      const AttentionMaskSet set = bernoulli_set(rng, H, nq, nk, rng.next_double());
      PartitionPlan p;
      for (uint32_t h = 0; h < H; ++h) p.head_assignment.push_back(uint32_t(rng.next_below(s.ulysses)));
      for (uint32_t q = 0; q < nq; ++q) p.q_assignment.push_back(uint32_t(rng.next_below(s.ring)));
      for (uint32_t k = 0; k < nk; ++k) p.kv_assignment.push_back(uint32_t(rng.next_below(s.ring)));
      const auto hc = blocks_per_head(set);
      ok = workload_table(set, s, p).total() == std::accumulate(hc.begin(), hc.end(), uint64_t(0));
    }
    expect(ok, "c2 300 random (mask, strategy, plan) triples conserve block totals");
  }
  // c3: LPT within 4/3 - 1/(3x) of the exhaustive optimum.
  {
    Rng rng(30001);
    bool ok = peak({7, 5, 3, 1}, partition_heads(weights_set({7, 5, 3, 1}, 9), 2), 2) == 8 &&
              peak({5, 4, 3}, partition_heads(weights_set({5, 4, 3}, 9), 2), 2) == 7;
    for (int i = 0; i < 300 && ok; ++i) {
      const uint32_t x = 2 + uint32_t(rng.next_below(2));
      const uint32_t H = x + uint32_t(rng.next_below(9 - x));
      std::vector<uint64_t> w(H);
      for (auto& v : w) v = rng.next_below(10);
      const AttentionMaskSet set = weights_set(w, 9);
      const double g = double(peak(w, partition_heads(set, x), x));
      const double o = double(peak(w, brute_force_heads(set, x), x));
      ok = g <= (4.0 / 3.0 - 1.0 / (3.0 * x)) * o + 1e-9;
    }
    expect(ok, "c3 LPT head greedy within the LPT bound of brute_force_heads");
  }
  // c4: block greedy within 1.15x of the joint oracle on 6x6 grids.
  {
    Rng rng(40001);
    double worst = 1.0;
    for (int i = 0; i < 60; ++i) {
      const AttentionMaskSet set = bernoulli_set(rng, 1, 6, 6, 0.5);
      const auto [qa, ka] = partition_blocks(set, 2, 0.0);
      const PartitionPlan p{{0}, qa, ka};
      const double g = imbalance_ratio(workload_table(set, {1, 2}, p));
      const double o = brute_force_blocks(summed_grid(set), 6, 6, 2).rho;
      worst = std::max(worst, g / o);
    }
    char buf[96];
    std::snprintf(buf, sizeof(buf), "c4 block greedy vs joint oracle, worst ratio %.4f <= 1.15", worst);
    expect(worst <= 1.15 + 1e-12, buf);
  }
  // c5: post-balance quality at scale.
  {
    int u_ok = 0, r_ok = 0;
    for (uint64_t seed = 0; seed < 30; ++seed) {
      GeneratorSpec spec;
      spec.num_heads = 40;
      spec.num_q_blocks = spec.num_kv_blocks = 64;
      spec.min_density = 0.2;
      spec.max_density = 0.8;
      spec.seed = 50000 + seed;
      const AttentionMaskSet set = generate_mask_set(spec);
      const PartitionPlan up{partition_heads(set, 8), std::vector<uint32_t>(64, 0),
                             std::vector<uint32_t>(64, 0)};
      u_ok += imbalance_ratio(workload_table(set, {8, 1}, up)) <= 1.1;
      auto [qa, ka] = partition_blocks(set, 8, 0.0);
      const PartitionPlan rp{std::vector<uint32_t>(40, 0), qa, ka};
      r_ok += imbalance_ratio(workload_table(set, {1, 8}, rp)) <= 1.05;
    }
    expect(u_ok >= 28 && r_ok >= 28, "c5 post-balance rho: Ulysses x=8 <= 1.1 and ring y=8 <= 1.05");
  }
  // c6: reward limits.
  {
    Rng rng(60001);
    bool ok = true;
    for (int i = 0; i < 40 && ok; ++i) {
      const uint32_t nq = 2 + uint32_t(rng.next_below(15)), nk = 2 + uint32_t(rng.next_below(15));
      const uint32_t H = 1 + uint32_t(rng.next_below(4));
      const AttentionMaskSet set = bernoulli_set(rng, H, nq, nk, i % 2 ? 0.5 : 0.125);
      const auto [qa, ka] = partition_blocks(set, 2, kInfiniteReward);
      ok = exchange_volume(set, {1, 2}, PartitionPlan{std::vector<uint32_t>(H, 0), qa, ka}) ==
           ExchangeVolume{};
    }
    expect(ok, "c6 R_b = inf keeps every block at its home rank");
  }
  // c8: Eq. 4 reductions.
  {
    const MachineProfile p = node();
    Rng rng(80001);
    const AttentionMaskSet set = bernoulli_set(rng, 8, 16, 16, 0.6);
    const bool a = predict_latency(set, {8, 1}, default_plan(set, {8, 1}), p).ring_p2p_exposed_s == 0.0;
    const bool b = predict_latency(set, {1, 8}, default_plan(set, {1, 8}), p).all2all_s == 0.0;
    CallInputs in;
    in.shape = mask_shape(set);
    in.strategy = {2, 4};
    in.density = 0.6;
    in.rho = 1.17;
    const double once = predict_from_inputs(in, p).attn_seconds();
    in.rho = 2.34;
    const double twice = predict_from_inputs(in, p).attn_seconds();
    expect(a && b && std::abs(twice - 2.0 * once) <= 1e-12 * std::max(1.0, twice),
           "c8 y=1 drops p2p, x=1 drops all2all, attention linear in rho");
  }
  // c9: select() is the argmin over the enumeration; infinite p2p pins U8R1.
  {
    const MachineProfile p = node();
    Rng rng(90001);
    bool ok = enumerate_strategies(8) == std::vector<ParallelStrategy>{{8, 1}, {4, 2}, {2, 4}, {1, 8}};
    for (int i = 0; i < 40 && ok; ++i) {
      const uint32_t H = 8u << rng.next_below(2), nb = 16u << rng.next_below(2);
      const AttentionMaskSet set = bernoulli_set(rng, H, nb, nb, 0.15 + 0.7 * rng.next_double());
      SelectorState st(8);
      const Selection sel = select(0, set, p, PlannerConfig{}, st);
      double best = std::numeric_limits<double>::infinity();
      for (ParallelStrategy s : enumerate_strategies(8))
        best = std::min(best, predict_latency(set, s, plan_dual(set, s, PlannerConfig{}).plan, p).total_s);
      ok = sel.latency.total_s == best && st.stored(0).has_value();
    }
    MachineProfile slow = node();
    for (uint32_t d : {2u, 4u, 8u})
      slow.p2p[d] = {{0.0, 1e12}, {std::numeric_limits<double>::infinity(),
                                   std::numeric_limits<double>::infinity()}};
    Rng rng2(90002);
    SelectorState st(8);
    ok = ok && select(0, bernoulli_set(rng2, 16, 16, 16, 0.5), slow, PlannerConfig{}, st).strategy ==
                   ParallelStrategy{8, 1};
    expect(ok, "c9 select() is the argmin of predict_latency over the strategies");
  }
  // Error classes (reference unit tests).
  {
    const AttentionMaskSet set = weights_set({3, 2, 1}, 3);
    bool ok = throws<config_error>([&] { partition_heads(set, 4); }) &&
              throws<config_error>([&] { enumerate_strategies(6); }) &&
              throws<config_error>([&] { parse_strategy("U0R4"); }) &&
              throws<config_error>([&] { default_plan(set, {8, 1}); }) &&
              throws<search_space_error>([&] { brute_force_heads(weights_set(std::vector<uint64_t>(30, 1), 1), 2); }) &&
              throws<config_error>([&] { plan_dual(set, {2, 1}, PlannerConfig{0.5, 0.0}); }) &&
              throws<contract_error>([&] {
                workload_table(set, {2, 1}, PartitionPlan{{0, 2, 0}, {0}, {0, 0, 0}});
              }) &&
              throws<config_error>([&] { BlockMask(0, 3); });
    expect(ok, "errors map to the reference exception classes");
  }
  // mask_io.hpp (reference mask_io.hpp:131-207) and save_profile (latency.hpp:377-379).
  {
    namespace fs = std::filesystem;
    const fs::path dir = fs::temp_directory_path() / ("dbsp_api_test_" + std::to_string(::getpid()));
    fs::create_directories(dir);
    Rng rng(777);
    const AttentionMaskSet set = bernoulli_set(rng, 3, 5, 70, 0.4);
    save_mask_set(set, dir / "m.bin");
    bool ok = load_mask_set(dir / "m.bin") == set;
    // a JSON fixture sidecar: 2 heads x 1 row, 12 KV blocks (2 bytes per row)
    {
      std::ofstream f(dir / "side.json");
      f << R"({"heads": 2, "q_blocks": 1, "kv_blocks": 12, "block_size": 64, "rows": ["0108", "ff0f"]})";
    }
    const AttentionMaskSet side = load_mask_set(dir / "side.json");
    ok = ok && side.head(0).get(0, 0) && side.head(0).get(0, 11) && side.head(0).row_popcount(0) == 2 &&
         side.head(1).row_popcount(0) == 12;
    {
      std::ofstream f(dir / "bad.bin", std::ios::binary);
      f << "DBSPMSK2garbage";
    }
    ok = ok && throws<parse_error>([&] { load_mask_set(dir / "bad.bin"); }) &&
         throws<io_error>([&] { load_mask_set(dir / "missing.bin"); });
    const MachineProfile prof = node();
    save_profile(prof, dir / "p.json");
    const MachineProfile back = load_profile(dir / "p.json");
    // the JSON stores samples and load_profile re-fits them (as the reference
    // does): curves come back exactly, the dense least-squares fit to rounding
    auto close = [](double a, double b) { return std::fabs(a - b) <= 1e-12 * std::max(1.0, std::fabs(b)); };
    ok = ok && close(back.dense_attn_seconds, prof.dense_attn_seconds) && close(back.launch_seconds, prof.launch_seconds) &&
         back.all2all.size() == prof.all2all.size() && back.p2p.size() == prof.p2p.size() &&
         back.all2all_at(8, 1e6) == prof.all2all_at(8, 1e6) && back.p2p_at(2, 3e5) == prof.p2p_at(2, 3e5);
    fs::remove_all(dir);
    expect(ok, "mask_io round trip + JSON sidecar + parse/io errors; save_profile -> load_profile");
  }
  std::printf("%d failure(s)\n", failures);
  return failures;
}
