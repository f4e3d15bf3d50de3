// Eq. 4 latency model — drop-in counterpart of the reference's
// proj/include/dbsp/latency.hpp (PiecewiseLinear :23-41, MachineProfile
// :45-67, ProfileSample / FitOptions / fit_profile :71-169, LatencyBreakdown
// :172-184, CallInputs / predict_from_inputs :199-268, predict_latency
// :270-283, predict_all :295-315, profile JSON :322-379).  Evaluation runs in
// libdbsp_b200.so and matches the reference to the last bit.
#pragma once

#include <cstdint>
#include <filesystem>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "../dbsp_b200.h"
#include "error.hpp"
#include "mask.hpp"
#include "metrics.hpp"
#include "planner.hpp"

namespace dbsp {

struct PiecewiseLinear {
  std::vector<double> xs;  // strictly increasing
  std::vector<double> ys;
  double eval(double x) const {
    if (xs.size() != ys.size()) throw contract_error("curve knots and values differ in length");
    double out = 0;
    detail::check(dbsp_pwl_eval(xs.data(), ys.data(), uint32_t(xs.size()), x, &out));
    return out;
  }
};

struct MachineProfile {
  std::map<uint32_t, PiecewiseLinear> all2all;  // Ulysses degree -> curve over per-GPU bytes
  std::map<uint32_t, PiecewiseLinear> p2p;      // ring degree -> curve over per-GPU bytes
  double dense_attn_seconds = 0.0;
  double launch_seconds = 0.0;
  double exchange_overlap = 1.0;
  double replan_seconds = 0.0;
  double bytes_per_token_per_head = 256.0;

  double all2all_at(uint32_t degree, double payload_bytes) const {
    const auto it = all2all.find(degree);
    if (it == all2all.end())
      throw config_error("profile missing all2all degree " + std::to_string(degree));
    return it->second.eval(payload_bytes);
  }
  double p2p_at(uint32_t degree, double payload_bytes) const {
    const auto it = p2p.find(degree);
    if (it == p2p.end()) throw config_error("profile missing p2p degree " + std::to_string(degree));
    return it->second.eval(payload_bytes);
  }
};

namespace detail {

// Flattened C view of a profile (keeps the arrays alive).
struct ProfileView {
  explicit ProfileView(const MachineProfile& p) {
    flatten(p.all2all, a_deg, a_off, a_x, a_y);
    flatten(p.p2p, p_deg, p_off, p_x, p_y);
    c.num_all2all = uint32_t(a_deg.size());
    c.all2all_degrees = a_deg.data();
    c.all2all_offsets = a_off.data();
    c.all2all_x = a_x.data();
    c.all2all_y = a_y.data();
    c.num_p2p = uint32_t(p_deg.size());
    c.p2p_degrees = p_deg.data();
    c.p2p_offsets = p_off.data();
    c.p2p_x = p_x.data();
    c.p2p_y = p_y.data();
    c.dense_attn_seconds = p.dense_attn_seconds;
    c.launch_seconds = p.launch_seconds;
    c.exchange_overlap = p.exchange_overlap;
    c.replan_seconds = p.replan_seconds;
    c.bytes_per_token_per_head = p.bytes_per_token_per_head;
  }
  ProfileView(const ProfileView&) = delete;
  ProfileView& operator=(const ProfileView&) = delete;
  const dbsp_profile* get() const { return &c; }

 private:
  static void flatten(const std::map<uint32_t, PiecewiseLinear>& t, std::vector<uint32_t>& deg,
                      std::vector<uint32_t>& off, std::vector<double>& x, std::vector<double>& y) {
    off.push_back(0);
    for (const auto& [d, curve] : t) {
      if (curve.xs.size() != curve.ys.size())
        throw contract_error("curve knots and values differ in length");
      deg.push_back(d);
      x.insert(x.end(), curve.xs.begin(), curve.xs.end());
      y.insert(y.end(), curve.ys.begin(), curve.ys.end());
      off.push_back(uint32_t(x.size()));
    }
  }
  std::vector<uint32_t> a_deg, a_off, p_deg, p_off;
  std::vector<double> a_x, a_y, p_x, p_y;
  dbsp_profile c{};
};

}  // namespace detail

// primitive: "all2all" | "p2p" (x = per-GPU payload bytes) | "dense" (x = density)
struct ProfileSample {
  std::string primitive;
  uint32_t degree = 1;
  double x = 0.0;
  double seconds = 0.0;
};

struct FitOptions {
  double exchange_overlap = 1.0;
  double replan_seconds = 0.0;
  double bytes_per_token_per_head = 256.0;
};

inline MachineProfile fit_profile(const std::vector<ProfileSample>& samples,
                                  const FitOptions& options = {}) {
  std::vector<dbsp_profile_sample> cs;
  cs.reserve(samples.size());
  for (const ProfileSample& s : samples) {
    uint32_t prim;
    if (s.primitive == "all2all")
      prim = 0;
    else if (s.primitive == "p2p")
      prim = 1;
    else if (s.primitive == "dense")
      prim = 2;
    else
      throw config_error("unknown profile primitive '" + s.primitive + "'");
    cs.push_back({prim, s.degree, s.x, s.seconds});
  }
  const size_t n = samples.size() + 1;
  std::vector<uint32_t> ad(n), ao(n + 1), pd(n), po(n + 1);
  std::vector<double> ax(n), ay(n), px(n), py(n);
  dbsp_profile_storage st{ad.data(), ao.data(), ax.data(), ay.data(),
                          pd.data(), po.data(), px.data(), py.data()};
  const dbsp_fit_options opt{options.exchange_overlap, options.replan_seconds,
                             options.bytes_per_token_per_head};
  dbsp_profile out{};
  detail::check(dbsp_fit_profile(cs.data(), uint32_t(cs.size()), &opt, &st, &out));
  MachineProfile p;
  for (uint32_t i = 0; i < out.num_all2all; ++i)
    p.all2all[ad[i]] = {std::vector<double>(ax.begin() + ao[i], ax.begin() + ao[i + 1]),
                        std::vector<double>(ay.begin() + ao[i], ay.begin() + ao[i + 1])};
  for (uint32_t i = 0; i < out.num_p2p; ++i)
    p.p2p[pd[i]] = {std::vector<double>(px.begin() + po[i], px.begin() + po[i + 1]),
                    std::vector<double>(py.begin() + po[i], py.begin() + po[i + 1])};
  p.dense_attn_seconds = out.dense_attn_seconds;
  p.launch_seconds = out.launch_seconds;
  p.exchange_overlap = out.exchange_overlap;
  p.replan_seconds = out.replan_seconds;
  p.bytes_per_token_per_head = out.bytes_per_token_per_head;
  return p;
}

struct LatencyBreakdown {
  double all2all_s = 0.0;
  double attn_compute_s = 0.0;
  double ring_p2p_exposed_s = 0.0;
  double imbalance_penalty_s = 0.0;
  double exchange_s = 0.0;
  double replan_s = 0.0;
  double total_s = 0.0;
  double attn_seconds() const { return attn_compute_s + ring_p2p_exposed_s + imbalance_penalty_s; }
};

struct MaskShape {
  uint32_t heads = 1;
  uint32_t q_blocks = 1;
  uint32_t kv_blocks = 1;
  uint32_t block_size = 1;
};

inline MaskShape mask_shape(const AttentionMaskSet& set) {
  return {set.num_heads(), set.num_q_blocks(), set.num_kv_blocks(), set.block_size()};
}

struct CallInputs {
  MaskShape shape;
  ParallelStrategy strategy;
  double density = 0.0;
  double rho = 1.0;
  ExchangeVolume exchange;
  bool charge_replan = false;
};

inline double exchange_payload_bytes(const MaskShape& shape, ParallelStrategy strategy,
                                     const ExchangeVolume& volume, const MachineProfile& profile) {
  return static_cast<double>(volume.token_payload) *
         (static_cast<double>(shape.heads) / strategy.ulysses) * profile.bytes_per_token_per_head;
}

namespace detail {
inline LatencyBreakdown from_c(const dbsp_latency& l) {
  return {l.all2all_s, l.attn_compute_s, l.ring_p2p_exposed_s, l.imbalance_penalty_s,
          l.exchange_s, l.replan_s, l.total_s};
}
}  // namespace detail

inline LatencyBreakdown predict_from_inputs(const CallInputs& in, const MachineProfile& profile) {
  const dbsp_call_inputs c{in.shape.heads, in.shape.q_blocks, in.shape.kv_blocks,
                           in.shape.block_size, detail::cs(in.strategy), in.density, in.rho,
                           {in.exchange.q_blocks_moved, in.exchange.kv_blocks_moved,
                            in.exchange.token_payload},
                           in.charge_replan ? 1 : 0};
  detail::ProfileView pv(profile);
  dbsp_latency out{};
  detail::check(dbsp_predict_from_inputs(&c, pv.get(), &out));
  return detail::from_c(out);
}

inline LatencyBreakdown predict_latency(const AttentionMaskSet& set, ParallelStrategy strategy,
                                        const PartitionPlan& plan, const MachineProfile& profile,
                                        bool charge_replan = false) {
  detail::check_dims(set, plan);
  detail::MaskView v(set);
  detail::ProfileView pv(profile);
  const dbsp_plan c = detail::cplan(plan);
  dbsp_latency out{};
  detail::check(dbsp_predict_latency(v.get(), detail::cs(strategy), &c, pv.get(),
                                     charge_replan ? 1 : 0, &out));
  return detail::from_c(out);
}

struct StrategyPrediction {
  ParallelStrategy strategy;
  PlanOutcome outcome;
  LatencyBreakdown latency;
};

inline std::vector<StrategyPrediction> predict_all(
    const AttentionMaskSet& set, const MachineProfile& profile, uint32_t total_gpus,
    const PlannerConfig& config, const std::map<ParallelStrategy, PartitionPlan>& prev_plans = {}) {
  detail::MaskView v(set);
  detail::ProfileView pv(profile);
  std::vector<dbsp_strategy> ps;
  std::vector<dbsp_plan> pp;
  for (const auto& [s, p] : prev_plans) {
    detail::check_dims(set, p);
    ps.push_back(detail::cs(s));
    pp.push_back(detail::cplan(p));
  }
  std::vector<PartitionPlan> plans(33, detail::sized_plan(set));
  std::vector<dbsp_plan> pc;
  for (PartitionPlan& p : plans) pc.push_back(detail::cplan(p));
  dbsp_prediction rows[33];
  uint32_t n = 0;
  const dbsp_planner_config cfg{config.reuse_threshold, config.exchange_reward};
  detail::check(dbsp_predict_all(v.get(), pv.get(), total_gpus, &cfg, ps.data(), pp.data(),
                                 uint32_t(ps.size()), rows, pc.data(), &n));
  std::vector<StrategyPrediction> out;
  for (uint32_t i = 0; i < n; ++i) {
    StrategyPrediction s;
    s.strategy = {rows[i].strategy.ulysses, rows[i].strategy.ring};
    s.outcome.plan = std::move(plans[i]);
    s.outcome.head_replanned = rows[i].outcome.head_replanned != 0;
    s.outcome.rho_pre = rows[i].outcome.rho_pre;
    s.outcome.rho_post = rows[i].outcome.rho_post;
    s.latency = detail::from_c(rows[i].latency);
    out.push_back(std::move(s));
  }
  return out;
}

#ifdef DBSP_HAVE_JSON
// Profile JSON (reference latency.hpp:318-379): stored as samples, re-fitted on load.
inline nlohmann::json profile_to_json(const MachineProfile& profile) {
  auto curves = [](const std::map<uint32_t, PiecewiseLinear>& t) {
    nlohmann::json a = nlohmann::json::array();
    for (const auto& [d, c] : t)
      for (size_t i = 0; i < c.xs.size(); ++i)
        a.push_back({{"degree", d}, {"payload_bytes", c.xs[i]}, {"seconds", c.ys[i]}});
    return a;
  };
  nlohmann::json j;
  j["all2all"] = curves(profile.all2all);
  j["p2p"] = curves(profile.p2p);
  j["dense"] = {{{"density", 0.0}, {"seconds", profile.launch_seconds}},
                {{"density", 1.0}, {"seconds", profile.launch_seconds + profile.dense_attn_seconds}}};
  j["exchange_overlap"] = profile.exchange_overlap;
  j["replan_seconds"] = profile.replan_seconds;
  j["bytes_per_token_per_head"] = profile.bytes_per_token_per_head;
  return j;
}

inline MachineProfile profile_from_json(const nlohmann::json& j,
                                        const std::string& origin = "profile") {
  try {
    std::vector<ProfileSample> samples;
    for (const char* prim : {"all2all", "p2p"})
      if (j.contains(prim))
        for (const auto& e : j.at(prim))
          samples.push_back({prim, e.at("degree").get<uint32_t>(),
                             e.at("payload_bytes").get<double>(), e.at("seconds").get<double>()});
    for (const auto& e : j.at("dense"))
      samples.push_back({"dense", 1, e.at("density").get<double>(), e.at("seconds").get<double>()});
    FitOptions o;
    o.exchange_overlap = j.value("exchange_overlap", 1.0);
    o.replan_seconds = j.value("replan_seconds", 0.0);
    o.bytes_per_token_per_head = j.value("bytes_per_token_per_head", 256.0);
    return fit_profile(samples, o);
  } catch (const nlohmann::json::exception& e) {
    throw parse_error(origin + ": invalid profile JSON: " + e.what());
  }
}

inline MachineProfile load_profile(const std::filesystem::path& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw io_error("cannot open " + path.string());
  std::stringstream ss;
  ss << f.rdbuf();
  nlohmann::json j;
  try {
    j = nlohmann::json::parse(ss.str());
  } catch (const nlohmann::json::exception& e) {
    throw parse_error(path.string() + ": invalid JSON: " + e.what());
  }
  return profile_from_json(j, path.string());
}

// Reference latency.hpp:377-379: the JSON above, pretty-printed, written
// atomically (a temp file in the same directory, then rename), io_error on
// failure.
inline void save_profile(const MachineProfile& profile, const std::filesystem::path& path) {
  const std::string text = profile_to_json(profile).dump(2) + "\n";
  std::filesystem::path tmp = path;
  tmp += ".tmp";
  {
    std::ofstream f(tmp, std::ios::binary | std::ios::trunc);
    if (!f) throw io_error("cannot open '" + tmp.string() + "' for writing");
    f.write(text.data(), std::streamsize(text.size()));
    if (!f) throw io_error("write failed for '" + tmp.string() + "'");
  }
  std::error_code ec;
  std::filesystem::rename(tmp, path, ec);
  if (ec) throw io_error("cannot rename '" + tmp.string() + "' to '" + path.string() + "': " + ec.message());
}
#endif

}  // namespace dbsp
