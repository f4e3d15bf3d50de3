// C ABI over the host planner core (include/dbsp_b200.h).  Every entry point
// catches, records the message thread-locally and returns a status code that
// mirrors the reference exception class (error.hpp:10-44).
#include <cstring>
#include <new>
#include <string>

#include "../../include/dbsp_b200.h"
#include "capi_util.hpp"
#include "planner_device.hpp"
#include "core.hpp"

using namespace dbsp_core;

namespace dbsp_capi {

thread_local std::string g_last_error;

int record(int code, const char* what) {
  g_last_error = what ? what : "";
  return code;
}

}  // namespace dbsp_capi

using dbsp_capi::guard;

namespace {

MaskView view_of(const dbsp_mask_set* s) {
  if (!s) fail(kContract, "null mask set");
  return make_view(s->heads, s->num_heads, s->num_q_blocks, s->num_kv_blocks, s->block_size);
}

Strategy strat(dbsp_strategy s) { return Strategy{s.ulysses, s.ring}; }

void need(const void* p, const char* what) {
  if (!p) fail(kContract, std::string("null pointer: ") + what);
}

Plan plan_of(const MaskView& m, const dbsp_plan* p) {
  need(p, "plan");
  need(p->head_assignment, "plan.head_assignment");
  need(p->q_assignment, "plan.q_assignment");
  need(p->kv_assignment, "plan.kv_assignment");
  Plan out;
  out.head.assign(p->head_assignment, p->head_assignment + m.H);
  out.q.assign(p->q_assignment, p->q_assignment + m.nq);
  out.kv.assign(p->kv_assignment, p->kv_assignment + m.nk);
  return out;
}

void write_plan(const Plan& src, dbsp_plan* dst) {
  need(dst, "output plan");
  need(dst->head_assignment, "plan.head_assignment");
  need(dst->q_assignment, "plan.q_assignment");
  need(dst->kv_assignment, "plan.kv_assignment");
  std::memcpy(dst->head_assignment, src.head.data(), src.head.size() * sizeof(uint32_t));
  std::memcpy(dst->q_assignment, src.q.data(), src.q.size() * sizeof(uint32_t));
  std::memcpy(dst->kv_assignment, src.kv.data(), src.kv.size() * sizeof(uint32_t));
}

PlannerConfig cfg_of(const dbsp_planner_config* c) {
  PlannerConfig p;
  if (c) {
    p.reuse_threshold = c->reuse_threshold;
    p.exchange_reward = c->exchange_reward;
  }
  return p;
}

Profile profile_of(const dbsp_profile* p) {
  need(p, "profile");
  Profile out;
  auto curves = [](uint32_t n, const uint32_t* deg, const uint32_t* off, const double* xs,
                   const double* ys, std::map<uint32_t, Curve>& dst) {
    if (n == 0) return;
    need(deg, "profile degrees");
    need(off, "profile offsets");
    for (uint32_t i = 0; i < n; ++i) {
      Curve c;
      if (off[i + 1] < off[i]) fail(kContract, "profile offsets must be non-decreasing");
      c.xs.assign(xs + off[i], xs + off[i + 1]);
      c.ys.assign(ys + off[i], ys + off[i + 1]);
      dst[deg[i]] = std::move(c);
    }
  };
  curves(p->num_all2all, p->all2all_degrees, p->all2all_offsets, p->all2all_x, p->all2all_y,
         out.all2all);
  curves(p->num_p2p, p->p2p_degrees, p->p2p_offsets, p->p2p_x, p->p2p_y, out.p2p);
  out.dense_attn_seconds = p->dense_attn_seconds;
  out.launch_seconds = p->launch_seconds;
  out.exchange_overlap = p->exchange_overlap;
  out.replan_seconds = p->replan_seconds;
  out.bytes_per_token_per_head = p->bytes_per_token_per_head;
  return out;
}

void write_latency(const Latency& l, dbsp_latency* o) {
  if (!o) return;
  o->all2all_s = l.all2all;
  o->attn_compute_s = l.compute;
  o->ring_p2p_exposed_s = l.exposed;
  o->imbalance_penalty_s = l.imbalance;
  o->exchange_s = l.exchange;
  o->replan_s = l.replan;
  o->total_s = l.total;
}

void write_outcome(const Outcome& oc, dbsp_plan_outcome* o) {
  if (!o) return;
  o->head_replanned = oc.head_replanned ? 1 : 0;
  o->rho_pre = oc.rho_pre;
  o->rho_post = oc.rho_post;
}

}  // namespace

struct dbsp_selector {
  explicit dbsp_selector(uint32_t g) : state(g) {}
  Selector state;
};

extern "C" {

const char* dbsp_last_error(void) { return dbsp_capi::g_last_error.c_str(); }

const char* dbsp_version(void) {
  return "dbsp_b200 0.1 (sm_100a tcgen05/TMEM/TMA block-sparse attention; host planner)";
}

uint64_t dbsp_mix_seed(uint64_t base, uint64_t a, uint64_t b) { return mix_seed(base, a, b); }

int dbsp_generate_mask_set(const dbsp_generator_spec* spec, uint64_t* words_out) {
  return guard([&] {
    need(spec, "spec");
    need(words_out, "words_out");
    GenSpec g;
    g.H = spec->num_heads;
    g.nq = spec->num_q_blocks;
    g.nk = spec->num_kv_blocks;
    g.block_size = spec->block_size;
    g.pattern = spec->pattern;
    g.dmin = spec->min_density;
    g.dmax = spec->max_density;
    g.skew = spec->skew;
    g.seed = spec->seed;
    generate_masks(g, words_out);
  });
}

int dbsp_perturb_mask_set(const dbsp_mask_set* set, double flip_rate, uint64_t seed,
                          uint64_t* words_out) {
  return guard([&] {
    need(words_out, "words_out");
    perturb_masks(view_of(set), flip_rate, seed, words_out);
  });
}

int dbsp_total_blocks(const dbsp_mask_set* set, uint64_t* out) {
  return guard([&] {
    need(out, "out");
    *out = total_blocks(view_of(set));
  });
}

int dbsp_blocks_per_head(const dbsp_mask_set* set, uint64_t* out) {
  return guard([&] {
    need(out, "out");
    const std::vector<uint64_t> c = head_counts(view_of(set));
    std::memcpy(out, c.data(), c.size() * sizeof(uint64_t));
  });
}

int dbsp_density(const dbsp_mask_set* set, double* out) {
  return guard([&] {
    need(out, "out");
    *out = density(view_of(set));
  });
}

int dbsp_enumerate_strategies(uint32_t total_gpus, dbsp_strategy* out, uint32_t* count) {
  return guard([&] {
    need(out, "out");
    need(count, "count");
    const auto all = enumerate_strategies(total_gpus);
    for (size_t i = 0; i < all.size(); ++i) out[i] = dbsp_strategy{all[i].x, all[i].y};
    *count = uint32_t(all.size());
  });
}

int dbsp_validate_plan(const dbsp_mask_set* set, dbsp_strategy s, const dbsp_plan* plan) {
  return guard([&] {
    const MaskView m = view_of(set);
    need(plan, "plan");
    validate_plan(m, strat(s), plan->head_assignment, plan->q_assignment, plan->kv_assignment);
  });
}

int dbsp_default_plan(const dbsp_mask_set* set, dbsp_strategy s, dbsp_plan* out) {
  return guard([&] { write_plan(default_plan(view_of(set), strat(s)), out); });
}

int dbsp_workload_table(const dbsp_mask_set* set, dbsp_strategy s, const dbsp_plan* plan,
                        uint64_t* counts, uint32_t* periods) {
  return guard([&] {
    const MaskView m = view_of(set);
    need(plan, "plan");
    need(counts, "counts");
    const Table t = workload_table(m, strat(s), plan->head_assignment, plan->q_assignment,
                                   plan->kv_assignment);
    std::memcpy(counts, t.counts.data(), t.counts.size() * sizeof(uint64_t));
    if (periods) *periods = t.periods;
  });
}

int dbsp_imbalance_ratio(const uint64_t* counts, uint32_t periods, uint32_t gpus, double* out) {
  return guard([&] {
    need(out, "out");
    if (periods * gpus) need(counts, "counts");
    *out = imbalance_ratio(counts, periods, gpus);
  });
}

int dbsp_exchange_volume(const dbsp_mask_set* set, dbsp_strategy s, const dbsp_plan* plan,
                         dbsp_exchange* out) {
  return guard([&] {
    const MaskView m = view_of(set);
    need(plan, "plan");
    need(out, "out");
    validate_plan(m, strat(s), plan->head_assignment, plan->q_assignment, plan->kv_assignment);
    const Exchange e = exchange_volume(m, strat(s), plan->q_assignment, plan->kv_assignment);
    *out = dbsp_exchange{e.q_moved, e.kv_moved, e.payload};
  });
}

int dbsp_summed_grid(const dbsp_mask_set* set, uint64_t* grid_out) {
  return guard([&] {
    need(grid_out, "grid_out");
    const std::vector<uint64_t> g = summed_grid(view_of(set));
    std::memcpy(grid_out, g.data(), g.size() * sizeof(uint64_t));
  });
}

int dbsp_head_level_imbalance(const uint64_t* weights, const uint32_t* assignment, uint32_t n,
                              uint32_t x, double* out) {
  return guard([&] {
    need(out, "out");
    if (x < 1) fail(kConfig, "Ulysses degree must be >= 1");
    if (n) {
      need(weights, "weights");
      need(assignment, "assignment");
    }
    *out = head_level_imbalance(weights, assignment, n, x);
  });
}

int dbsp_partition_heads(const dbsp_mask_set* set, uint32_t x, uint32_t* out) {
  return guard([&] {
    need(out, "out");
    const MaskView m = view_of(set);
    const std::vector<uint32_t> a = partition_heads(m, x, nullptr);
    std::memcpy(out, a.data(), a.size() * sizeof(uint32_t));
  });
}

int dbsp_partition_blocks(const dbsp_mask_set* set, uint32_t y, double reward, uint32_t* q_out,
                          uint32_t* kv_out) {
  return guard([&] {
    need(q_out, "q_out");
    need(kv_out, "kv_out");
    std::vector<uint32_t> q, kv;
    partition_blocks(view_of(set), y, reward, nullptr, q, kv);
    std::memcpy(q_out, q.data(), q.size() * sizeof(uint32_t));
    std::memcpy(kv_out, kv.data(), kv.size() * sizeof(uint32_t));
  });
}

int dbsp_biased_greedy(const uint64_t* weights, uint32_t n, uint32_t y, double reward,
                       uint32_t* out) {
  return guard([&] {
    if (y < 1) fail(kConfig, "ring degree must be >= 1");
    if (n) {
      need(weights, "weights");
      need(out, "out");
    }
    const std::vector<uint32_t> a = biased_greedy(weights, n, y, reward);
    if (n) std::memcpy(out, a.data(), a.size() * sizeof(uint32_t));
  });
}

int dbsp_plan_dual(const dbsp_mask_set* set, dbsp_strategy s, const dbsp_planner_config* cfg,
                   const dbsp_plan* prev, dbsp_plan* out, dbsp_plan_outcome* outcome) {
  return guard([&] {
    const MaskView m = view_of(set);
    Plan prev_plan;
    if (prev) prev_plan = plan_of(m, prev);
    const Outcome oc = plan_dual(m, strat(s), cfg_of(cfg), prev ? &prev_plan : nullptr);
    write_plan(oc.plan, out);
    write_outcome(oc, outcome);
  });
}

int dbsp_brute_force_heads(const dbsp_mask_set* set, uint32_t x, uint32_t* out) {
  return guard([&] {
    need(out, "out");
    const std::vector<uint32_t> a = brute_force_heads(view_of(set), x);
    std::memcpy(out, a.data(), a.size() * sizeof(uint32_t));
  });
}

int dbsp_brute_force_blocks(const uint64_t* grid, uint32_t nq, uint32_t nk, uint32_t y,
                            uint32_t* q_out, uint32_t* kv_out, double* rho_out) {
  return guard([&] {
    need(grid, "grid");
    need(q_out, "q_out");
    need(kv_out, "kv_out");
    need(rho_out, "rho_out");
    std::vector<uint32_t> q, kv;
    brute_force_blocks(grid, nq, nk, y, q, kv, *rho_out);
    std::memcpy(q_out, q.data(), q.size() * sizeof(uint32_t));
    std::memcpy(kv_out, kv.data(), kv.size() * sizeof(uint32_t));
  });
}

int dbsp_fit_profile(const dbsp_profile_sample* samples, uint32_t n_samples,
                     const dbsp_fit_options* options, dbsp_profile_storage* st,
                     dbsp_profile* out) {
  return guard([&] {
    need(st, "storage");
    need(out, "out");
    if (n_samples) need(samples, "samples");
    std::vector<Sample> v(n_samples);
    for (uint32_t i = 0; i < n_samples; ++i)
      v[i] = Sample{samples[i].primitive, samples[i].degree, samples[i].x, samples[i].seconds};
    FitOptions o;
    if (options) {
      o.exchange_overlap = options->exchange_overlap;
      o.replan_seconds = options->replan_seconds;
      o.bytes_per_token_per_head = options->bytes_per_token_per_head;
    }
    const Profile p = fit_profile(v, o);
    auto dump = [](const std::map<uint32_t, Curve>& cs, uint32_t* deg, uint32_t* off, double* xs,
                   double* ys) {
      uint32_t i = 0, k = 0;
      off[0] = 0;
      for (const auto& [d, c] : cs) {
        deg[i] = d;
        for (size_t j = 0; j < c.xs.size(); ++j, ++k) {
          xs[k] = c.xs[j];
          ys[k] = c.ys[j];
        }
        off[++i] = k;
      }
      return i;
    };
    std::memset(out, 0, sizeof(*out));
    if (!p.all2all.empty()) {
      need(st->all2all_degrees, "storage.all2all");
      out->num_all2all =
          dump(p.all2all, st->all2all_degrees, st->all2all_offsets, st->all2all_x, st->all2all_y);
    }
    if (!p.p2p.empty()) {
      need(st->p2p_degrees, "storage.p2p");
      out->num_p2p = dump(p.p2p, st->p2p_degrees, st->p2p_offsets, st->p2p_x, st->p2p_y);
    }
    out->all2all_degrees = st->all2all_degrees;
    out->all2all_offsets = st->all2all_offsets;
    out->all2all_x = st->all2all_x;
    out->all2all_y = st->all2all_y;
    out->p2p_degrees = st->p2p_degrees;
    out->p2p_offsets = st->p2p_offsets;
    out->p2p_x = st->p2p_x;
    out->p2p_y = st->p2p_y;
    out->dense_attn_seconds = p.dense_attn_seconds;
    out->launch_seconds = p.launch_seconds;
    out->exchange_overlap = p.exchange_overlap;
    out->replan_seconds = p.replan_seconds;
    out->bytes_per_token_per_head = p.bytes_per_token_per_head;
  });
}

int dbsp_pwl_eval(const double* xs, const double* ys, uint32_t n, double x, double* out) {
  return guard([&] {
    need(out, "out");
    Curve c;
    if (n) {
      need(xs, "xs");
      need(ys, "ys");
      c.xs.assign(xs, xs + n);
      c.ys.assign(ys, ys + n);
    }
    *out = c.eval(x);
  });
}

int dbsp_predict_from_inputs(const dbsp_call_inputs* in, const dbsp_profile* profile,
                             dbsp_latency* out) {
  return guard([&] {
    need(in, "inputs");
    need(out, "out");
    CallInputs c;
    c.heads = in->heads;
    c.q_blocks = in->q_blocks;
    c.kv_blocks = in->kv_blocks;
    c.block_size = in->block_size;
    c.strategy = strat(in->strategy);
    c.density = in->density;
    c.rho = in->rho;
    c.exchange = Exchange{in->exchange.q_blocks_moved, in->exchange.kv_blocks_moved,
                          in->exchange.token_payload};
    c.charge_replan = in->charge_replan != 0;
    write_latency(predict_from_inputs(c, profile_of(profile)), out);
  });
}

int dbsp_predict_latency(const dbsp_mask_set* set, dbsp_strategy s, const dbsp_plan* plan,
                         const dbsp_profile* profile, int32_t charge_replan, dbsp_latency* out) {
  return guard([&] {
    need(out, "out");
    const MaskView m = view_of(set);
    const Plan p = plan_of(m, plan);
    write_latency(predict_latency(m, strat(s), p, profile_of(profile), charge_replan != 0), out);
  });
}

int dbsp_selector_create(uint32_t total_gpus, dbsp_selector** out) {
  return guard([&] {
    need(out, "out");
    *out = new dbsp_selector(total_gpus);
  });
}

void dbsp_selector_destroy(dbsp_selector* state) { delete state; }

int dbsp_selector_stored(const dbsp_selector* state, int64_t layer, int32_t* found,
                         dbsp_strategy* strategy, uint32_t* sizes, dbsp_plan* plan) {
  return guard([&] {
    need(state, "selector");
    need(found, "found");
    Strategy s;
    Plan p;
    *found = state->state.stored(layer, s, p) ? 1 : 0;
    if (!*found) return;
    if (strategy) *strategy = dbsp_strategy{s.x, s.y};
    if (sizes) {
      sizes[0] = uint32_t(p.head.size());
      sizes[1] = uint32_t(p.q.size());
      sizes[2] = uint32_t(p.kv.size());
    }
    if (plan) write_plan(p, plan);
  });
}

int dbsp_selector_store(dbsp_selector* state, int64_t layer, dbsp_strategy s,
                        const dbsp_plan* plan, const uint32_t* sizes) {
  return guard([&] {
    need(state, "selector");
    need(plan, "plan");
    need(sizes, "sizes");
    Plan p;
    p.head.assign(plan->head_assignment, plan->head_assignment + sizes[0]);
    p.q.assign(plan->q_assignment, plan->q_assignment + sizes[1]);
    p.kv.assign(plan->kv_assignment, plan->kv_assignment + sizes[2]);
    state->state.store(layer, strat(s), std::move(p));
  });
}

int dbsp_predict_all(const dbsp_mask_set* set, const dbsp_profile* profile, uint32_t total_gpus,
                     const dbsp_planner_config* cfg, const dbsp_strategy* prev_strategies,
                     const dbsp_plan* prev_plans, uint32_t n_prev, dbsp_prediction* out,
                     dbsp_plan* plans_out, uint32_t* count) {
  return guard([&] {
    need(out, "out");
    need(count, "count");
    const MaskView m = view_of(set);
    std::map<Strategy, Plan> prev;
    for (uint32_t i = 0; i < n_prev; ++i) prev[strat(prev_strategies[i])] = plan_of(m, &prev_plans[i]);
    const std::vector<Prediction> all = predict_all(m, profile_of(profile), total_gpus,
                                                    cfg_of(cfg), prev);
    for (size_t i = 0; i < all.size(); ++i) {
      out[i].strategy = dbsp_strategy{all[i].strategy.x, all[i].strategy.y};
      write_outcome(all[i].outcome, &out[i].outcome);
      write_latency(all[i].latency, &out[i].latency);
      if (plans_out) write_plan(all[i].outcome.plan, &plans_out[i]);
    }
    *count = uint32_t(all.size());
  });
}

int dbsp_select(dbsp_selector* state, int64_t layer, const dbsp_mask_set* set,
                const dbsp_profile* profile, const dbsp_planner_config* cfg,
                dbsp_strategy* strategy_out, dbsp_plan* plan_out,
                dbsp_plan_outcome* outcome_out, dbsp_latency* latency_out) {
  return guard([&] {
    need(state, "selector");
    const MaskView m = view_of(set);
    const Prediction p = select(state->state, layer, m, profile_of(profile), cfg_of(cfg));
    if (strategy_out) *strategy_out = dbsp_strategy{p.strategy.x, p.strategy.y};
    if (plan_out) write_plan(p.outcome.plan, plan_out);
    write_outcome(p.outcome, outcome_out);
    write_latency(p.latency, latency_out);
  });
}

namespace {
void write_selection(const Prediction& p, dbsp_strategy* strategy_out, dbsp_plan* plan_out,
                     dbsp_plan_outcome* outcome_out, dbsp_latency* latency_out) {
  if (strategy_out) *strategy_out = dbsp_strategy{p.strategy.x, p.strategy.y};
  if (plan_out) write_plan(p.outcome.plan, plan_out);
  write_outcome(p.outcome, outcome_out);
  write_latency(p.latency, latency_out);
}
}  // namespace

int dbsp_select_two_phase(dbsp_selector* state, int64_t layer, const dbsp_mask_set* set,
                          const dbsp_profile* profile, const dbsp_planner_config* cfg,
                          dbsp_strategy* strategy_out, dbsp_plan* plan_out,
                          dbsp_plan_outcome* outcome_out, dbsp_latency* latency_out) {
  return guard([&] {
    need(state, "selector");
    const MaskView m = view_of(set);
    const MaskStats st = mask_stats(m, true);
    auto host_tables = [&](const std::vector<TableJob>& jobs) {
      std::vector<Table> t;
      for (const TableJob& j : jobs)
        t.push_back(workload_table(m, j.s, j.plan->head.data(), j.plan->q.data(), j.plan->kv.data(), &st));
      return t;
    };
    write_selection(select_batched(state->state, layer, m, st, profile_of(profile), cfg_of(cfg), host_tables),
                    strategy_out, plan_out, outcome_out, latency_out);
  });
}

int dbsp_select_device(dbsp_selector* state, int64_t layer, const uint64_t* d_words, uint32_t heads,
                       uint32_t q_blocks, uint32_t kv_blocks, uint32_t block_size,
                       const dbsp_profile* profile, const dbsp_planner_config* cfg,
                       dbsp_strategy* strategy_out, dbsp_plan* plan_out,
                       dbsp_plan_outcome* outcome_out, dbsp_latency* latency_out, void* stream) {
  return guard([&] {
    need(state, "selector");
    need(d_words, "device mask words");
    if (q_blocks == 0 || kv_blocks == 0) fail(kConfig, "BlockMask dimensions must be positive");
    if (heads == 0) fail(kConfig, "mask set needs at least one head");
    if (block_size == 0) fail(kConfig, "block_size must be positive");
    MaskView m;  // dimensions only: every mask-dependent integer comes from the GPU
    m.H = heads;
    m.nq = q_blocks;
    m.nk = kv_blocks;
    m.block_size = block_size;
    m.wpr = (size_t(kv_blocks) + 63) / 64;
    const MaskStats st = dbsp_device_planner::mask_stats(d_words, heads, q_blocks, kv_blocks, stream);
    auto dev_tables = [&](const std::vector<TableJob>& jobs) {
      return dbsp_device_planner::workload_tables(d_words, m, st, jobs, stream);
    };
    write_selection(select_batched(state->state, layer, m, st, profile_of(profile), cfg_of(cfg), dev_tables),
                    strategy_out, plan_out, outcome_out, latency_out);
  });
}

}  // extern "C"
