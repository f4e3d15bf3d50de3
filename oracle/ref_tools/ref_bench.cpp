// ORACLE tool — test / baseline infrastructure only.  Compiled against the
// UNMODIFIED reference headers into oracle/_ref/ref_bench; bench.py runs it
// as the reference CPU planner baseline (single thread, as the reference
// library is: it parallelises only compare/sweep, simulator.hpp:320,388).
//
// usage: ref_bench H Nq Nk pattern dmin dmax seed gpus reps profile.json [masks.bin]
// prints one JSON line: per-strategy plan_dual ms, select() ms per call, rho.
// With masks.bin, the generated set is also written there by the reference's
// own save_mask_set (DBSPMSK1): bench.py's reference arm takes its masks from
// it, so that arm never loads the product library.
#include <chrono>
#include <cstdio>
#include <string>

#include "dbsp/latency.hpp"
#include "dbsp/mask.hpp"
#include "dbsp/mask_io.hpp"
#include "dbsp/metrics.hpp"
#include "dbsp/planner.hpp"
#include "dbsp/selector.hpp"

using namespace dbsp;
using clk = std::chrono::steady_clock;

int main(int argc, char** argv) {
  if (argc < 11) {
    std::fprintf(stderr, "usage: ref_bench H Nq Nk pattern dmin dmax seed gpus reps profile.json\n");
    return 2;
  }
  GeneratorSpec sp;
  sp.num_heads = std::stoul(argv[1]);
  sp.num_q_blocks = std::stoul(argv[2]);
  sp.num_kv_blocks = std::stoul(argv[3]);
  sp.pattern = parse_pattern(argv[4]);
  sp.min_density = std::stod(argv[5]);
  sp.max_density = std::stod(argv[6]);
  sp.seed = std::stoull(argv[7]);
  const uint32_t gpus = std::stoul(argv[8]);
  const int reps = std::stoi(argv[9]);
  const MachineProfile prof = load_profile(argv[10]);
  const AttentionMaskSet set = generate_mask_set(sp);
  if (argc > 11) save_mask_set(set, argv[11]);

  std::string per = "{";
  bool first = true;
  for (ParallelStrategy s : enumerate_strategies(gpus)) {
    if (s.ulysses > set.num_heads() || s.ring > std::min(set.num_q_blocks(), set.num_kv_blocks()))
      continue;
    const auto t0 = clk::now();
    PlanOutcome oc;
    for (int i = 0; i < reps; ++i) oc = plan_dual(set, s, PlannerConfig{});
    const double ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count() / reps;
    char buf[256];
    std::snprintf(buf, sizeof(buf), "%s\"%s\": {\"plan_dual_ms\": %.6f, \"rho_pre\": %.17g, \"rho_post\": %.17g}",
                  first ? "" : ", ", to_string(s).c_str(), ms, oc.rho_pre, oc.rho_post);
    per += buf;
    first = false;
  }
  per += "}";
  const auto t0 = clk::now();
  Selection sel;
  for (int i = 0; i < reps; ++i) {
    SelectorState st(gpus);
    sel = select(0, set, prof, PlannerConfig{}, st);
  }
  const double sel_ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count() / reps;
  std::printf("{\"select_ms\": %.6f, \"selected\": \"%s\", \"rho_post\": %.17g, \"total_s\": %.17g, "
              "\"strategies\": %s, \"reps\": %d, \"threads\": 1}\n",
              sel_ms, to_string(sel.strategy).c_str(), sel.outcome.rho_post, sel.latency.total_s,
              per.c_str(), reps);
  return 0;
}
