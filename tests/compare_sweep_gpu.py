"""Measured compare / sweep harness: the reference
simulator's `compare` and `sweep` (simulator.hpp:283-415) with the analytic
attention term replaced by K4 times measured on one B200.

A schedule of masks (ScheduleMasks chain, simulator.hpp:53-113: layer seeds
mix_seed(seed, layer), per-step flips mix_seed(seed, layer, step)) is replayed
under every policy:
  fixed strategy, unbalanced (default plan)  -- uniform USP
  fixed strategy, balanced (plan_dual with the per-layer previous plan, P_s reuse)
  dynamic (select() per call)
For each call the plan's per-rank kernels are timed (sp.time_ranks_on_one_gpu;
critical path = sum over periods of the max over ranks) and the Eq. 4
communication terms of the same plan come from the B200 profile
(predict_latency: all-to-all + exposed ring p2p + balancing exchange).  The
sweep varies P_s or R_b under the dynamic policy, like simulator.hpp `sweep`.
Speedups follow the reference: fixed cells against their own unbalanced
strategy, the dynamic row against the best unbalanced one.
GPU-box tool: python tests/compare_sweep_gpu.py [steps] [layers] [flip] > out.json"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_23113_b200 as D  # noqa: E402
from paper_2511_23113_b200.sp import time_ranks_on_one_gpu, time_scratch  # noqa: E402


def crit(t):
    return float(sum(max(r) for r in t))


def comm_s(lat):
    return lat.all2all_s + lat.ring_p2p_exposed_s + lat.exchange_s


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    layers = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    flip = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
    G = 8
    prof = D.MachineProfile.from_json(json.loads(
        (ROOT / "paper_2511_23113_b200" / "profiles" / "b200_wan_measured.json").read_text()))
    base = D.GeneratorSpec(40, 512, 512, 64, "clustered", 0.15, 0.45, 1.0, 1)
    # the mask schedule, materialised once
    sched = []
    cur = [D.generate_mask_set(D.GeneratorSpec(**{**base.__dict__, "seed": D.mix_seed(base.seed, l)}))
           for l in range(layers)]
    for step in range(steps):
        if step > 0 and flip > 0:
            cur = [D.perturb_mask_set(m, flip, D.mix_seed(base.seed, l, step)) for l, m in enumerate(cur)]
        sched.append(list(cur))
    S, H, d = 32768, 40, 128
    g = torch.Generator(device="cuda").manual_seed(1234)
    q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(3))
    scratch = time_scratch(q, k, v)
    cache = {}

    def measured(masks, st, plan):
        key = (id(masks), str(st), plan.head_assignment.tobytes(), plan.q_assignment.tobytes(),
               plan.kv_assignment.tobytes())
        if key not in cache:
            cache[key] = crit(time_ranks_on_one_gpu(q, k, v, masks, st, plan, scratch, reps=1)) / 1e3
        return cache[key]

    def run_policy(mode, st=None, balanced=False, cfg=None):
        cfg = cfg or D.PlannerConfig()
        state = D.SelectorState(G)
        prev = {}
        attn = comm = 0.0
        replans = 0
        xbytes = 0
        rho = []
        for step in range(steps):
            for layer in range(layers):
                m = sched[step][layer]
                if mode == "dynamic":
                    sel = D.select(layer, m, prof, cfg, state)
                    s_, plan, oc = sel.strategy, sel.outcome.plan, sel.outcome
                elif balanced:
                    oc = D.plan_dual(m, st, cfg, prev.get(layer))
                    s_, plan = st, oc.plan
                    prev[layer] = plan
                else:
                    s_, plan, oc = st, D.default_plan(m, st), None
                replans += int(bool(oc and oc.head_replanned and step > 0))
                attn += measured(m, s_, plan)
                lat = D.predict_latency(m, s_, plan, prof)
                comm += comm_s(lat)
                ex = D.exchange_volume(m, s_, plan)
                xbytes += ex.token_payload * H * d * 2  # balancing moves, all heads, bf16
                rho.append(D.imbalance_ratio(D.workload_table(m, s_, plan)))
        return {"attn_s_measured": round(attn, 6), "comm_s_modelled": round(comm, 6),
                "total_s": round(attn + comm, 6), "replans": replans, "exchange_bytes": int(xbytes),
                "mean_rho_s": round(float(np.mean(rho)), 4)}

    cells = {}
    for st in D.enumerate_strategies(G):
        for balanced in (False, True):
            cells[f"{st}/{'balanced' if balanced else 'unbalanced'}"] = run_policy("fixed", st, balanced)
    cells["dynamic"] = run_policy("dynamic")
    best_unb = min((c for k_, c in cells.items() if k_.endswith("unbalanced")), key=lambda c: c["total_s"])
    for key, c in cells.items():
        base_c = best_unb if key == "dynamic" else cells[key.split("/")[0] + "/unbalanced"]
        c["speedup_total"] = round(base_c["total_s"] / c["total_s"], 4)
        c["speedup_attn"] = round(base_c["attn_s_measured"] / c["attn_s_measured"], 4)
    sweep = {"Ps": {}, "Rb": {}}
    for ps in (1.0, 1.05, 1.1, 1.3, 2.0):
        sweep["Ps"][str(ps)] = run_policy("dynamic", cfg=D.PlannerConfig(reuse_threshold=ps))
    for rb in (0.0, 0.25, 1.0, float("inf")):
        sweep["Rb"][str(rb)] = run_policy("dynamic", cfg=D.PlannerConfig(exchange_reward=rb))
    print(json.dumps({"schedule": {"steps": steps, "layers": layers, "flip": flip, "gpus": G,
                                   "layer_shape": "wan2.1-14b-480p-C"},
                      "compare": cells, "sweep": sweep,
                      "note": "attention: per-rank K4 times measured on one B200 (critical path); "
                              "communication: Eq. 4 terms of the B200 profile (not measured: one GPU)"}))


if __name__ == "__main__":
    main()
