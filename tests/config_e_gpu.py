"""Config E on the GPU (BASELINE.json configs[4]): the Wan2.1-14B
50-step x 40-layer sweep with per-step / per-layer varying masks
(ScheduleMasks chain, simulator.hpp:53-113).  For every call the host runs
select() (selector.hpp:55-75) on the live masks, then every rank's K4 launches
of the chosen U x R split and plan are timed on this one B200
(sp.time_ranks_on_one_gpu).  The same call is also timed under the static
best uniform USP split (picked by measurement on call 0).  Reports the measured
attention critical path (sum over periods of the max over ranks) for both, the
measured rho_s, the selector's modelled communication for the chosen split,
and the per-call planning time.  GPU-box tool: python tests/config_e_gpu.py [steps] [layers] [flip] > out.json"""
import collections
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_23113_b200 as D  # noqa: E402
from paper_2511_23113_b200.sp import measured_rho, time_ranks_on_one_gpu, time_scratch  # noqa: E402


def crit(t):
    return float(sum(max(row) for row in t))


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    layers = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    flip = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
    G = 8
    prof_path = ROOT / "paper_2511_23113_b200" / "profiles" / "b200_wan_measured.json"
    profile = D.MachineProfile.from_json(json.loads(prof_path.read_text()))
    base = D.GeneratorSpec(40, 512, 512, 64, "clustered", 0.15, 0.45, 1.0, 1)
    cur = [D.generate_mask_set(D.GeneratorSpec(**{**base.__dict__, "seed": D.mix_seed(base.seed, l)}))
           for l in range(layers)]
    S, H, d = 32768, 40, 128
    g = torch.Generator(device="cuda").manual_seed(1234)
    q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(3))
    reps = 2
    scratch = time_scratch(q, k, v)
    # static best uniform split, chosen by measurement on call 0
    uni = {}
    for st in D.enumerate_strategies(G):
        uni[str(st)] = crit(time_ranks_on_one_gpu(q, k, v, cur[0], st, D.default_plan(cur[0], st), scratch, reps))
    best_uniform = min(uni, key=uni.get)
    st_uni = D.parse_strategy(best_uniform)

    state = D.SelectorState(G)
    host_state = D.SelectorState(G)
    hist = collections.Counter()
    rec = {"dbsp_ms": [], "uniform_ms": [], "rho_dbsp": [], "rho_uniform": [], "select_ms": [],
           "modelled_comm_ms": [], "replans": 0}
    for step in range(steps):
        for layer in range(layers):
            if step > 0 and flip > 0:
                cur[layer] = D.perturb_mask_set(cur[layer], flip, D.mix_seed(base.seed, layer, step))
            m = cur[layer]
            # the GPU selector on the live mask words (H2D of the words included)
            t0 = time.perf_counter()
            words = torch.from_numpy(np.ascontiguousarray(m.words).view(np.int64)).cuda()
            sel = D.select_device(layer, words, m.num_kv_blocks, profile, D.PlannerConfig(), state)
            rec["select_ms"].append((time.perf_counter() - t0) * 1e3)
            if step < 2:  # the host selector agrees bit for bit
                ref = D.select(layer, m, profile, D.PlannerConfig(), host_state)
                assert str(ref.strategy) == str(sel.strategy) and ref.latency == sel.latency
            hist[str(sel.strategy)] += 1
            rec["replans"] += int(sel.outcome.head_replanned)
            lat = sel.latency
            rec["modelled_comm_ms"].append((lat.all2all_s + lat.ring_p2p_exposed_s + lat.exchange_s) * 1e3)
            td = time_ranks_on_one_gpu(q, k, v, m, sel.strategy, sel.outcome.plan, scratch, reps)
            tu = time_ranks_on_one_gpu(q, k, v, m, st_uni, D.default_plan(m, st_uni), scratch, reps)
            rec["dbsp_ms"].append(crit(td))
            rec["uniform_ms"].append(crit(tu))
            rec["rho_dbsp"].append(measured_rho(td))
            rec["rho_uniform"].append(measured_rho(tu))
    a = {k_: np.asarray(v_) for k_, v_ in rec.items() if isinstance(v_, list)}
    res = {
        "config": "E", "steps": steps, "layers": layers, "flip": flip, "calls": steps * layers,
        "gpus_simulated": G, "profile": prof_path.name,
        "static_uniform_split": best_uniform, "uniform_call0_ms": {k_: round(v_, 4) for k_, v_ in uni.items()},
        "strategies_selected": dict(hist), "head_replans": rec["replans"],
        "attn_critical_path_total_s": {"dbsp_dynamic": round(a["dbsp_ms"].sum() / 1e3, 4),
                                       "uniform_static": round(a["uniform_ms"].sum() / 1e3, 4)},
        "speedup_dbsp_vs_uniform": round(float(a["uniform_ms"].sum() / a["dbsp_ms"].sum()), 4),
        "per_call_ms": {"dbsp_mean": round(float(a["dbsp_ms"].mean()), 4),
                        "uniform_mean": round(float(a["uniform_ms"].mean()), 4)},
        "rho_s_measured": {"dbsp_mean": round(float(a["rho_dbsp"].mean()), 4),
                           "dbsp_max": round(float(a["rho_dbsp"].max()), 4),
                           "uniform_mean": round(float(a["rho_uniform"].mean()), 4)},
        "select_ms_per_call": {"path": "dbsp_select_device (checked equal to the host select on the first 2 steps)",
                               "mean": round(float(a["select_ms"].mean()), 3),
                               "p95": round(float(np.percentile(a["select_ms"], 95)), 3)},
        "modelled_comm_ms_mean": round(float(a["modelled_comm_ms"].mean()), 4),
        "note": "kernel times measured per (period, rank) on one B200; communication not measured "
                "(one GPU) -- modelled_comm_ms is the selector's Eq. 4 comm term for the chosen split",
    }
    print(json.dumps(res))


if __name__ == "__main__":
    main()
