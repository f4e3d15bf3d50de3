"""Config E (BASELINE.json configs[4]): Wan2.1-14B 50 steps x 40 layers with
per-step / per-layer varying masks, exercising the dynamic U x R selection
(selector.hpp:55-75) per call.  Masks follow the reference ScheduleMasks chain
(simulator.hpp:53-113): layer seeds mix_seed(seed, layer), per-step flips
with mix_seed(seed, layer, step).  Reports the planner's per-call host time,
the chosen strategies, head replans and predicted latency.  CPU tool:
    python tests/config_e.py [steps] [layers] [flip] [profile.json]"""
import collections
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2511_23113_b200 as D  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    layers = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    flip = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
    prof_path = Path(sys.argv[4]) if len(sys.argv) > 4 else \
        ROOT / "paper_2511_23113_b200" / "profiles" / "b200_wan_measured.json"
    profile = D.MachineProfile.from_json(json.loads(prof_path.read_text()))
    base = D.GeneratorSpec(40, 512, 512, 64, "clustered", 0.15, 0.45, 1.0, 1)
    cur = []
    for layer in range(layers):
        sp = D.GeneratorSpec(**{**base.__dict__, "seed": D.mix_seed(base.seed, layer)})
        cur.append(D.generate_mask_set(sp))
    state = D.SelectorState(8)
    hist = collections.Counter()
    replans = 0
    total_pred = 0.0
    plan_s = 0.0
    rho = []
    for step in range(steps):
        for layer in range(layers):
            if step > 0 and flip > 0:
                cur[layer] = D.perturb_mask_set(cur[layer], flip, D.mix_seed(base.seed, layer, step))
            t0 = time.perf_counter()
            sel = D.select(layer, cur[layer], profile, D.PlannerConfig(), state)
            plan_s += time.perf_counter() - t0
            hist[str(sel.strategy)] += 1
            replans += sel.outcome.head_replanned
            total_pred += sel.latency.total_s
            rho.append(sel.outcome.rho_post)
    calls = steps * layers
    out = {"config": "E", "steps": steps, "layers": layers, "flip": flip, "calls": calls,
           "select_ms_per_call": round(plan_s / calls * 1e3, 3), "strategies": dict(hist),
           "head_replans": int(replans), "rho_post_mean": round(sum(rho) / len(rho), 4),
           "rho_post_max": round(max(rho), 4), "predicted_attention_s_total": round(total_pred, 4),
           "profile": prof_path.name}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
