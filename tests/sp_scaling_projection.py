"""Per-rank K4 times of every U x R split at G = 2, 4, 8, measured on one B200
(sp.time_ranks_on_one_gpu), for the CogVideoX (B), Wan (C) and HunyuanVideo
(D) layers, under the uniform USP plan and the db-SP plan.  The attention
critical path is sum over periods of the max over ranks; the selector's
modelled communication (Eq. 4 terms of the measured B200 profile) is added
beside it, not measured (one GPU).  GPU-box tool:
    python tests/sp_scaling_projection.py > out.json"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2511_23113_b200 as D  # noqa: E402
from paper_2511_23113_b200.attention import AttentionSchedule  # noqa: E402
from paper_2511_23113_b200.sp import measured_rho, time_ranks_on_one_gpu, time_scratch  # noqa: E402
from paper_2511_23113_b200.sp_bench import load_profile  # noqa: E402
from paper_2511_23113_b200.workloads import WORKLOADS  # noqa: E402


def crit(t):
    return float(sum(max(r) for r in t))


def main():
    names = sys.argv[1:] or ["cogvideox", "wan", "hunyuan"]
    out = {}
    for name in names:
        wl = WORKLOADS[name]
        masks = D.generate_mask_set(wl.spec())
        H, S, d = wl.heads, wl.tokens, wl.head_dim
        g = torch.Generator(device="cuda").manual_seed(1234)
        q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(3))
        sc = AttentionSchedule().build(masks, kv_tokens_global=S, head_dim=d)
        sc.upload()
        o = torch.empty_like(q)
        for _ in range(2):
            sc.launch(q, k, v, o)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            sc.launch(q, k, v, o)
        e1.record()
        torch.cuda.synchronize()
        one = e0.elapsed_time(e1) / 5
        scratch = time_scratch(q, k, v)
        prof = load_profile(name)
        res = {"1": {"attn_ms": round(one, 4)}}
        for G in (2, 4, 8):
            rows = {}
            for st in D.enumerate_strategies(G):
                if st.ulysses > H:
                    continue
                for bal in ("uniform", "dbsp"):
                    plan = D.default_plan(masks, st) if bal == "uniform" else D.plan_dual(masks, st).plan
                    t = time_ranks_on_one_gpu(q, k, v, masks, st, plan, scratch, reps=2)
                    lat = D.predict_latency(masks, st, plan, prof)
                    comm = (lat.all2all_s + lat.ring_p2p_exposed_s + lat.exchange_s) * 1e3
                    rows[f"{st}/{bal}"] = {"attn_ms": round(crit(t), 4), "rho_s_measured": round(measured_rho(t), 4),
                                           "rho_s_plan": round(D.imbalance_ratio(D.workload_table(masks, st, plan)), 4),
                                           "modelled_comm_ms": round(comm, 4)}
            bu = min((k_ for k_ in rows if k_.endswith("uniform")), key=lambda k_: rows[k_]["attn_ms"])
            bd = min((k_ for k_ in rows if k_.endswith("dbsp")), key=lambda k_: rows[k_]["attn_ms"])
            res[str(G)] = {"splits": rows, "best_uniform": bu, "best_dbsp": bd,
                           "speedup_attn": round(rows[bu]["attn_ms"] / rows[bd]["attn_ms"], 4),
                           "speedup_attn_plus_modelled_comm": round(
                               (rows[bu]["attn_ms"] + rows[bu]["modelled_comm_ms"]) /
                               (rows[bd]["attn_ms"] + rows[bd]["modelled_comm_ms"]), 4)}
        out[wl.name] = res
        del q, k, v, o, scratch
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
