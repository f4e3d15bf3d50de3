"""Times the CTA-pair split-KV kernel (schedule flags 1|8|16|128,
attn_kernel_pd.cuh) against the default K4 on one workload, for each
DBSP_PD_POLY setting (one subprocess each: the setting is read once), and
checks it against the default kernel's output.
GPU-box tool: python tests/pd_probe.py [workload] [polys]"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def one(workload):
    sys.path.insert(0, str(ROOT))
    import torch
    import paper_2511_23113_b200 as D
    from paper_2511_23113_b200.attention import AttentionSchedule
    from paper_2511_23113_b200.workloads import WORKLOADS
    wl = WORKLOADS[workload]
    masks = D.generate_mask_set(wl.spec())
    S, H, d = wl.tokens, wl.heads, wl.head_dim
    g = torch.Generator(device="cuda").manual_seed(1234)
    q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(3))
    flop = 4.0 * 64 * 64 * d * D.total_blocks(masks)
    res = {}
    outs = {}
    for name, flags in (("default", 1), ("pd", 1 | 8 | 16 | 128), ("default2", 1), ("pd2", 1 | 8 | 16 | 128)):
        sc = AttentionSchedule().build(masks, kv_tokens_global=S, flags=flags)
        sc.upload()
        o = torch.empty_like(q)
        for _ in range(3):
            sc.launch(q, k, v, o)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sc.launch(q, k, v, o)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        st = sc.stats()
        res[name] = {"ms_median": round(ts[5], 4), "ms_min": round(ts[0], 4),
                     "tflops": round(flop / ts[5] / 1e9, 1), "tile_visits": st["tile_visits"]}
        outs[name[:2]] = o
    res["max_abs_vs_default"] = float((outs["pd"].float() - outs["de"].float()).abs().max())
    return res


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        print("RESULT " + json.dumps(one(sys.argv[2])))
        sys.exit(0)
    workload = sys.argv[1] if len(sys.argv) > 1 else "wan"
    polys = sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "1", "2", "3"]
    for pn in polys:
        env = dict(os.environ, DBSP_PD_POLY=pn)
        r = subprocess.run([sys.executable, __file__, "--one", workload], env=env, capture_output=True, text=True)
        line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
        print(json.dumps({"workload": workload, "poly": int(pn),
                          **(json.loads(line[0][7:]) if line else {"error": r.stderr[-1500:]})}), flush=True)
