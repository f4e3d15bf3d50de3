"""Interleaved A/B timing of K4 variants selected by an environment switch
read at launch time (e.g. DBSP_K4_SUB=32 vs 64), on one workload.  GPU-box
tool: python tests/ab_env_probe.py workload VAR val1 val2 ... [--rounds R]."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_23113_b200 as D  # noqa: E402
from paper_2511_23113_b200.attention import AttentionSchedule  # noqa: E402
from paper_2511_23113_b200.workloads import WORKLOADS  # noqa: E402


def main():
    args = sys.argv[1:]
    rounds = 5
    if "--rounds" in args:
        i = args.index("--rounds")
        rounds = int(args[i + 1])
        args = args[:i] + args[i + 2:]
    wl = WORKLOADS[args[0]]
    var, vals = args[1], args[2:]
    masks = D.generate_mask_set(wl.spec())
    S, H, d = wl.tokens, wl.heads, wl.head_dim
    g = torch.Generator(device="cuda").manual_seed(1234)
    q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(3))
    flop = 4.0 * 64 * 64 * d * D.total_blocks(masks)
    sc = AttentionSchedule().build(masks, kv_tokens_global=S, flags=1)
    sc.upload()
    outs = {}
    for val in vals:
        os.environ[var] = val
        o = torch.zeros_like(q)
        for _ in range(3):
            sc.launch(q, k, v, o)
        outs[val] = o
    torch.cuda.synchronize()
    base = outs[vals[0]].float()
    import ctypes
    from paper_2511_23113_b200 import _lib
    probe = _lib.lib().dbsp_debug_set_clock_probe
    probe.argtypes = [ctypes.c_void_p]
    cbuf = torch.zeros(4, dtype=torch.int64, device="cuda")
    mhz = {x: [] for x in vals}
    res = {x: [] for x in vals}
    for _ in range(rounds):
        for val in vals:
            os.environ[var] = val
            ts = []
            for _ in range(8):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                sc.launch(q, k, v, outs[val])
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[val].append(float(np.median(ts)))
            probe(ctypes.c_void_p(cbuf.data_ptr()))  # SM clock inside one more launch (CTA 0)
            sc.launch(q, k, v, outs[val])
            torch.cuda.synchronize()
            probe(None)
            c0, t0, c1, t1 = (int(x) for x in cbuf.cpu().tolist())
            if t1 > t0:
                mhz[val].append((c1 - c0) / (t1 - t0) * 1e3)
    out = {"workload": wl.name, "var": var}
    for val in vals:
        r = np.array(res[val])
        out[val] = {"ms_median": round(float(np.median(r)), 4), "ms_min_round": round(float(r.min()), 4),
                    "tflops": round(flop / float(np.median(r)) / 1e9, 1),
                    "mhz_cta0": round(float(np.median(mhz[val])), 1) if mhz[val] else None,
                    "mcycles": round(float(np.median(r)) * float(np.median(mhz[val])) / 1e3, 3) if mhz[val] else None,
                    "maxabs_vs_first": float((outs[val].float() - base).abs().max())}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
