"""Per-CTA start/end (globaltimer) and SM id of one K4 launch on the Wan
layer (DBSP_TRACE_CTA build): occupancy over time, per-item cost vs KV
count, and the tail.  GPU-box tool: python tests/trace_cta.py [sched_flags [workload]]"""
import ctypes
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    sched_flags = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    workload = sys.argv[2] if len(sys.argv) > 2 else "wan"
    subprocess.run([sys.executable, str(ROOT / "paper_2511_23113_b200" / "build.py"), "-f"], check=True,
                   env=dict(os.environ, DBSP_NVCC_FLAGS="-DDBSP_TRACE_CTA"), capture_output=True)
    import torch
    import paper_2511_23113_b200 as D
    from paper_2511_23113_b200 import _lib
    from paper_2511_23113_b200.attention import AttentionSchedule
    from paper_2511_23113_b200.workloads import WORKLOADS
    wl = WORKLOADS[workload]
    H, S, d = wl.heads, wl.tokens, wl.head_dim
    m = D.generate_mask_set(wl.spec())
    q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    sc = AttentionSchedule().build(m, kv_tokens_global=S, flags=sched_flags)
    items, _ = sc.download()
    n = len(items)
    buf = torch.zeros(max(4 * n, 16 * 256 * 8), dtype=torch.int64, device="cuda")
    fn = _lib.lib().dbsp_debug_set_trace
    fn.argtypes = [ctypes.c_void_p]
    out = torch.empty_like(q)
    for _ in range(2):
        sc.launch(q, k, v, out)
    fn(ctypes.c_void_p(buf.data_ptr()))
    sc.launch(q, k, v, out)
    torch.cuda.synchronize()
    fn(None)
    tr = buf[:4 * n].view(n, 4).cpu().numpy()
    t0 = tr[:, 0].min()
    st, en, sm = tr[:, 0] - t0, tr[:, 1] - t0, tr[:, 2]
    dur = en - st
    wall = en.max()
    cnt = items[:, 4].astype(np.int64)
    if sched_flags & 128:  # CTA-pair kernel: count in 128-key steps
        cnt = (cnt + 1) // 2
    # concurrency over time
    grid = np.linspace(0, wall, 200)
    conc = [(np.sum((st <= x) & (en > x))) for x in grid]
    per_tile = dur / np.maximum(cnt, 1)
    order = np.argsort(cnt)
    dec = np.array_split(order, 10)
    res = {
        "wall_us": wall / 1e3, "items": n, "sms": int(len(np.unique(sm))),
        "sum_item_us_per_slot": float(dur.sum() / 1e3 / (74 if sched_flags & 128 else 2 * 148)),
        "mean_concurrency": float(np.mean(conc)), "conc_profile": [int(c) for c in conc[::10]],
        "tail_us_last_10pct_items_start": float((wall - np.percentile(st, 90)) / 1e3),
        "ns_per_tile_by_count_decile": [[int(cnt[i].mean()), float(np.median(per_tile[i]))] for i in dec],
        "fixed_ns_fit": None,
        "sm_clock_mhz_in_kernel": float(np.median(tr[:, 3] / np.maximum(dur, 1)) * 1e3),
    }
    # Per SM: time with fewer than 2 resident CTAs (between the first start
    # and the last end on that SM), and the end -> next start gaps.
    lows, gaps = [], []
    for s_id in np.unique(sm):
        idx = np.where(sm == s_id)[0]
        ev = sorted([(st[i], 1) for i in idx] + [(en[i], -1) for i in idx])
        cur, last_t, low = 0, ev[0][0], 0
        for t, dlt in ev:
            if cur < 2:
                low += t - last_t
            cur += dlt
            last_t = t
        lows.append(low / max(1, en[idx].max() - st[idx].min()))
        ends = np.sort(en[idx])
        starts = np.sort(st[idx])
        for e in ends[:-2]:
            nxt = starts[starts >= e]
            if len(nxt):
                gaps.append(nxt[0] - e)
    res["per_sm_frac_time_below_2_ctas"] = float(np.median(lows))
    res["cta_turnover_gap_ns_median"] = float(np.median(gaps)) if gaps else None
    res["cta_turnover_gap_ns_p90"] = float(np.percentile(gaps, 90)) if gaps else None
    A = np.vstack([cnt, np.ones_like(cnt)]).T.astype(np.float64)
    coef, *_ = np.linalg.lstsq(A, dur.astype(np.float64), rcond=None)
    res["fixed_ns_fit"] = {"ns_per_tile": float(coef[0]), "ns_fixed": float(coef[1])}
    cyc, *_ = np.linalg.lstsq(A, tr[:, 3].astype(np.float64), rcond=None)
    res["fixed_cycles_fit"] = {"cycles_per_step": float(cyc[0]), "cycles_fixed": float(cyc[1])}
    print(json.dumps(res))
    subprocess.run([sys.executable, str(ROOT / "paper_2511_23113_b200" / "build.py"), "-f"], check=True,
                   capture_output=True)


if __name__ == "__main__":
    main()
