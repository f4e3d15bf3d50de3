"""Per-tile clock64 timeline of K4 (DBSP_TRACE build) on the Wan layer.
GPU-box tool: rebuilds with -DDBSP_TRACE, runs once, prints per-event
latency statistics (cycles), restores the normal build."""
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
    flags = "-DDBSP_TRACE " + " ".join(sys.argv[1:])
    subprocess.run([sys.executable, str(ROOT / "paper_2511_23113_b200" / "build.py"), "-f"], check=True,
                   env=dict(os.environ, DBSP_NVCC_FLAGS=flags), capture_output=True)
    import torch
    import paper_2511_23113_b200 as D
    from paper_2511_23113_b200 import _lib
    from paper_2511_23113_b200.attention import AttentionSchedule
    B, T, E = 16, 256, 8
    buf = torch.zeros(B * T * E, dtype=torch.int64, device="cuda")
    fn = _lib.lib().dbsp_debug_set_trace
    fn.argtypes = [ctypes.c_void_p]
    fn(ctypes.c_void_p(buf.data_ptr()))
    H, S, d = 40, 32768, 128
    m = D.generate_mask_set(D.GeneratorSpec(H, S // 64, S // 64, 64, "clustered", 0.15, 0.45, 1.0, 1))
    q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    sc = AttentionSchedule().build(m, kv_tokens_global=S)
    out = torch.empty_like(q)
    for _ in range(3):
        sc.launch(q, k, v, out)
    torch.cuda.synchronize()
    tr = buf.view(B, T, E).cpu().numpy().astype(np.int64)
    fn(None)
    names = ["soft_start", "soft_end", "mma_S", "mma_PV", "soft_start_hi", "soft_end_hi", "load_K", "load_V"]
    stats = {}
    for b in range(B):
        t = tr[b]
        n = int((t[:, 0] > 0).sum())
        if n < 8:
            continue
        t = t[:n]
        soft = t[:, 1] - t[:, 0]
        wait_s = t[1:, 0] - t[:-1, 1]          # softmax idle waiting for the next S
        s_lat = t[:, 0] - t[:, 2]              # S issue (commit) -> softmax sees it
        pv_lag = t[:, 3] - t[:, 1]             # P arrive -> PV issued
        period = np.diff(t[:, 0])
        k_lead = t[:, 2] - t[:, 6]             # K load issued -> S issued
        for key, arr in [("softmax", soft), ("wait_for_S", wait_s), ("S_issue_to_soft", s_lat),
                         ("P_to_PV_issue", pv_lag), ("period", period), ("Kload_to_S_issue", k_lead)]:
            stats.setdefault(key, []).append(np.median(arr[2:]) if len(arr) > 4 else np.median(arr))
        if b < 2:
            print(f"block {b}: n={n}")
            base = t[0, 6]
            for j in range(min(n, 12)):
                print("  j=%2d " % j + " ".join(f"{nm}={int(t[j, e] - base):7d}" for e, nm in enumerate(names)))
    print(json.dumps({k: float(np.median(v)) for k, v in stats.items()}))
    subprocess.run([sys.executable, str(ROOT / "paper_2511_23113_b200" / "build.py"), "-f"], check=True,
                   capture_output=True)


if __name__ == "__main__":
    main()
