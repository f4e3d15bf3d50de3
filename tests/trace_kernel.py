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
    args = sys.argv[1:]
    sched_flags = 1
    if args[:1] == ["--sched"]:
        sched_flags = int(args[1])
        args = args[2:]
    fine = args[:1] == ["--fine"]
    if fine:
        args = args[1:] + ["-DDBSP_TRACE_FINE"]
    workload = "wan"
    if args[:1] == ["--workload"]:
        workload = args[1]
        args = args[2:]
    fine1 = args[:1] == ["--fine1"]
    if fine1:
        args = args[1:] + ["-DDBSP_TRACE_FINE1"]
        if args[:1] == ["--warp"]:
            args = args[2:] + [f"-DDBSP_TRACE_WARP={args[1]}"]
    fine2 = args[:1] == ["--fine2"]
    if fine2:
        args = args[1:] + ["-DDBSP_TRACE_FINE2"]
    exps_mode = args[:1] == ["--exps"]
    if exps_mode:
        args = args[1:] + ["-DDBSP_TRACE_EXPS"]
    mma = args[:1] == ["--mma"]
    if mma:
        args = args[1:] + ["-DDBSP_TRACE_MMA"]
    flags = "-DDBSP_TRACE " + " ".join(args)
    subprocess.run([sys.executable, str(ROOT / "paper_2511_23113_b200" / "build.py"), "-f"], check=True,
                   env=dict(os.environ, DBSP_NVCC_FLAGS=flags), capture_output=True)
    import torch
    import paper_2511_23113_b200 as D
    from paper_2511_23113_b200 import _lib
    from paper_2511_23113_b200.attention import AttentionSchedule
    B, T, E = (296, 128, 8) if exps_mode else (16, 256, 8)
    buf = torch.zeros(B * T * E, dtype=torch.int64, device="cuda")
    fn = _lib.lib().dbsp_debug_set_trace
    fn.argtypes = [ctypes.c_void_p]
    fn(ctypes.c_void_p(buf.data_ptr()))
    from paper_2511_23113_b200.workloads import WORKLOADS
    wl = WORKLOADS[workload]
    H, S, d = wl.heads, wl.tokens, wl.head_dim
    m = D.generate_mask_set(wl.spec())
    q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    sc = AttentionSchedule().build(m, kv_tokens_global=S, flags=sched_flags)
    out = torch.empty_like(q)
    for _ in range(3):
        sc.launch(q, k, v, out)
    torch.cuda.synchronize()
    tr = buf.view(B, T, E).cpu().numpy().astype(np.int64)
    fn(None)
    if mma:
        names = ["Sfree", "QK_t+2_issued", "Pfull", "Vfull", "PV_issued", "Kfull_t+2"]
        for b in (0, 2):
            t = tr[b].astype(np.int64)
            n = int((t[:, 4] > 0).sum())
            base = t[0, 2]
            print(f"block {b}: steps={n}")
            for j in range(min(n, 14)):
                print("  t=%2d " % j + " ".join(f"{nm}={int(t[j, e] - base):7d}" for e, nm in enumerate(names)))
        subprocess.run([sys.executable, str(ROOT / "paper_2511_23113_b200" / "build.py"), "-f"], check=True,
                       capture_output=True)
        return
    if fine2:
        stats = {}
        for b in range(B):
            t = tr[b].astype(np.int64)
            n = int((t[:, 0] > 0).sum())
            if n < 8:
                continue
            t = t[2:n]
            ends = t[:, 4:8]
            ok = (ends > 0).all(axis=1)
            ends = ends[ok]
            first = ends.min(axis=1)
            for w in range(4):
                stats.setdefault(f"warp{w}_after_first", []).append(float(np.median(ends[:, w] - first)))
            stats.setdefault("last_minus_first", []).append(float(np.median(ends.max(axis=1) - first)))
            stats.setdefault("last_is_warp", []).append(float(np.bincount(ends.argmax(axis=1), minlength=4).argmax()))
        print(json.dumps({k: float(np.median(v)) for k, v in stats.items()}))
        subprocess.run([sys.executable, str(ROOT / "paper_2511_23113_b200" / "build.py"), "-f"], check=True,
                       capture_output=True)
        return
    if exps_mode:
        exps_overlap_report(tr)
        subprocess.run([sys.executable, str(ROOT / "paper_2511_23113_b200" / "build.py"), "-f"], check=True,
                       capture_output=True)
        return
    if fine1:
        stats = {}
        for b in range(B):
            t = tr[b].astype(np.int64)
            n = int((t[:, 0] > 0).sum())
            if n < 8:
                continue
            t = t[2:n]
            dense = t[:, 4] > 0  # steps where this warp's rows were dense
            t = t[dense]
            for key, arr in [("ld_S", t[:, 4] - t[:, 0]), ("max", t[:, 5] - t[:, 4]),
                             ("exps", t[:, 6] - t[:, 5]), ("store_wait", t[:, 7] - t[:, 6]),
                             ("fence_arrive", t[:, 1] - t[:, 7]), ("softmax", t[:, 1] - t[:, 0]),
                             ("wait_next_S", t[1:, 0] - t[:-1, 1]), ("period", np.diff(t[:, 0])),
                             ("P_to_PV_issued", t[:, 3] - t[:, 1]),
                             ("S_issued_to_soft_start", t[:, 0] - t[:, 2])]:
                stats.setdefault(key, []).append(float(np.median(arr)))
        print(json.dumps({k: float(np.median(v)) for k, v in stats.items()}))
        subprocess.run([sys.executable, str(ROOT / "paper_2511_23113_b200" / "build.py"), "-f"], check=True,
                       capture_output=True)
        return
    if sched_flags & 8 and fine:
        fine_report(tr)
        subprocess.run([sys.executable, str(ROOT / "paper_2511_23113_b200" / "build.py"), "-f"], check=True,
                       capture_output=True)
        return
    if sched_flags & 8:
        duo_report(tr)
        subprocess.run([sys.executable, str(ROOT / "paper_2511_23113_b200" / "build.py"), "-f"], check=True,
                       capture_output=True)
        return
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


def exps_overlap_report(tr):
    """DBSP_TRACE_EXPS: how much of one CTA's exp loop overlaps the exp loop of
    the other CTA's softmax warp on the same SM sub-partition (1 = lockstep,
    0 = perfectly staggered), and the exp-loop length when overlapped vs alone."""
    B, T, _ = tr.shape
    hdr = tr[:, T - 1, :]
    by_sm = {}
    for b in range(B):
        if hdr[b, 4] == 0 and b > 0:
            continue
        by_sm.setdefault(int(hdr[b, 4]), []).append(b)
    fr, len_ov, len_alone = [], [], []
    for sm, blocks in by_sm.items():
        if len(blocks) != 2:
            continue
        a, c = blocks
        for wa in range(4):
            smsp = int(hdr[a, wa]) % 4
            wc = [w for w in range(4) if int(hdr[c, w]) % 4 == smsp]
            if not wc:
                continue
            ia = [(int(tr[a, j, 2 * wa]), int(tr[a, j, 2 * wa + 1])) for j in range(T - 1) if tr[a, j, 2 * wa] > 0]
            ic = [(int(tr[c, j, 2 * wc[0]]), int(tr[c, j, 2 * wc[0] + 1])) for j in range(T - 1)
                  if tr[c, j, 2 * wc[0]] > 0]
            if len(ia) < 8 or len(ic) < 8:
                continue
            t0, t1 = max(ia[0][0], ic[0][0]), min(ia[-1][1], ic[-1][1])
            for s0, s1 in ia:
                if s0 < t0 or s1 > t1 or s1 <= s0:
                    continue
                ov = sum(max(0, min(s1, e1) - max(s0, e0)) for e0, e1 in ic)
                fr.append(ov / (s1 - s0))
                (len_ov if ov / (s1 - s0) > 0.5 else len_alone).append(s1 - s0)
    print(json.dumps({"pairs_measured": len(fr), "overlap_frac_median": float(np.median(fr)) if fr else None,
                      "overlap_frac_mean": float(np.mean(fr)) if fr else None,
                      "frac_mostly_overlapped": float(np.mean(np.array(fr) > 0.5)) if fr else None,
                      "exps_cycles_when_overlapped": float(np.median(len_ov)) if len_ov else None,
                      "exps_cycles_when_alone": float(np.median(len_alone)) if len_alone else None}))


def fine_report(tr):
    """Stage-0 softmax phases of the CTA-pair kernel (DBSP_TRACE_FINE, attn_kernel_pd3.cuh)."""
    stats = {}
    for b in range(tr.shape[0]):
        t = tr[b].astype(np.int64)
        n = int((t[:, 0] > 0).sum())
        if n < 8:
            continue
        t = t[2:n]
        for key, arr in [("ld_S", t[:, 2] - t[:, 0]), ("max_exchange", t[:, 6] - t[:, 2]),
                         ("reload_release", t[:, 3] - t[:, 6]), ("exps", t[:, 5] - t[:, 3]),
                         ("pvwait_store", t[:, 4] - t[:, 5]), ("rescale_fence_arrive", t[:, 1] - t[:, 4]),
                         ("total", t[:, 1] - t[:, 0]), ("P_to_PV0", t[:, 7] - t[:, 1]),
                         ("wait_next_S", t[1:, 0] - t[:-1, 1]), ("period", np.diff(t[:, 0]))]:
            stats.setdefault(key, []).append(float(np.median(arr)))
        if b < 4:
            print(f"block {b}: " + json.dumps({k: v[-1] for k, v in stats.items()}))
    print(json.dumps({k: float(np.median(v)) for k, v in stats.items()}))


def duo_report(tr):
    """Two-stage kernel events per 128-key step t (attn_kernel_duo.cuh)."""
    names = ["sm0_start", "sm0_end", "sm1_start", "sm1_end", "S0_issued", "PV0_start", "S1_issued", "PV1_start"]
    stats = {}
    for b in range(tr.shape[0]):
        t = tr[b]
        n = int((t[:, 0] > 0).sum())
        if n < 8:
            continue
        t = t[:n].astype(np.int64)
        for key, arr in [("softmax0", t[:, 1] - t[:, 0]), ("softmax1", t[:, 3] - t[:, 2]),
                         ("sm0_wait_for_S", t[1:, 0] - t[:-1, 1]), ("sm1_wait_for_S", t[1:, 2] - t[:-1, 3]),
                         ("P0_to_PV0", t[:, 5] - t[:, 1]), ("P1_to_PV1", t[:, 7] - t[:, 3]),
                         ("S0_issue_to_sm0", t[:, 0] - t[:, 4]), ("S1_issue_to_sm1", t[:, 2] - t[:, 6]),
                         ("step_period", np.diff(t[:, 0]))]:
            arr = arr[2:] if len(arr) > 4 else arr
            stats.setdefault(key, []).append(float(np.median(arr)))
        if b < 2:
            print(f"block {b}: steps={n}")
            base = t[0, 0]
            for j in range(min(n, 10)):
                print("  t=%2d " % j + " ".join(f"{nm}={int(t[j, e] - base):7d}" for e, nm in enumerate(names)))
    print(json.dumps({k: float(np.median(v)) for k, v in stats.items()}))


if __name__ == "__main__":
    main()
