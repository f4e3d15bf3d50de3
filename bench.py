#!/usr/bin/env python
"""Benchmark of the db-SP hot path on B200: block-sparse DiT attention layer
latency (ms) at N GPUs and the sparse imbalance ratio rho_s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload wan|cogvideox|hunyuan|toy]
                  [--impl ours|reference] [--strategy auto|UxRy] [--balance dbsp|uniform]

N=1: one launch of the sm_100a kernel (K4) over the whole Wan2.1-14B-shaped layer
(40 heads, d=128, 32768 tokens, clustered masks at mean density 0.30), inputs
resident in HBM.  N>1 (torchrun, one rank per GPU): the full SP call -- fused
Ulysses+balancing all-to-allv, ring KV exchange overlapped with per-period
kernels, reverse all-to-allv -- timed as the max over ranks.

Prints ONE JSON line on rank 0 (see README / DESIGN.md for the keys).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "sparse-attn layer latency ms at 1/2/4/8 B200; sparse imbalance ratio rho_s"


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return {"bf16_tflops": j["bf16_tflops"], "bf16_tflops_sustained": j.get("bf16_tflops_sustained"),
                "hbm_gbs": j["hbm_gbs"], "source": "measured (MEASURED_PEAKS.json)"}
    return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0,
            "source": "fallback (B200_PROFILING.md)"}


# ----------------------------------------------------------------------------- clocks
REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, device_index: int):
        self.idx = device_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        if self.proc is None or not self.path:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], None, set()
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 4:
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
                bits = int(parts[3], 16) if parts[3].startswith("0x") else int(parts[3])
            except ValueError:
                continue
            mx = m
            if s > 0.5 * m:  # under load
                sm.append(s)
            for b, n in REASON_BITS.items():
                if bits & b and n != "gpu_idle":
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU baselines
_QKV_CACHE = {}


def cpu_attention_baseline(wl, masks, budget_s: float = 8.0, seed: int = 7) -> dict:
    """Oracle fp32 attention (C, OpenMP on every host core) on a bounded sample
    of (head, Q-block) rows of this workload, extrapolated to the full layer by
    the dense-tile share of the sample."""
    import numpy as np

    import oracle
    H, S, d, nb = wl.heads, wl.tokens, wl.head_dim, wl.blocks
    rng = np.random.default_rng(seed)
    if wl.name not in _QKV_CACHE:
        g = np.random.default_rng(1234)
        _QKV_CACHE[wl.name] = tuple(g.standard_normal((S, H, d), dtype=np.float32) for _ in range(3))
    q, k, v = _QKV_CACHE[wl.name]
    rows_all = [(h, b) for h in range(H) for b in range(nb)]
    order = rng.permutation(len(rows_all))
    per_row = np.array([int(np.unpackbits(masks.words[h, b].view(np.uint8)).sum()) for h, b in rows_all])
    total_tiles = int(per_row.sum())
    done_tiles, done_rows, elapsed, i = 0, 0, 0.0, 0
    batch = 16
    while elapsed < budget_s and i < len(order):
        idx = order[i:i + batch]
        rows = np.array([rows_all[j] for j in idx], np.int32)
        t0 = time.perf_counter()
        oracle.sparse_attention(q, k, v, masks.words, nb, rows=rows)
        elapsed += time.perf_counter() - t0
        done_tiles += int(per_row[idx].sum())
        done_rows += len(idx)
        i += batch
        batch = min(batch * 2, 256)
    full_s = elapsed * total_tiles / max(done_tiles, 1)
    return {"value": full_s * 1e3, "unit": "ms", "cores": oracle.num_threads(), "kind": "port",
            "sample": f"{done_rows} of {len(rows_all)} (head, Q-block) rows "
                      f"({100.0 * done_tiles / total_tiles:.2f}% of dense tiles) timed in {elapsed:.1f} s, "
                      "extrapolated by dense-tile share; fp32 in / fp64 accumulate oracle "
                      "(oracle/attention_ref.c)",
            "sampled_seconds": elapsed}


def wl_key(wl) -> str:
    from paper_2511_23113_b200.workloads import WORKLOADS
    return next((k for k, v in WORKLOADS.items() if v is wl), "")


def reference_planner_baseline(wl, gpus: int = 8, reps: int = 2) -> dict | None:
    """The reference's own planner (compiled from its headers into
    oracle/_ref/ref_bench; single thread as in the reference) on this
    workload's masks: select() and plan_dual per strategy."""
    tool = ROOT / "oracle" / "_ref" / "ref_bench"
    prof = ROOT / "paper_2511_23113_b200" / "profiles" / f"b200_{wl_key(wl)}_measured.json"
    if not prof.exists():
        prof = ROOT / "paper_2511_23113_b200" / "profiles" / "b200_nominal.json"
    if not tool.exists() or not prof.exists():
        return None
    out = subprocess.run([str(tool), str(wl.heads), str(wl.blocks), str(wl.blocks), wl.pattern,
                          str(wl.min_density), str(wl.max_density), str(wl.seed), str(gpus), str(reps),
                          str(prof)], capture_output=True, text=True, timeout=600)
    if out.returncode != 0:
        return None
    return json.loads(out.stdout.strip().splitlines()[-1])


# ----------------------------------------------------------------------------- our arm, N = 1
def kernel_clock_mhz(launch) -> float | None:
    """SM clock inside one K4 launch: CTA 0 stamps clock64 and %globaltimer at
    start and end (dbsp_debug_set_clock_probe); nvidia-smi's sampled clock can
    miss the power-capped in-kernel value."""
    import ctypes
    import torch
    from paper_2511_23113_b200 import _lib
    fn = getattr(_lib.lib(), "dbsp_debug_set_clock_probe", None)
    if fn is None:
        return None
    fn.argtypes = [ctypes.c_void_p]
    buf = torch.zeros(4, dtype=torch.int64, device="cuda")
    fn(ctypes.c_void_p(buf.data_ptr()))
    try:
        launch()
        torch.cuda.synchronize()
    finally:
        fn(None)
    c0, t0, c1, t1 = (int(x) for x in buf.cpu().tolist())
    return round((c1 - c0) / (t1 - t0) * 1e3, 1) if t1 > t0 else None


def run_single(args, wl):
    import numpy as np
    import torch

    import paper_2511_23113_b200 as D
    from paper_2511_23113_b200.attention import AttentionSchedule, sparse_attention

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    masks = D.generate_mask_set(wl.spec())
    total = D.total_blocks(masks)
    H, S, d = wl.heads, wl.tokens, wl.head_dim
    g = torch.Generator(device=dev).manual_seed(1234)
    q = torch.randn(S, H, d, device=dev, dtype=torch.bfloat16, generator=g)
    k = torch.randn(S, H, d, device=dev, dtype=torch.bfloat16, generator=g)
    v = torch.randn(S, H, d, device=dev, dtype=torch.bfloat16, generator=g)
    out = torch.empty_like(q)

    # Host-built schedule: stats / layout for the report, and the host cost.
    t0 = time.perf_counter()
    hsched = AttentionSchedule().build(masks, kv_tokens_global=S, head_dim=d)
    build_ms = (time.perf_counter() - t0) * 1e3
    stats = hsched.stats()
    lay = hsched.layout()
    del hsched
    # One step = one call with live masks: K2 builds the work list on the GPU
    # from the device-resident mask words (both layouts + the device-side
    # kernel choice), then K4.  Events bracket K2 and K4 separately.
    words = torch.from_numpy(np.ascontiguousarray(masks.words).view(np.int64)).to(dev)
    stream = torch.cuda.current_stream(dev)
    # K2 for step i+1 runs on a side stream while K4 of step i runs (two
    # schedule buffers, the planning-ahead pipeline of the SP runtime); every
    # step's K2 is inside the timed region, the first one exposed.
    scheds = [AttentionSchedule(), AttentionSchedule()]
    sched = scheds[0]
    # High priority, as the SP runtime's planner stream: the K2 kernels then take SM
    # slots ahead of the running K4's queued CTAs and finish under it.  At default
    # priority they were dispatched after all of K4's CTAs, so each step's K4 waited
    # ~47 us for its schedule (CogVideoX: step 1.576 ms vs K4 1.529 ms).
    side = torch.cuda.Stream(dev, priority=-1)
    built = [torch.cuda.Event() for _ in range(2)]
    used = [torch.cuda.Event() for _ in range(2)]

    def build(i):
        b = i % 2
        side.wait_event(used[b])  # the K4 that last read this buffer (step i-2)
        scheds[b].build_device(words, masks.num_kv_blocks, kv_tokens_global=S, head_dim=d, stream=side)
        built[b].record(side)

    def run(i, ev_pair=None):
        b = i % 2
        stream.wait_event(built[b])
        if ev_pair:
            ev_pair[0].record(stream)
        scheds[b].launch(q, k, v, out, stream=stream)
        if ev_pair:
            ev_pair[1].record(stream)
        used[b].record(stream)

    for i in range(args.warmup):
        build(i)
        run(i)
    torch.cuda.synchronize()
    # K2 alone (no K4 beside it), for the report: on the side stream each build
    # waits for SM slots the concurrent K4 holds, so its span there is not its cost.
    iso = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    for r in range(3):
        iso[2 * r].record(stream)
        scheds[0].build_device(words, masks.num_kv_blocks, kv_tokens_global=S, head_dim=d, stream=stream)
        iso[2 * r + 1].record(stream)
    torch.cuda.synchronize()
    k2_isolated = [iso[2 * r].elapsed_time(iso[2 * r + 1]) for r in range(3)]
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    from paper_2511_23113_b200 import _lib
    n_launch0 = _lib.lib().dbsp_launch_count()
    w = args.warmup
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        t_start.record(stream)
        side.wait_stream(stream)
        build(w)
        for i in range(args.steps):
            if i + 1 < args.steps:
                build(w + i + 1)
            run(w + i, ev[i])
        t_end.record(stream)
        torch.cuda.synchronize()
    n_launches = _lib.lib().dbsp_launch_count() - n_launch0
    ms = t_start.elapsed_time(t_end) / args.steps
    per = [e[0].elapsed_time(e[1]) for e in ev]          # K4 (both gated launches)
    k2 = k2_isolated  # K2 device schedule build, timed alone
    k4_ms = statistics.mean(per)
    device_build_ms = round(statistics.mean(k2), 4)
    kernel_mhz = kernel_clock_mhz(lambda: sched.launch(q, k, v, out))
    flops = wl.flops_per_block() * total
    pk = peaks()
    achieved = flops / (k4_ms * 1e-3) / 1e12
    roofline = {"bound": "tensor", "achieved": round(achieved, 1), "peak": pk["bf16_tflops"],
                "unit": "TFLOP/s", "frac": round(achieved / pk["bf16_tflops"], 4),
                "frac_of_sustained": round(achieved / pk["bf16_tflops_sustained"], 4)
                if pk.get("bf16_tflops_sustained") else None,
                "traffic": ncu_traffic(wl.name), "peak_source": pk["source"],
                "algorithmic_flops_per_launch": flops,
                "per_unit": f"4*64*64*{d} FLOP per dense 64x64 tile x {total} dense tiles",
                "issued_tile_frac": round(stats["dense_tiles"] / (lay["q_blocks_per_item"] * stats["tile_visits"]), 4),
                "kernel_ms_mean": round(k4_ms, 4), "kernel_ms_min": round(min(per), 4),
                "kernel_ms_median": round(statistics.median(per), 4),
                "kernel": lay["kernel"],
                "timing": "CUDA events around each step's K4 launch on its stream; value (ms_per_step) "
                          "is the whole timed region / steps: every step's K2 device schedule build runs "
                          "inside it, on a high-priority side stream overlapping the previous step's K4 (the first "
                          "one exposed)"}
    # Second ceiling: the softmax's exp2 on the MUFU pipe, 16 per clock per SM on B200
    # (tests/ex2h_bench.cu), at the clock measured inside the kernel.  At d=64 a 64x64
    # tile's 4096 exps take twice its tensor time, so d=64 layers are exp-bound.
    exps = total * 64 * 64
    mufu_peak = 16 * torch.cuda.get_device_properties(dev).multi_processor_count * (kernel_mhz or 1965.0) * 1e6
    roofline["softmax_exp2"] = {"per_launch": exps, "achieved_per_s": round(exps / (k4_ms * 1e-3), 1),
                                "peak_per_s": round(mufu_peak, 1), "frac": round(exps / (k4_ms * 1e-3) / mufu_peak, 4),
                                "peak_basis": "16 ex2/clk/SM x SMs x in-kernel SM clock; d=64 runs 2 of 8 exp pairs "
                                              "on the FMA pipe, so frac may exceed 1 there"}

    # ---- e2e through the public API with host buffers (pinned), every step:
    # H2D of Q/K/V, host schedule build from the masks (C++), upload, kernel, D2H of O.
    qh, kh, vh = (t.cpu().pin_memory() for t in (q, k, v))
    oh = torch.empty_like(qh).pin_memory()
    e2e_steps = max(2, min(args.steps, 5))
    h2d = 3 * qh.numel() * 2
    d2h = oh.numel() * 2
    from paper_2511_23113_b200.e2e import HostStreamingAttention
    streaming = HostStreamingAttention(S, H, d, chunks=args.e2e_chunks, device=dev)
    for it in range(e2e_steps + 1):  # first iteration is warm-up
        if it == 1:
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        streaming(qh, kh, vh, masks, oh)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    sched_bytes = masks.words.nbytes  # mask words go H2D; K2 builds the list on the device
    res = {
        "metric": METRIC, "value": round(ms, 4), "unit": "ms", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": bench_config(wl, 1),
        "details": {"strategy": "U1R1", "density": round(D.density(masks), 4), "dense_tiles": total,
                    "schedule": {**stats, **lay, "host_build_ms": round(build_ms, 2),
                                 "device_build_ms": device_build_ms}},
        "rho_s": 1.0,
        "roofline": roofline,
        "e2e": {"value": round(e2e_ms, 3), "unit": "ms", "h2d_bytes_per_step": h2d + sched_bytes,
                "d2h_bytes_per_step": d2h,
                "note": "public API HostStreamingAttention per step: pinned host q/k/v streamed H2D in "
                        f"{args.e2e_chunks} head chunks (cudaMemcpy2DAsync), mask words H2D, K2 list build + K4 "
                        "per chunk on the GPU, D2H of o -- copies overlap the kernel on 3 streams"},
        "gpu_launches": n_launches,
        "gpu_launches_note": "our kernels in the timed region (dbsp_launch_count): per step the K2 "
                             "device schedule build (k2_count, k2_plan_fused, k2_write_fused; larger "
                             "layers take the k2_count / CUB sort / k2_sorted_counts / k2_write path, "
                             "CUB kernels not counted) and one K4 launch",
        "clocks": {**clk.summary(), "sm_mhz_in_kernel": kernel_mhz,
                   "note": "sm_mhz: nvidia-smi samples over the timed region; sm_mhz_in_kernel: "
                           "clock64 / %globaltimer of CTA 0 inside one more K4 launch right after it"},
    }
    res["planner"] = planner_timing(masks, workload=args.workload)
    if args.sp_sim > 1:
        res["sp_projection"] = sp_projection(q, k, v, masks, args.sp_sim)
    if not args.no_cpu_baseline:
        cb = cpu_attention_baseline(wl, masks, budget_s=args.cpu_budget)
        rp = reference_planner_baseline(wl)
        if rp:
            cb["reference_planner"] = {"select_ms_per_call": rp["select_ms"], "kind": "reference",
                                       "cores": 1, "gpus_planned": 8,
                                       "plan_dual_ms": {s: v["plan_dual_ms"] for s, v in rp["strategies"].items()}}
        res["cpu_baseline"] = cb
    return res


def planner_timing(masks, G: int = 8, reps: int = 5, workload: str = None) -> dict:
    """Our host planner on the bench masks: select() over the G-GPU strategies
    (fresh SelectorState per call, as ref_bench times the reference)."""
    import paper_2511_23113_b200 as D
    from paper_2511_23113_b200.sp_bench import PROFILE, load_profile
    prof = load_profile(workload)
    measured = PROFILE.parent / f"b200_{workload}_measured.json"
    D.select(0, masks, prof, D.PlannerConfig(), D.SelectorState(G))
    t0 = time.perf_counter()
    for i in range(reps):
        sel = D.select(i, masks, prof, D.PlannerConfig(), D.SelectorState(G))
    ms = (time.perf_counter() - t0) / reps * 1e3
    dev_ms = None
    try:  # the GPU selector (dbsp_select_device) on device-resident mask words
        import numpy as np
        import torch
        words = torch.from_numpy(np.ascontiguousarray(masks.words).view(np.int64)).cuda()
        sd = D.select_device(0, words, masks.num_kv_blocks, prof, D.PlannerConfig(), D.SelectorState(G))
        assert str(sd.strategy) == str(sel.strategy) and sd.outcome.rho_post == sel.outcome.rho_post
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(reps):
            D.select_device(i, words, masks.num_kv_blocks, prof, D.PlannerConfig(), D.SelectorState(G))
        dev_ms = round((time.perf_counter() - t0) / reps * 1e3, 3)
    except Exception as e:  # reported, never silently replaced
        dev_ms = f"failed: {e}"
    return {"select_ms_per_call": round(ms, 3), "select_device_ms_per_call": dev_ms,
            "gpus_planned": G, "selected": str(sel.strategy),
            "rho_s_post": round(sel.outcome.rho_post, 4),
            "profile": measured.name if workload and measured.exists() else "b200_nominal.json",
            "threads": os.cpu_count()}


def sp_projection(q, k, v, masks, G: int = 8) -> dict:
    """Every rank's per-period K4 launches of each U x R split run on this one
    GPU (sp.simulate_on_one_gpu) under the uniform USP plan and the db-SP
    plan.  Reports the measured attention critical path sum_p max_r t[p][r]
    (communication excluded), the measured rho_s of kernel times and the
    plan's rho_s; checks the partitioned output against the one-shot kernel."""
    import torch

    import paper_2511_23113_b200 as D
    from paper_2511_23113_b200.attention import sparse_attention
    from paper_2511_23113_b200.sp import measured_rho, simulate_on_one_gpu

    from paper_2511_23113_b200.sp_bench import load_profile, profile_comm_source, profile_path
    prof = load_profile("wan")
    ref = sparse_attention(q, k, v, masks)
    out = {}
    for st in D.enumerate_strategies(G):
        if st.ulysses > masks.num_heads:
            continue
        for name, plan in (("uniform", D.default_plan(masks, st)), ("dbsp", D.plan_dual(masks, st).plan)):
            o, t = simulate_on_one_gpu(q, k, v, masks, st, plan)
            crit = float(sum(max(row) for row in t))
            err = float((o.float() - ref.float()).abs().max())
            # Eq. 4 communication of the same plan (latency.hpp:225-268): the
            # Ulysses all-to-all, the ring p2p not hidden behind compute and
            # the balancing exchange, from the B200 profile.
            lat = D.predict_latency(masks, st, plan, prof)
            comm_ms = (lat.all2all_s + lat.ring_p2p_exposed_s + lat.exchange_s) * 1e3
            out[f"{st}/{name}"] = {"attn_critical_path_ms": round(crit, 4),
                                   "comm_modelled_ms": round(comm_ms, 4),
                                   "layer_ms_with_modelled_comm": round(crit + comm_ms, 4),
                                   "rho_s_measured": round(measured_rho(t), 4),
                                   "rho_s_plan": round(D.imbalance_ratio(D.workload_table(masks, st, plan)), 4),
                                   "max_abs_vs_single_gpu": round(err, 5)}
    planning = planning_on_critical_path(q, k, v, masks, G)

    def best(suffix, key):
        return min(v[key] for k_, v in out.items() if k_.endswith(suffix))
    best_uniform, best_dbsp = best("uniform", "attn_critical_path_ms"), best("dbsp", "attn_critical_path_ms")
    bu_c, bd_c = best("uniform", "layer_ms_with_modelled_comm"), best("dbsp", "layer_ms_with_modelled_comm")
    return {"gpus_simulated": G, "splits": out, "best_uniform_ms": best_uniform, "best_dbsp_ms": best_dbsp,
            "speedup_dbsp_vs_best_uniform": round(best_uniform / best_dbsp, 4),
            "best_uniform_ms_with_modelled_comm": bu_c, "best_dbsp_ms_with_modelled_comm": bd_c,
            "speedup_dbsp_vs_best_uniform_with_modelled_comm": round(bu_c / bd_c, 4),
            "comm_profile": f"{profile_path('wan').name} (comm curves {profile_comm_source('wan')})",
            "planning_on_critical_path": planning,
            "note": "per-rank kernels measured on one B200 (median of 5 launches each); communication: "
                    "attention-only figures exclude it, the *_with_modelled_comm ones add the Eq. 4 terms "
                    "of the B200 profile (nominal NVLink curves until the NCCL sweep runs on >1 GPU)"}


def planning_on_critical_path(q, k, v, masks, G: int = 8, calls: int = 20) -> dict:
    """Per-call select() beside the G-GPU critical path, measured on this GPU:
    the heaviest rank's K4 launches of the selected split's db-SP plan run
    back to back (fixed plan), then with the GPU selector (dbsp_select_device,
    G GPUs) planning the next call on a second stream while each call's
    kernels run (the SPLayerRunner pipeline), then with the selection run
    before each call (not overlapped).  exposed = per-call time minus fixed."""
    import numpy as np
    import torch

    import paper_2511_23113_b200 as D
    from paper_2511_23113_b200.sp import rank_launcher, time_ranks_on_one_gpu
    from paper_2511_23113_b200.sp_bench import load_profile
    prof = load_profile("wan")
    sel = D.select(0, masks, prof, D.PlannerConfig(), D.SelectorState(G))
    st, plan = sel.strategy, sel.outcome.plan
    t = time_ranks_on_one_gpu(q, k, v, masks, st, plan)
    crit = max(range(G), key=lambda r: sum(t[p][r] for p in range(st.ring)))
    launch = rank_launcher(q, k, v, masks, st, plan, crit)
    words = torch.from_numpy(np.ascontiguousarray(masks.words).view(np.int64)).to(q.device)
    plan_stream = torch.cuda.Stream(q.device, priority=-1)  # as SPLayerRunner's planner stream
    state = D.SelectorState(G)
    comp = torch.cuda.current_stream(q.device)

    def select_next(layer):
        with torch.cuda.stream(plan_stream):
            return D.select_device(layer, words, masks.num_kv_blocks, prof, D.PlannerConfig(), state,
                                   stream=plan_stream)

    def timed(mode: str) -> float:
        for _ in range(3):
            launch()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(comp)
        for i in range(calls):
            if mode == "sequential":
                select_next(i)
            launch()
            if mode == "overlapped":
                select_next(i)  # the host waits for the planner stream only
        e1.record(comp)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / calls

    fixed = timed("fixed")
    ovl = timed("overlapped")
    seq = timed("sequential")
    t0 = time.perf_counter()
    for i in range(5):
        select_next(i)
    sel_ms = (time.perf_counter() - t0) / 5 * 1e3
    return {"split": str(st), "critical_rank": crit, "rank_ms_fixed_plan": round(fixed, 4),
            "ms_per_call_overlapped": round(ovl, 4), "ms_per_call_sequential": round(seq, 4),
            "exposed_ms_overlapped": round(ovl - fixed, 4), "exposed_ms_sequential": round(seq - fixed, 4),
            "select_device_ms": round(sel_ms, 4),
            "exposed_frac_overlapped": round((ovl - fixed) / fixed, 4),
            "note": "GPU selector for G GPUs planning the next call on a second stream while the heaviest "
                    "rank's kernels run (PAPER.md:513-514: planning <= 5% of the call)"}


def ncu_traffic(workload_name: str):
    """DRAM bytes per launch from the committed ncu --set full capture."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        j = json.loads(p.read_text())
        return j.get(workload_name, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# ----------------------------------------------------------------------------- shared config
def bench_config(wl, n_gpus: int) -> dict:
    """The `config` both arms print (the driver compares them key for key):
    the workload and the GPU count, nothing arm-specific."""
    mb = wl.tokens * wl.heads * wl.head_dim * 2 / 1e6
    l2 = ("inputs larger than L2 (Q/K/V bf16 %d MB each vs 126 MB L2), no flush" % round(mb)) if 3 * mb > 126 else \
        ("inputs fit in L2 (Q/K/V bf16 %.1f MB each), no flush: K/V re-reads hit L2 by design" % mb)
    return {**wl.describe(), "parallelism": "single-gpu (U1R1)" if n_gpus == 1 else
            f"sp{n_gpus}: per-call U x R selection, db-SP plan", "l2": l2}


# ----------------------------------------------------------------------------- reference arm
def reference_masks(wl, gpus: int):
    """The workload's masks generated by the COMPILED REFERENCE
    (oracle/_ref/ref_bench: generate_mask_set + save_mask_set, DBSPMSK1), read
    with numpy; falls back to the pure-Python restatement oracle/planner_ref.py.
    The product library is never loaded on this arm."""
    import numpy as np

    import oracle
    tool = oracle.ref_tool("ref_bench")
    prof = ROOT / "paper_2511_23113_b200" / "profiles" / "b200_nominal.json"
    if tool.exists():
        fd, path = tempfile.mkstemp(suffix=".dbspmsk")
        os.close(fd)
        try:
            r = subprocess.run([str(tool), str(wl.heads), str(wl.blocks), str(wl.blocks), wl.pattern,
                                str(wl.min_density), str(wl.max_density), str(wl.seed), str(max(gpus, 1)), "1",
                                str(prof), path], capture_output=True, text=True, timeout=600)
            if r.returncode == 0:
                words, _ = oracle.load_mask_words(path)
                return words, "oracle/_ref/ref_bench (compiled reference generate_mask_set + save_mask_set)"
        finally:
            os.unlink(path)
    from oracle import planner_ref as R
    m = R.generate_mask_set(wl.heads, wl.blocks, wl.blocks, wl.pattern, wl.min_density, wl.max_density, 1.0,
                            wl.seed)
    return np.ascontiguousarray(m, np.uint64), "oracle/planner_ref.py (pure-Python restatement)"


def run_reference(args, wl, rank: int) -> dict | None:
    """The reference's CPU path of this hot path on the host cores, rank 0
    only.  The reference has no attention numerics, so a
    step is (i) the reference's own select() for N GPUs (compiled reference,
    oracle/_ref/ref_bench, single thread as the reference runs it) on the
    workload's masks, plus (ii) the fp32 attention oracle (C, OpenMP on every
    host core) over a FIXED bounded sample of (head, Q-block) rows.  `value`
    is the measured time of that step; the full-layer extrapolation of (ii)
    is reported separately."""
    if rank != 0:
        return None
    import numpy as np

    import oracle
    words, masks_from = reference_masks(wl, args.gpus)
    H, S, d, nb = wl.heads, wl.tokens, wl.head_dim, wl.blocks
    g = np.random.default_rng(1234)
    q, k, v = (g.standard_normal((S, H, d), dtype=np.float32) for _ in range(3))
    per_row = np.array([[int(np.unpackbits(words[h, b].view(np.uint8)).sum()) for b in range(nb)]
                        for h in range(H)])
    total_tiles = int(per_row.sum())
    order = np.random.default_rng(7).permutation(H * nb)
    # calibrate the fixed sample to about --ref-budget seconds per step
    probe = np.array([(i // nb, i % nb) for i in order[:16]], np.int32)
    t0 = time.perf_counter()
    oracle.sparse_attention(q, k, v, words, nb, rows=probe)
    t_probe = time.perf_counter() - t0
    tiles_probe = max(int(per_row[probe[:, 0], probe[:, 1]].sum()), 1)
    want_tiles = tiles_probe * args.ref_budget / max(t_probe, 1e-6)
    cum = np.cumsum(per_row.reshape(-1)[order])
    n_rows = int(min(len(order), max(16, np.searchsorted(cum, want_tiles) + 1)))
    rows = np.array([(i // nb, i % nb) for i in order[:n_rows]], np.int32)
    sample_tiles = int(per_row[rows[:, 0], rows[:, 1]].sum())

    # (i) the reference planner, per call, on the same masks (N > 1 only: at
    # N = 1 there is nothing to select)
    planner_ms, rp = 0.0, None
    if args.gpus > 1:
        rp = reference_planner_baseline(wl, gpus=args.gpus, reps=max(args.steps, 1))
        planner_ms = rp["select_ms"] if rp else 0.0
    vals = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.sparse_attention(q, k, v, words, nb, rows=rows)
        ms = (time.perf_counter() - t0) * 1e3
        if i >= args.warmup:
            vals.append(ms + planner_ms)
    value = statistics.mean(vals)
    attn_ms = value - planner_ms
    sample = (f"{n_rows} of {H * nb} (head, Q-block) rows = {sample_tiles} of {total_tiles} dense tiles "
              f"({100.0 * sample_tiles / total_tiles:.2f}%), the same rows every step; fp32 in / fp64 accumulate "
              "oracle (oracle/attention_ref.c)" +
              (f" + reference select() for {args.gpus} GPUs ({planner_ms:.2f} ms/call, 1 thread)" if args.gpus > 1
               else ""))
    cb = {"value": round(value, 3), "unit": "ms", "cores": oracle.num_threads(), "kind": "port", "sample": sample}
    res = {"metric": METRIC, "value": round(value, 3), "unit": "ms", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(value, 3), "higher_is_better": False,
           "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": bench_config(wl, args.gpus), "impl": "reference",
           "cpu_baseline": cb,
           "e2e": {"value": round(value, 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "extrapolated_full_layer_ms": round(attn_ms * total_tiles / sample_tiles + planner_ms, 1),
           "extrapolation": "attention sample time x (all dense tiles / sampled dense tiles) + select(); "
                            "not measured, for scale only",
           "masks_from": masks_from}
    if rp:
        res["reference_planner"] = rp
    res["native_so_loaded"] = loaded_native_libs()
    return res


def loaded_native_libs() -> list:
    """In-tree shared objects mapped into this process (/proc/self/maps)."""
    try:
        maps = Path("/proc/self/maps").read_text().splitlines()
    except OSError:
        return []
    out = sorted({ln.split()[-1] for ln in maps if ln.split() and ln.split()[-1].startswith(str(ROOT))
                  and ".so" in ln.split()[-1]})
    return [str(Path(p).relative_to(ROOT)) for p in out]


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch_ranks(args) -> int:
    """`bench.py --gpus N` without torchrun: re-run this script under
    torch.distributed.run with N ranks on 127.0.0.1 (one process per GPU)."""
    if not args.dry_run and args.impl == "ours":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, this node has {have}", file=sys.stderr)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve())]
    cmd += sys.argv[1:]
    env = dict(os.environ, DBSP_BENCH_LAUNCHED="1")
    return subprocess.run(cmd, env=env).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="wan")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--strategy", default="auto")
    ap.add_argument("--balance", default="dbsp", choices=["dbsp", "uniform"])
    ap.add_argument("--executor", default="native", choices=["native", "python"],
                    help="N>1: the C++ SP executor (default) or the Python one")
    ap.add_argument("--planner", default="device", choices=["device", "host"],
                    help="N>1: per-call select() on the GPU (default) or on the host")
    ap.add_argument("--dry-run", action="store_true",
                    help="N>1 launcher/loop check on CPU (gloo, no attention compute); not a measurement")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=8.0)
    ap.add_argument("--ref-budget", type=float, default=4.0)
    ap.add_argument("--e2e-chunks", type=int, default=8)
    ap.add_argument("--sp-sim", type=int, default=8,
                    help="N=1 only: simulate every rank of each UxRy split for this many GPUs (0 = off)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")

    from paper_2511_23113_b200.workloads import WORKLOADS
    wl = WORKLOADS[args.workload]
    rank = int(os.environ.get("RANK", "0"))
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None and args.gpus > 1:
        # N ranks requested without a launcher: become the launcher
        sys.exit(launch_ranks(args))
    world = int(world_env or "1")
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch with --nproc-per-node {args.gpus}",
              file=sys.stderr)
        sys.exit(2)

    if args.impl == "reference":
        res = run_reference(args, wl, rank)
        if res is not None:
            print(json.dumps(res), flush=True)
        return

    if world > 1:
        from paper_2511_23113_b200.sp_bench import run_distributed
        res = run_distributed(args, wl, rank, world)
        if res is not None:
            # the details of this arm's run leave `config`, which both arms share
            res["details"] = {k: v for k, v in res["config"].items() if k not in wl.describe()}
            res["config"] = bench_config(wl, world)
    else:
        res = run_single(args, wl)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
