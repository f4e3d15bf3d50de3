"""bench.py's N>1 leg: one process per GPU (torchrun), NCCL over NVLink.

Times the full sequence-parallel attention call of sp.SPAttention (fused
all-to-all(v), y ring periods of K4 overlapped with the KV send/recv, reverse
all-to-all(v)) on the workload's global Q/K/V sharded by token blocks; the
reported latency is the max over ranks of CUDA-event time.
"""
from __future__ import annotations

import json
import os
import statistics
from pathlib import Path

import numpy as np

from . import planner as P
from .sp import SPAttention, home_range, rank_layouts

ROOT = Path(__file__).resolve().parents[1]
PROFILE = Path(__file__).resolve().parent / "profiles" / "b200_nominal.json"


def load_profile(workload: str = None) -> P.MachineProfile:
    """B200 MachineProfile for the selector: the measured one for this
    workload shape (tests/measure_profile.py) when present, else nominal."""
    if workload:
        measured = PROFILE.parent / f"b200_{workload}_measured.json"
        if measured.exists():
            return P.MachineProfile.from_json(json.loads(measured.read_text()))
    return P.MachineProfile.from_json(json.loads(PROFILE.read_text()))


def choose(masks, world: int, strategy: str, balance: str, workload: str = None):
    """Strategy + plan for this call: `auto` runs the U x R selector
    (selector.hpp:55-75) on the live masks; otherwise the named split."""
    if strategy == "auto":
        sel = P.select(0, masks, load_profile(workload), P.PlannerConfig(), P.SelectorState(world))
        st = sel.strategy
    else:
        st = P.parse_strategy(strategy)
    plan = P.plan_dual(masks, st).plan if balance == "dbsp" else P.default_plan(masks, st)
    return st, plan


def run_distributed(args, wl, rank: int, world: int):
    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", rank))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    # A collective over all ranks first: batch_isend_irecv as the first NCCL
    # call of a group must involve every rank, which the ragged exchanges
    # need not do.
    dist.barrier()
    try:
        masks = P.generate_mask_set(wl.spec())
        st, plan = choose(masks, world, args.strategy, args.balance, args.workload)
        H, S, d, nb = wl.heads, wl.tokens, wl.head_dim, wl.blocks
        g = torch.Generator(device=dev).manual_seed(1234)
        q = torch.randn(S, H, d, device=dev, dtype=torch.bfloat16, generator=g)
        k = torch.randn(S, H, d, device=dev, dtype=torch.bfloat16, generator=g)
        v = torch.randn(S, H, d, device=dev, dtype=torch.bfloat16, generator=g)
        lo, hi = home_range(rank, world, nb)
        qh, kh, vh = (t[lo * 64:hi * 64].contiguous() for t in (q, k, v))
        del q, k, v
        torch.cuda.empty_cache()

        # per-period kernel timing (events on the compute stream) for a measured rho_s
        times = {}
        # DBSP_FUSE_RETURN=1: O returns home inside K4's epilogue (symmetric
        # memory peer stores) instead of the NCCL reverse all-to-all(v).
        fuse = os.environ.get("DBSP_FUSE_RETURN", "0") == "1"
        sp = SPAttention(masks, st, plan, S, d, rank, world, dev, fuse_return=fuse)
        base_fn = sp.attn_fn
        record = {"on": False}

        def timed_fn(layout, period, *a):
            if not record["on"]:
                return base_fn(layout, period, *a)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            base_fn(layout, period, *a)
            e1.record()
            times.setdefault(period, []).append((e0, e1))
        sp.attn_fn = timed_fn
        # DBSP_SP_NATIVE=1: the timed call is the C++ executor (csrc/sp_exec.cu,
        # dbsp_sp_attention); the per-period instrumentation below still runs
        # the Python executor, which issues the same kernels.
        native = os.environ.get("DBSP_SP_NATIVE", "0") == "1"
        if native:
            from .sp import NativeSPContext

            def bcast(b):
                obj = [b]
                dist.broadcast_object_list(obj, src=0)
                return obj[0]
            nctx = NativeSPContext(rank, world, bcast)
            call = lambda qq, kk, vv, oo=None: nctx(masks, st, plan, qq, kk, vv, oo)
        else:
            call = sp

        out = torch.empty_like(qh)
        for _ in range(args.warmup):
            call(qh, kh, vh, out)
        torch.cuda.synchronize()
        dist.barrier()
        from bench import ClockSampler, peaks
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            torch.cuda.synchronize()
            ev0.record()
            for _ in range(args.steps):
                call(qh, kh, vh, out)
            ev1.record()
            torch.cuda.synchronize()
        dist.barrier()
        ms = ev0.elapsed_time(ev1) / args.steps
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())

        # one extra instrumented call: per-period kernel ms on every rank
        record["on"] = True
        sp(qh, kh, vh, out)
        torch.cuda.synchronize()
        record["on"] = False
        y = st.ring
        per = [statistics.mean(e0.elapsed_time(e1) for e0, e1 in times.get(p, [])) if times.get(p) else 0.0
               for p in range(y)]
        allt = torch.tensor(per, device=dev, dtype=torch.float64)
        gathered = [torch.zeros_like(allt) for _ in range(world)]
        dist.all_gather(gathered, allt)
        kernel_times = np.stack([x.cpu().numpy() for x in gathered], axis=1)  # [period, rank]
        rho_meas = float(kernel_times.max(axis=1).sum() * world / max(kernel_times.sum(), 1e-12))
        rho_plan = P.imbalance_ratio(P.workload_table(masks, st, plan))

        # e2e: pinned host shard -> device, call, result -> pinned host, every step
        hq, hk, hv = (x.cpu().pin_memory() for x in (qh, kh, vh))
        ho = torch.empty_like(hq).pin_memory()
        e2e_steps = max(2, min(args.steps, 5))
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(e2e_steps):
            dq, dk, dv = (x.to(dev, non_blocking=True) for x in (hq, hk, hv))
            ho.copy_(call(dq, dk, dv), non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1) / e2e_steps], device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)

        total_blocks = P.total_blocks(masks)
        flops = wl.flops_per_block() * total_blocks
        clocks = clk.summary()
        if rank != 0:
            return None
        pk = peaks()
        lay = rank_layouts(st, plan, nb, nb)
        return {
            "metric": "sparse-attn layer latency ms at 1/2/4/8 B200; sparse imbalance ratio rho_s",
            "value": round(ms_max, 4), "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max, 4), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {**wl.describe(), "parallelism": f"sp-{st}", "strategy": str(st),
                       "o_return": "fused K4 epilogue (symmetric memory)" if fuse else "NCCL all-to-allv",
                       "executor": "C++ (dbsp_sp_attention)" if native else "Python (sp.SPAttention)",
                       "balance": args.balance, "selector": args.strategy,
                       "l2": "inputs larger than L2 (per-rank shards + exchanged buffers)"},
            "rho_s": round(rho_plan, 4), "rho_s_measured": round(rho_meas, 4),
            "kernel_ms_per_period_per_rank": np.round(kernel_times, 4).tolist(),
            "roofline": {"bound": "tensor", "achieved": round(flops / (ms_max * 1e-3) / 1e12, 1),
                         "peak": pk["bf16_tflops"] * world, "unit": "TFLOP/s",
                         "frac": round(flops / (ms_max * 1e-3) / 1e12 / (pk["bf16_tflops"] * world), 4),
                         "traffic": None, "note": "layer-level (incl. communication) over N x measured peak"},
            "e2e": {"value": round(float(te.item()), 3), "unit": "ms",
                    "h2d_bytes_per_step": 3 * hq.numel() * 2, "d2h_bytes_per_step": ho.numel() * 2},
            "gpu_launches": args.steps * (y + (1 if y > 1 else 0)),  # K4 per period + accum init
            "clocks": clocks,
            "per_rank_work": {"heads": [len(l.heads) for l in lay], "q_blocks": [len(l.q_blocks) for l in lay]},
        }
    finally:
        dist.destroy_process_group()
