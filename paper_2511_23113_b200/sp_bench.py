"""bench.py's N>1 leg: one process per GPU, NCCL over NVLink.

One JSON line (rank 0) reports, for the workload's global Q/K/V sharded by
token blocks (home layout) and its masks:

  value      ms per call of the per-call runtime (sp.SPLayerRunner): select()
             on the live masks for every call (selector.hpp:55-75), its
             planning for the next call overlapped with this call's GPU work,
             then the C++ SP executor (csrc/sp_exec.cu: fused all-to-all(v),
             y ring periods of K4 with the KV exchange on a second stream,
             reverse all-to-all(v)) under the selected split and the db-SP plan;
             CUDA-event time, max over ranks;
  splits     every U x R split of N GPUs under the uniform USP plan
             (default_plan, metrics.hpp:103-113) and the db-SP plan (plan_dual,
             planner.hpp:175-217), same kernels and executor: ms per call (max
             over ranks), the measured rho_s of per-(period, rank) K4 times and
             the planned rho_s of the workload table (metrics.hpp:133-186);
  best_uniform / best_dbsp and their ratio -- the north-star comparison;
  planning   host ms per selection, and the exposed part: value minus the
             same split and plan run with no selection in the loop.

--dry-run (CPU, gloo): the same loops with the Python executor, CPU tensors
and no attention compute (the exchanges only), on a small workload -- a check
of the launcher, the rank/world handling and the per-split loop on a machine
without GPUs.  Its numbers are not measurements.
"""
from __future__ import annotations

import json
import os
import time
from pathlib import Path

import numpy as np

from . import planner as P
from .sp import NativeSPContext, SPAttention, SPLayerRunner, home_range, measured_rho

ROOT = Path(__file__).resolve().parents[1]
PROFILE = Path(__file__).resolve().parent / "profiles" / "b200_nominal.json"
METRIC = "sparse-attn layer latency ms at 1/2/4/8 B200; sparse imbalance ratio rho_s"


def load_profile(workload: str = None) -> P.MachineProfile:
    """B200 MachineProfile for the selector: the measured one for this
    workload shape (tests/measure_profile.py) when present, else nominal."""
    return P.MachineProfile.from_json(json.loads(profile_path(workload).read_text()))


def profile_path(workload: str = None) -> Path:
    if workload:
        measured = PROFILE.parent / f"b200_{workload}_measured.json"
        if measured.exists():
            return measured
    return PROFILE


def profile_comm_source(workload: str = None) -> str:
    """'measured' when the profile's all2all/p2p curves came from an NCCL sweep
    (tests/measure_profile.py --comm), else 'nominal'."""
    try:
        j = json.loads(profile_path(workload).read_text())
    except Exception:
        return "nominal"
    return "measured" if j.get("comm_source") == "measured" else "nominal"


def choose(masks, world: int, strategy: str, balance: str, workload: str = None):
    """Strategy + plan for one call: `auto` runs the U x R selector
    (selector.hpp:55-75) on the masks; otherwise the named split."""
    if strategy == "auto":
        sel = P.select(0, masks, load_profile(workload), P.PlannerConfig(), P.SelectorState(world))
        st = sel.strategy
    else:
        st = P.parse_strategy(strategy)
    plan = P.plan_dual(masks, st).plan if balance == "dbsp" else P.default_plan(masks, st)
    return st, plan


def _zero_attn_fn(layout, period, q_loc, k_buf, v_buf, out_loc, o_acc, lse_acc, first, last, kv_blocks):
    """--dry-run: no attention compute (the exchanges alone are exercised)."""
    if last:
        out_loc.zero_()


class _Clock:
    """Device time of K calls on `stream` (CUDA events), or wall time on CPU."""

    def __init__(self, cuda: bool, stream=None):
        self.cuda, self.stream = cuda, stream

    def __enter__(self):
        import torch
        if self.cuda:
            torch.cuda.synchronize()
            self.e0 = torch.cuda.Event(enable_timing=True)
            self.e1 = torch.cuda.Event(enable_timing=True)
            self.e0.record(self.stream)
        else:
            self.t0 = time.perf_counter()
        return self

    def __exit__(self, *exc):
        import torch
        if self.cuda:
            self.e1.record(self.stream)
            torch.cuda.synchronize()
            self.ms = self.e0.elapsed_time(self.e1)
        else:
            self.ms = (time.perf_counter() - self.t0) * 1e3


def run_distributed(args, wl, rank: int, world: int):
    import torch
    import torch.distributed as dist

    dry = bool(getattr(args, "dry_run", False))
    local = int(os.environ.get("LOCAL_RANK", rank))
    if dry:
        dev = torch.device("cpu")
        dist.init_process_group("gloo")
    else:
        dev = torch.device("cuda", local)
        torch.cuda.set_device(dev)
        dist.init_process_group("nccl", device_id=dev)
    # A collective over all ranks first: batched send/recv as the first NCCL
    # call of a group must involve every rank, which the ragged exchanges need not.
    dist.barrier()
    try:
        return _run(args, wl, rank, world, dev, dry)
    finally:
        dist.destroy_process_group()


def _max_over_ranks(x: float, dev) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _gather(vals, dev) -> np.ndarray:
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return np.stack([o.cpu().numpy() for o in out], axis=1)  # [len(vals), world]


def _run(args, wl, rank: int, world: int, dev, dry: bool):
    import torch
    import torch.distributed as dist

    cuda = not dry
    masks = P.generate_mask_set(wl.spec())
    H, S, d, nb = wl.heads, wl.tokens, wl.head_dim, wl.blocks
    if S % 64:
        raise P.ConfigError("the SP path needs a token count that is a multiple of 64")
    # Global inputs from one seed on every rank (1/2/4/8 GPUs see the same layer), home shard kept.
    g = torch.Generator(device=dev).manual_seed(1234)
    dt = torch.float32 if dry else torch.bfloat16
    lo, hi = home_range(rank, world, nb)
    shards = []
    for _ in range(3):
        full = torch.randn(S, H, d, device=dev, dtype=dt, generator=g)
        shards.append(full[lo * 64:hi * 64].contiguous())
        del full
    qh, kh, vh = shards
    if cuda:
        torch.cuda.empty_cache()
    out = torch.empty_like(qh)
    stream = torch.cuda.Stream(dev) if cuda else None
    executor = "python" if (dry or args.executor == "python") else "native"

    def bcast(b):
        obj = [b]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    native = NativeSPContext(rank, world, bcast) if executor == "native" else None
    profile = load_profile(args.workload)

    def run_fixed(st, plan, spa=None):
        if native is not None:
            return native(masks, st, plan, qh, kh, vh, out, stream=stream)
        return spa(qh, kh, vh, out)

    # ---- every split x {uniform, db-SP}: fixed plan, same kernels and executor
    splits = {}
    for st in P.enumerate_strategies(world):
        if st.ulysses > H:
            continue
        for bal in ("uniform", "dbsp"):
            plan = P.plan_dual(masks, st).plan if bal == "dbsp" else P.default_plan(masks, st)
            spa = None if native is not None else SPAttention(
                masks, st, plan, S, d, rank, world, dev, attn_fn=_zero_attn_fn if dry else None)
            with (torch.cuda.stream(stream) if cuda else _Null()):
                for _ in range(args.warmup):
                    run_fixed(st, plan, spa)
                if cuda:
                    native.synchronize(stream) if native is not None else torch.cuda.synchronize()
                dist.barrier()
                with _Clock(cuda, stream) as clk:
                    for _ in range(args.steps):
                        run_fixed(st, plan, spa)
                ms = _max_over_ranks(clk.ms / args.steps, dev)
                # one more call with per-period K4 events: measured rho_s
                per = [0.0] * st.ring
                if native is not None:
                    native.set_timing(True)
                    run_fixed(st, plan, spa)
                    per = native.period_ms()
                    native.set_timing(False)
            kt = _gather(per, dev)  # [period, rank]
            splits[f"{st}/{bal}"] = {
                "ms": round(ms, 4),
                "rho_s_measured": round(measured_rho(kt), 4) if kt.sum() > 0 else None,
                "rho_s_plan": round(P.imbalance_ratio(P.workload_table(masks, st, plan)), 4),
                "kernel_ms_per_period_per_rank": np.round(kt, 4).tolist(),
            }

    # ---- headline: the per-call runtime (select on the live masks every call)
    runner = SPLayerRunner(rank, world, profile, executor=executor, planner="host" if dry else args.planner,
                           device=dev, broadcast_id=bcast, attn_fn=_zero_attn_fn if dry else None,
                           balance=args.balance, native_ctx=native)  # one communicator per process
    words = None
    if cuda and args.planner == "device":
        words = torch.from_numpy(np.ascontiguousarray(masks.words).view(np.int64)).to(dev)
    layer = 0
    with (torch.cuda.stream(stream) if cuda else _Null()):
        for _ in range(args.warmup):
            runner(layer, masks, qh, kh, vh, out, words=words)
            runner.prefetch(layer, masks, words)
        if cuda:
            torch.cuda.synchronize()
        dist.barrier()
        runner.plan_host_ms.clear()
        runner.exposed_host_ms = 0.0
        n_launch0 = _launches()
        with _Clock(cuda, stream) as clk:
            for _ in range(args.steps):
                runner(layer, masks, qh, kh, vh, out, words=words)
                runner.prefetch(layer, masks, words)  # next call's plan, under this call's GPU work
        if native is not None:
            native.synchronize(stream, timeout_ms=600000)
    n_launches = _launches() - n_launch0
    ms_runtime = _max_over_ranks(clk.ms / args.steps, dev)
    sel = runner.last
    chosen = f"{sel.strategy}/{args.balance}"
    # every rank must have selected the same split and plan
    import zlib
    sig = float(zlib.crc32(str(sel.strategy).encode() + sel.outcome.plan.head_assignment.tobytes() +
                           sel.outcome.plan.q_assignment.tobytes() + sel.outcome.plan.kv_assignment.tobytes()))
    agree = bool(np.all(_gather([sig], dev) == sig))

    # ---- e2e: pinned host shard -> device, call (with selection), result -> pinned host
    e2e = None
    if cuda:
        hq, hk, hv = (x.cpu().pin_memory() for x in (qh, kh, vh))
        ho = torch.empty_like(hq).pin_memory()
        e2e_steps = max(2, min(args.steps, 5))
        dq, dk, dv = (torch.empty_like(x) for x in (qh, kh, vh))
        with torch.cuda.stream(stream):
            torch.cuda.synchronize()
            dist.barrier()
            with _Clock(True, stream) as ec:
                for _ in range(e2e_steps):
                    for hsrc, ddst in ((hq, dq), (hk, dk), (hv, dv)):
                        ddst.copy_(hsrc, non_blocking=True)
                    runner(layer, masks, dq, dk, dv, out, words=words)
                    ho.copy_(out, non_blocking=True)
                    runner.prefetch(layer, masks, words)
        e2e = {"value": round(_max_over_ranks(ec.ms / e2e_steps, dev), 3), "unit": "ms",
               "h2d_bytes_per_step": 3 * hq.numel() * hq.element_size(),
               "d2h_bytes_per_step": ho.numel() * ho.element_size(),
               "note": "per rank: pinned home shards H2D, per-call select + SP call, O shard D2H"}

    plan_ms = float(np.mean(runner.plan_host_ms)) if runner.plan_host_ms else 0.0
    plan_ms = _max_over_ranks(plan_ms, dev)
    if rank != 0:
        return None
    uni = {k: v for k, v in splits.items() if k.endswith("/uniform")}
    dbs = {k: v for k, v in splits.items() if k.endswith("/dbsp")}
    best_u = min(uni, key=lambda k: uni[k]["ms"])
    best_d = min(dbs, key=lambda k: dbs[k]["ms"])
    fixed_ms = splits.get(chosen, {}).get("ms")
    flops = wl.flops_per_block() * P.total_blocks(masks)
    from bench import peaks  # noqa: E402  (bench.py is the caller)
    pk = peaks()
    res = {
        "metric": METRIC, "value": round(ms_runtime, 4), "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_runtime, 4), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32" if dry else "bf16",
        "data": "synthetic",
        "config": {**wl.describe(),
                   "selected": str(sel.strategy), "balance": args.balance,
                   "executor": "Python (sp.SPAttention, gloo)" if dry else
                   ("C++ (dbsp_sp_attention, NCCL)" if executor == "native" else "Python (sp.SPAttention, NCCL)"),
                   "planner": "host" if dry else args.planner},
        "rho_s": splits.get(chosen, {}).get("rho_s_plan"),
        "rho_s_measured": splits.get(chosen, {}).get("rho_s_measured"),
        "splits": splits,
        "best_uniform": {"split": best_u, "ms": uni[best_u]["ms"]},
        "best_dbsp": {"split": best_d, "ms": dbs[best_d]["ms"]},
        "speedup_dbsp_vs_best_uniform": round(uni[best_u]["ms"] / max(dbs[best_d]["ms"], 1e-9), 4),
        "planning": {"planner": "host" if dry else args.planner, "host_ms_per_selection": round(plan_ms, 4),
                     "fixed_plan_ms": fixed_ms,
                     "exposed_ms_per_call": round(ms_runtime - fixed_ms, 4) if fixed_ms is not None else None,
                     "ranks_agree": agree,
                     "note": "selection for call t+1 runs while call t's GPU work executes; exposed = value "
                             "minus the same split and plan with no selection in the loop"},
        "profile_comm": profile_comm_source(args.workload),
        "roofline": {"bound": "tensor", "achieved": round(flops / (ms_runtime * 1e-3) / 1e12, 1),
                     "peak": round(pk["bf16_tflops"] * world, 1), "unit": "TFLOP/s",
                     "frac": round(flops / (ms_runtime * 1e-3) / 1e12 / (pk["bf16_tflops"] * world), 4),
                     "traffic": None, "note": "layer level (communication and planning included) over N x peak"},
        "e2e": e2e,
        "gpu_launches": None,
    }
    if dry:
        res["dry_run"] = True
        res["note"] = "dry run: gloo on CPU, no attention compute; not a measurement"
    else:
        res["gpu_launches"] = n_launches
    return res


def _launches() -> int:
    from . import _lib
    try:
        return int(_lib.lib().dbsp_launch_count())
    except ImportError:
        return 0


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False
