"""Sequence-parallel execution of one block-sparse attention call (the
execution layer the reference only models: SURVEY.md §2.2 C1-C4, K5).

Home layout: rank g holds token blocks [floor(g*nb/G), floor((g+1)*nb/G)) of
Q, K, V with all heads, bf16 [tokens, H, d].  A call under strategy UxRy and
partition plan (head_assignment, q_assignment, kv_assignment) runs on GPU
g = u*y + r (metrics.hpp:116):

1. one all-G all-to-all(v) (C1 Ulysses head scatter fused with C2, the
   db-SP balancing moves -- NVSwitch is uniform, so one exchange costs the
   same as the Ulysses one): GPU (u, r) receives Q blocks {q : q_assign = r}
   and KV blocks {k : kv_assign = r} for heads {h : head_assign = u};
2. y ring periods (C3): in period p the GPU holds KV group (r + p) mod y
   (metrics.hpp:131-132), runs K4 on it in accumulate mode (K5 merge in the
   epilogue) while the next group travels to it from ring neighbour r+1 over
   NCCL send/recv on NCCL's stream;
3. the reverse all-to-all(v) returns O to the home layout.

The same per-rank layout drives three executors: the NCCL one (one process
per GPU), a single-process simulation that runs every rank's kernels on one
GPU (for parity and for measured per-rank kernel times, i.e. a measured
rho_s), and CPU/gloo tests that inject an oracle compute function.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence

import numpy as np

from . import planner as _P
from .planner import (AttentionMaskSet, ConfigError, ContractError, MachineProfile, ParallelStrategy,
                      PartitionPlan, PlannerConfig, SelectorState)


def home_range(rank: int, world: int, nblocks: int):
    return (rank * nblocks) // world, ((rank + 1) * nblocks) // world


@dataclass
class RankLayout:
    rank: int
    u: int
    r: int
    heads: np.ndarray                 # global head ids on this GPU (ascending)
    q_blocks: np.ndarray              # global Q block ids (ascending) -> local Q buffer order
    kv_groups: List[np.ndarray]       # per ring group g: global KV block ids (ascending)
    period_groups: List[int] = field(default_factory=list)  # group held in period p

    @property
    def y(self) -> int:
        return len(self.kv_groups)


def rank_layouts(strategy: ParallelStrategy, plan: PartitionPlan, nq: int, nk: int) -> List[RankLayout]:
    x, y = strategy.ulysses, strategy.ring
    ha = np.asarray(plan.head_assignment)
    qa = np.asarray(plan.q_assignment)
    ka = np.asarray(plan.kv_assignment)
    if len(qa) != nq or len(ka) != nk:
        raise ContractError("plan dimensions do not match the block grid")
    groups = [np.flatnonzero(ka == g).astype(np.int64) for g in range(y)]
    out = []
    for u in range(x):
        heads = np.flatnonzero(ha == u).astype(np.int64)
        for r in range(y):
            out.append(RankLayout(u * y + r, u, r, heads, np.flatnonzero(qa == r).astype(np.int64),
                                  groups, [(r + p) % y for p in range(y)]))
    return out


@dataclass
class ExchangePlan:
    """Token/head index lists of the fused all-to-all(v) for one rank."""
    # per peer: (home-local token rows to gather for Q, for KV) on the send side
    send_q_rows: List[np.ndarray]
    send_kv_rows: List[np.ndarray]
    send_heads: List[np.ndarray]
    # per peer: number of Q / KV blocks received (contiguous, peer order)
    recv_q_blocks: List[int]
    recv_kv_blocks: List[int]


def exchange_plan(rank: int, world: int, layouts: List[RankLayout], nb: int) -> ExchangePlan:
    lo, hi = home_range(rank, world, nb)
    me = layouts[rank]
    sq, skv, sh, rq, rkv = [], [], [], [], []
    for d in range(world):
        dst = layouts[d]
        qb = dst.q_blocks[(dst.q_blocks >= lo) & (dst.q_blocks < hi)]
        kb = dst.kv_groups[dst.r]
        kb = kb[(kb >= lo) & (kb < hi)]
        sq.append(_rows(qb - lo))
        skv.append(_rows(kb - lo))
        sh.append(dst.heads)
        slo, shi = home_range(d, world, nb)
        rq.append(int(((me.q_blocks >= slo) & (me.q_blocks < shi)).sum()))
        g = me.kv_groups[me.r]
        rkv.append(int(((g >= slo) & (g < shi)).sum()))
    return ExchangePlan(sq, skv, sh, rq, rkv)


def _rows(local_blocks: np.ndarray) -> np.ndarray:
    if len(local_blocks) == 0:
        return np.zeros(0, np.int64)
    return (local_blocks[:, None] * 64 + np.arange(64)[None, :]).reshape(-1)


# ----------------------------------------------------------------------------- executor
AttnFn = Callable[..., None]
"""attn_fn(layout, period, q_local, k_buf, v_buf, out_local, o_acc, lse_acc,
first: bool, last: bool, kv_blocks) -- computes K4 for one ring period,
merging into (o_acc, lse_acc) and writing out_local on the last period."""


class SPAttention:
    """One process per GPU.  Torch tensors on `device`; collectives through
    torch.distributed (NCCL on GPUs, gloo in CPU tests)."""

    def __init__(self, masks: AttentionMaskSet, strategy: ParallelStrategy, plan: PartitionPlan,
                 tokens: int, head_dim: int, rank: int, world: int, device, attn_fn: AttnFn = None,
                 group=None, fuse_return: bool = False):
        """fuse_return: step 3 runs inside K4's epilogue -- every rank's home
        output shard lives in torch symmetric memory and the final launch
        stores O rows straight into the home shards over NVLink
        (dbsp_attention_launch_scatter), so there is no separate O exchange.
        The CUDA attention path only."""
        if strategy.gpus() != world:
            raise ContractError(f"strategy {strategy} needs {strategy.gpus()} ranks, have {world}")
        if tokens % 64:
            raise ContractError("the SP path needs a token count that is a multiple of 64")
        self.masks, self.strategy, self.plan = masks, strategy, plan
        self.S, self.d, self.rank, self.world = tokens, head_dim, rank, world
        self.nb = tokens // 64
        self.device = device
        self.group = group
        self.layouts = rank_layouts(strategy, plan, masks.num_q_blocks, masks.num_kv_blocks)
        self.me = self.layouts[rank]
        self.xp = exchange_plan(rank, world, self.layouts, self.nb)
        # reverse exchange: what each peer sends back to me / I send back to each home
        self._symm = None
        self._scatter = None
        if fuse_return:
            if attn_fn is not None:
                raise ContractError("fuse_return needs the CUDA attention path")
            self._setup_fused_return(masks.num_heads)
        self.attn_fn = attn_fn or _cuda_attn_fn(masks, self.me, tokens, self._scatter)
        self._prepare_indices()

    def _setup_fused_return(self, H: int):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        from .attention import OutScatter
        rows = max(home_range(r, self.world, self.nb)[1] - home_range(r, self.world, self.nb)[0]
                   for r in range(self.world)) * 64
        self._home_out = symm.empty(rows, H, self.d, dtype=torch.bfloat16, device=self.device)
        self._symm = symm.rendezvous(self._home_out, self.group or dist.group.WORLD)
        peers = [int(ptr) + int(self._symm.offset) for ptr in self._symm.buffer_ptrs]
        qmap, hmap = scatter_maps(self.me, self.world, self.nb, self.S)
        self._scatter = OutScatter(peers, qmap, hmap, H, self.device)

    # -- index tensors (host -> device once per plan)
    def _prepare_indices(self):
        import torch
        dev = self.device
        t = lambda a: torch.as_tensor(np.asarray(a, np.int64), device=dev)
        self.send_q_rows = [t(a) for a in self.xp.send_q_rows]
        self.send_kv_rows = [t(a) for a in self.xp.send_kv_rows]
        self.send_heads = [t(a) for a in self.xp.send_heads]
        # reverse: my O_local rows per home rank (contiguous slices) and, on the
        # receiving side, where peer pieces land in my home shard
        lo, hi = home_range(self.rank, self.world, self.nb)
        self.o_slices = []
        off = 0
        for s in range(self.world):
            n = self.xp.recv_q_blocks[s]
            self.o_slices.append((off * 64, (off + n) * 64))
            off += n
        self.back_rows, self.back_heads = [], []
        for s in range(self.world):
            src = self.layouts[s]
            qb = src.q_blocks[(src.q_blocks >= lo) & (src.q_blocks < hi)]
            self.back_rows.append(t(_rows(qb - lo)))
            self.back_heads.append(t(src.heads))

    def __call__(self, q_home, k_home, v_home, out_home=None):
        import torch
        import torch.distributed as dist
        H = self.masks.num_heads
        Hu = len(self.me.heads)
        d = self.d
        dev = self.device
        dt = q_home.dtype
        world, rank = self.world, self.rank
        nq_loc = len(self.me.q_blocks)
        group_sizes = [len(g) for g in self.me.kv_groups]
        max_g = max(group_sizes) if group_sizes else 0
        q_loc = torch.empty(nq_loc * 64, Hu, d, device=dev, dtype=dt)
        kbuf = [torch.empty(max(max_g, 1) * 64, Hu, d, device=dev, dtype=dt) for _ in range(2)]
        vbuf = [torch.empty(max(max_g, 1) * 64, Hu, d, device=dev, dtype=dt) for _ in range(2)]

        # ---- 1. fused Ulysses + balancing all-to-all(v)
        ops, sends = [], []
        qoff = kvoff = 0
        for s in range(world):
            nq_s, nkv_s = self.xp.recv_q_blocks[s], self.xp.recv_kv_blocks[s]
            qdst = q_loc[qoff * 64:(qoff + nq_s) * 64]
            kdst = kbuf[0][kvoff * 64:(kvoff + nkv_s) * 64]
            vdst = vbuf[0][kvoff * 64:(kvoff + nkv_s) * 64]
            qoff += nq_s
            kvoff += nkv_s
            # what I send to s
            hq = self.send_heads[s]
            pq = q_home.index_select(0, self.send_q_rows[s]).index_select(1, hq) if len(self.send_q_rows[s]) else None
            pk = k_home.index_select(0, self.send_kv_rows[s]).index_select(1, hq) if len(self.send_kv_rows[s]) else None
            pv = v_home.index_select(0, self.send_kv_rows[s]).index_select(1, hq) if len(self.send_kv_rows[s]) else None
            if s == rank:
                if pq is not None:
                    qdst.copy_(pq)
                if pk is not None:
                    kdst.copy_(pk)
                    vdst.copy_(pv)
                continue
            # zero-size pieces are skipped on both sides (sizes are derived from
            # the same plan on sender and receiver, so the op lists match)
            for buf, dst in ((pq, qdst), (pk, kdst), (pv, vdst)):
                if buf is not None and buf.numel():
                    buf = buf.contiguous()
                    sends.append(buf)
                    ops.append(dist.P2POp(dist.isend, buf, s, group=self.group))
                if dst.numel():
                    ops.append(dist.P2POp(dist.irecv, dst, s, group=self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

        # ---- 2. ring periods: compute on the held group while the next arrives
        y = self.strategy.ring
        o_loc = torch.empty(nq_loc * 64, Hu, d, device=dev, dtype=dt)
        o_acc = torch.empty(nq_loc * 64, Hu, d, device=dev, dtype=torch.float32) if y > 1 else None
        lse_acc = torch.empty(Hu, nq_loc * 64, device=dev, dtype=torch.float32) if y > 1 else None
        cur = 0
        nxt_rank = self.me.u * y + (self.me.r + 1) % y
        prv_rank = self.me.u * y + (self.me.r - 1) % y
        for p in range(y):
            g = self.me.period_groups[p]
            n = group_sizes[g]
            reqs = []
            if p < y - 1:
                gn = self.me.period_groups[p + 1]
                nn = group_sizes[gn]
                ops = []
                if n and Hu:
                    ops += [dist.P2POp(dist.isend, kbuf[cur][:n * 64], prv_rank, group=self.group),
                            dist.P2POp(dist.isend, vbuf[cur][:n * 64], prv_rank, group=self.group)]
                if nn and Hu:
                    ops += [dist.P2POp(dist.irecv, kbuf[1 - cur][:nn * 64], nxt_rank, group=self.group),
                            dist.P2POp(dist.irecv, vbuf[1 - cur][:nn * 64], nxt_rank, group=self.group)]
                if ops:
                    reqs = dist.batch_isend_irecv(ops)
            self.attn_fn(self.me, p, q_loc, kbuf[cur][:n * 64], vbuf[cur][:n * 64], o_loc, o_acc, lse_acc,
                         p == 0, p == y - 1, self.me.kv_groups[g])
            for w in reqs:
                w.wait()
            cur = 1 - cur

        # ---- 3. reverse all-to-all(v): O back to the home layout
        T_home = q_home.shape[0]
        if self._symm is not None:
            # Rows already went home in the final launch's epilogue.  A rank
            # whose last period held no KV block launched nothing: its (merged
            # or zero) rows go home by peer-tensor copies instead.
            if len(self.me.kv_groups[self.me.period_groups[y - 1]]) == 0 and nq_loc and Hu:
                qmap, _ = scatter_maps(self.me, world, self.nb, self.S)
                hs = torch.as_tensor(self.me.heads, device=dev)
                elem_off = int(self._symm.offset) // self._home_out.element_size()
                for i, (r, row0, _n) in enumerate(qmap):
                    # the same peer address the kernel stores to (buffer_ptrs + offset)
                    peer = self._symm.get_buffer(int(r), tuple(self._home_out.shape), dt, storage_offset=elem_off)
                    peer[int(row0):int(row0) + 64, hs] = o_loc[i * 64:(i + 1) * 64]
            self._symm.barrier()
            res = self._home_out[:T_home]
            if out_home is None:
                return res.clone()
            out_home.copy_(res)
            return out_home
        if out_home is None:
            out_home = torch.empty(T_home, H, d, device=dev, dtype=dt)
        ops, recvs = [], []
        for s in range(world):
            a, b = self.o_slices[s]
            rows, heads = self.back_rows[s], self.back_heads[s]
            if s == rank:
                if b > a:
                    out_home[rows[:, None], heads[None, :]] = o_loc[a:b]
                continue
            if b > a and Hu:
                ops.append(dist.P2POp(dist.isend, o_loc[a:b].contiguous(), s, group=self.group))
            if len(rows) and len(heads):
                buf = torch.empty(len(rows), len(heads), d, device=dev, dtype=dt)
                recvs.append((buf, rows, heads))
                ops.append(dist.P2POp(dist.irecv, buf, s, group=self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        for buf, rows, heads in recvs:
            out_home[rows[:, None], heads[None, :]] = buf
        return out_home


def _cuda_attn_fn(masks: AttentionMaskSet, me: RankLayout, tokens: int, scatter=None) -> AttnFn:
    """K4 per ring period on the local buffers; schedules built once per plan.
    scatter: the final launch returns O to the home shards (fused step 3)."""
    from .attention import AttentionSchedule, accum_init

    scheds: Dict[int, AttentionSchedule] = {}

    def fn(layout, period, q_loc, k_buf, v_buf, out_loc, o_acc, lse_acc, first, last, kv_blocks):
        if len(layout.q_blocks) == 0 or len(layout.heads) == 0:
            return
        g = layout.period_groups[period]
        if g not in scheds:
            if len(kv_blocks) == 0:
                scheds[g] = None
            else:
                scheds[g] = AttentionSchedule().build(masks, head_ids=layout.heads, q_block_ids=layout.q_blocks,
                                                      kv_block_ids=kv_blocks, kv_tokens_global=tokens,
                                                      head_dim=q_loc.shape[-1])
        sc = scheds[g]
        y = layout.y
        if y == 1:
            if sc is None:
                out_loc.zero_()
            else:
                sc.launch(q_loc, k_buf, v_buf, out_loc, scatter=scatter)
            return
        if first:
            accum_init(o_acc, lse_acc)
        if sc is not None:
            sc.launch(q_loc, k_buf, v_buf, out_loc, o_accum=o_acc, lse_accum=lse_acc, accumulate=True,
                      finalize=last, scatter=scatter if last else None)
        elif last:
            out_loc.copy_(o_acc.to(out_loc.dtype))

    return fn


def scatter_maps(layout: RankLayout, world: int, nb: int, tokens: int):
    """Tables of the fused O return for one rank (dbsp_out_scatter): for each
    local Q block (ascending global id = local order) its home rank, first row
    in the home shard and valid rows; and local -> global heads."""
    starts = np.array([home_range(r, world, nb)[0] for r in range(world)], np.int64)
    qb = np.asarray(layout.q_blocks, np.int64)
    home = np.searchsorted(starts, qb, side="right") - 1
    row0 = (qb - starts[home]) * 64
    valid = np.minimum(64, tokens - qb * 64)
    return np.stack([home, row0, valid], axis=1), np.asarray(layout.heads, np.int64)


# ----------------------------------------------------------------------------- single-GPU simulation
def simulate_on_one_gpu(q, k, v, masks: AttentionMaskSet, strategy: ParallelStrategy, plan: PartitionPlan,
                        time_kernels: bool = True, reps: int = 5, fuse_return: bool = False):
    """Run every rank's per-period kernels of UxRy on ONE GPU (no exchange:
    the local buffers are gathered from the global tensors), merge exactly as
    the distributed path does, and time each (rank, period) launch with CUDA
    events.  fuse_return: the final launch of each rank writes O straight into
    G separate home-shard buffers through the kernel's scatter epilogue (the
    fused reverse all-to-all; on one GPU the "peers" are local allocations),
    and the result is their concatenation.  Returns (out [S,H,d],
    times_ms[period][rank]); each time is the median of `reps` launches."""
    import torch
    from .attention import AttentionSchedule, OutScatter, accum_init

    S, H, d = q.shape
    nb = S // 64
    layouts = rank_layouts(strategy, plan, masks.num_q_blocks, masks.num_kv_blocks)
    y = strategy.ring
    out = torch.zeros_like(q)
    G = len(layouts)
    homes = [torch.zeros((home_range(r, G, nb)[1] - home_range(r, G, nb)[0]) * 64, H, d, device=q.device,
                         dtype=q.dtype) for r in range(G)] if fuse_return else None
    times = [[0.0] * len(layouts) for _ in range(y)]
    for lay in layouts:
        if len(lay.heads) == 0 or len(lay.q_blocks) == 0:
            continue
        hs = torch.as_tensor(lay.heads, device=q.device)
        rows = torch.as_tensor(_rows(lay.q_blocks), device=q.device)
        q_loc = q.index_select(0, rows).index_select(1, hs).contiguous()
        o_loc = torch.empty_like(q_loc)
        o_acc = torch.empty(q_loc.shape, device=q.device, dtype=torch.float32)
        lse_acc = torch.empty(len(lay.heads), q_loc.shape[0], device=q.device, dtype=torch.float32)
        accum_init(o_acc, lse_acc)
        scat = None
        if fuse_return:
            qmap, hmap = scatter_maps(lay, G, nb, S)
            scat = OutScatter([t.data_ptr() for t in homes], qmap, hmap, H, q.device)
        for p in range(y):
            g = lay.period_groups[p]
            kvb = lay.kv_groups[g]
            if len(kvb) == 0:
                if p == y - 1:
                    o_loc.copy_(o_acc.to(o_loc.dtype)) if y > 1 else o_loc.zero_()
                    if fuse_return:  # no launch left to carry the return: copy as the NCCL path would
                        lo = np.asarray([home_range(r, G, nb)[0] for r in range(G)])
                        for i, b in enumerate(lay.q_blocks):
                            r = int(np.searchsorted(lo, b, side="right") - 1)
                            homes[r][(b - lo[r]) * 64:(b - lo[r] + 1) * 64, hs] = o_loc[i * 64:(i + 1) * 64]
                continue
            kr = torch.as_tensor(_rows(kvb), device=q.device)
            k_loc = k.index_select(0, kr).index_select(1, hs).contiguous()
            v_loc = v.index_select(0, kr).index_select(1, hs).contiguous()
            sc = AttentionSchedule().build(masks, head_ids=lay.heads, q_block_ids=lay.q_blocks,
                                           kv_block_ids=kvb, kv_tokens_global=S, head_dim=q.shape[-1])
            sc.upload()
            if time_kernels:
                # time on a scratch accumulator so the merge below is not disturbed
                oa = torch.empty_like(o_acc)
                la = torch.empty_like(lse_acc)
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                samples = []
                for _ in range(reps):
                    accum_init(oa, la)
                    ev[0].record()
                    if y == 1:
                        sc.launch(q_loc, k_loc, v_loc, o_loc)
                    else:
                        sc.launch(q_loc, k_loc, v_loc, o_loc, o_accum=oa, lse_accum=la, accumulate=True)
                    ev[1].record()
                    torch.cuda.synchronize()
                    samples.append(ev[0].elapsed_time(ev[1]))
                times[p][lay.rank] = float(np.median(samples))  # median: not the best-clock sample
            last = p == y - 1
            sk = scat if last else None
            if y == 1:
                sc.launch(q_loc, k_loc, v_loc, o_loc, scatter=sk)
            else:
                sc.launch(q_loc, k_loc, v_loc, o_loc, o_accum=o_acc, lse_accum=lse_acc, accumulate=True,
                          finalize=last, scatter=sk)
        if not fuse_return:
            out[rows[:, None], hs[None, :]] = o_loc
    torch.cuda.synchronize()
    if fuse_return:
        out = torch.cat(homes, 0)
    return out, times


def measured_rho(times: Sequence[Sequence[float]]) -> float:
    """rho_s of measured per-(period, rank) kernel times (Eq. 1 on seconds)."""
    t = np.asarray(times, dtype=np.float64)
    total = t.sum()
    if total == 0:
        return 1.0
    return float(t.max(axis=1).sum() * t.shape[1] / total)


def time_ranks_on_one_gpu(q, k, v, masks: AttentionMaskSet, strategy: ParallelStrategy, plan: PartitionPlan,
                          scratch=None, reps: int = 1, flags: Optional[int] = None):
    """Kernel times only: every (period, rank) K4 launch of UxRy timed on this
    GPU without gathering the local buffers.  K4's cost depends on the work
    list and the buffer footprint, not on the values, so each launch runs on
    contiguous views [local tokens, local heads, d] carved from flat scratch
    buffers of the global size (filled once from q/k/v).  Used for long
    measured sweeps (config E), where the per-call gathers of
    simulate_on_one_gpu would dominate.  Returns times_ms[period][rank]."""
    import torch
    from .attention import AttentionSchedule

    S, H, d = q.shape
    layouts = rank_layouts(strategy, plan, masks.num_q_blocks, masks.num_kv_blocks)
    y = strategy.ring
    if scratch is None:
        scratch = time_scratch(q, k, v)
    qf, kf, vf, of, af, lf = scratch
    times = [[0.0] * len(layouts) for _ in range(y)]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for lay in layouts:
        hl, nq = len(lay.heads), len(lay.q_blocks)
        if hl == 0 or nq == 0:
            continue
        sq = nq * 64
        q_loc = qf[:sq * hl * d].view(sq, hl, d)
        o_loc = of[:sq * hl * d].view(sq, hl, d)
        o_acc = af[:sq * hl * d].view(sq, hl, d)
        l_acc = lf[:sq * hl].view(hl, sq)
        for p in range(y):
            kvb = lay.kv_groups[lay.period_groups[p]]
            if len(kvb) == 0:
                continue
            sk = len(kvb) * 64
            k_loc = kf[:sk * hl * d].view(sk, hl, d)
            v_loc = vf[:sk * hl * d].view(sk, hl, d)
            sc = AttentionSchedule().build(masks, head_ids=lay.heads, q_block_ids=lay.q_blocks,
                                           kv_block_ids=kvb, kv_tokens_global=S, flags=flags, head_dim=d)
            sc.upload()
            best = float("inf")
            for _ in range(reps):
                ev[0].record()
                if y == 1:
                    sc.launch(q_loc, k_loc, v_loc, o_loc)
                else:
                    sc.launch(q_loc, k_loc, v_loc, o_loc, o_accum=o_acc, lse_accum=l_acc, accumulate=True)
                ev[1].record()
                ev[1].synchronize()
                best = min(best, ev[0].elapsed_time(ev[1]))
            times[p][lay.rank] = best
    return times


def rank_launcher(q, k, v, masks: AttentionMaskSet, strategy: ParallelStrategy, plan: PartitionPlan,
                  rank: int, scratch=None):
    """A callable that launches ONE rank's per-period K4 kernels of UxRy on
    this GPU (the same launches as time_ranks_on_one_gpu: contiguous views of
    the rank's local footprint), for measuring what runs beside that rank's
    critical path -- e.g. the next call's planning."""
    from .attention import AttentionSchedule, accum_init
    S, H, d = q.shape
    lay = rank_layouts(strategy, plan, masks.num_q_blocks, masks.num_kv_blocks)[rank]
    y = strategy.ring
    if scratch is None:
        scratch = time_scratch(q, k, v)
    qf, kf, vf, of, af, lf = scratch
    hl, nq = len(lay.heads), len(lay.q_blocks)
    sq = nq * 64
    q_loc, o_loc = qf[:sq * hl * d].view(sq, hl, d), of[:sq * hl * d].view(sq, hl, d)
    o_acc, l_acc = af[:sq * hl * d].view(sq, hl, d), lf[:sq * hl].view(hl, sq)
    calls = []
    for p in range(y):
        kvb = lay.kv_groups[lay.period_groups[p]]
        if len(kvb) == 0 or hl == 0 or nq == 0:
            continue
        sk = len(kvb) * 64
        sc = AttentionSchedule().build(masks, head_ids=lay.heads, q_block_ids=lay.q_blocks, kv_block_ids=kvb,
                                       kv_tokens_global=S, head_dim=d)
        sc.upload()
        calls.append((sc, kf[:sk * hl * d].view(sk, hl, d), vf[:sk * hl * d].view(sk, hl, d), p == y - 1))

    def launch(stream=None):
        if y > 1 and calls:
            accum_init(o_acc, l_acc)
        for sc, k_loc, v_loc, last in calls:
            if y == 1:
                sc.launch(q_loc, k_loc, v_loc, o_loc, stream=stream)
            else:
                sc.launch(q_loc, k_loc, v_loc, o_loc, o_accum=o_acc, lse_accum=l_acc, accumulate=True,
                          finalize=last, stream=stream)
    return launch


def time_scratch(q, k, v):
    """Flat scratch buffers for time_ranks_on_one_gpu (values copied from q/k/v)."""
    import torch
    S, H, d = q.shape
    f32 = dict(device=q.device, dtype=torch.float32)
    return (q.reshape(-1).clone(), k.reshape(-1).clone(), v.reshape(-1).clone(),
            torch.empty(S * H * d, device=q.device, dtype=q.dtype), torch.zeros(S * H * d, **f32),
            torch.full((H * S,), float("-inf"), **f32))


# ----------------------------------------------------------------------------- C++ executor (C ABI)
class NativeSPContext:
    """The C-ABI sequence-parallel call (csrc/sp_exec.cu): NCCL communicator,
    fused all-to-all(v), ring periods of K4 with the KV exchange on a
    communication stream, reverse all-to-all(v) -- all in C++.  One per
    process/GPU; rank 0's NCCL id reaches the others through `broadcast_id`
    (e.g. torch.distributed.broadcast_object_list)."""

    def __init__(self, rank: int, world: int, broadcast_id: Callable[[bytes], bytes]):
        import ctypes as C
        from . import _lib as L
        from .planner import check
        buf = (C.c_uint8 * 128)()
        if rank == 0:
            check(L.lib().dbsp_nccl_unique_id(C.cast(buf, C.c_void_p), 128))
        uid = broadcast_id(bytes(buf) if rank == 0 else b"")
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        check(L.lib().dbsp_sp_context_create(rank, world, C.cast(buf, C.c_void_p), C.byref(h)))
        self._h = h
        self.rank, self.world = rank, world

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            from . import _lib as L
            L.lib().dbsp_sp_context_destroy(h)
            self._h = None

    def __call__(self, masks: AttentionMaskSet, strategy: ParallelStrategy, plan: PartitionPlan,
                 q_home, k_home, v_home, out_home=None, stream=None):
        import ctypes as C
        import torch
        from . import _lib as L
        from .planner import check
        S = masks.num_q_blocks * 64
        d = q_home.shape[2]
        if out_home is None:
            out_home = torch.empty_like(q_home)
        st = stream if stream is not None else torch.cuda.current_stream(q_home.device)
        check(L.lib().dbsp_sp_attention(self._h, C.byref(masks.c()), L.StrategyT(strategy.ulysses, strategy.ring),
                                        C.byref(plan.c()), C.c_void_p(q_home.data_ptr()),
                                        C.c_void_p(k_home.data_ptr()), C.c_void_p(v_home.data_ptr()),
                                        C.c_void_p(out_home.data_ptr()), S, d, C.c_void_p(st.cuda_stream)))
        return out_home

    def set_timing(self, on: bool) -> None:
        """Per-period K4 events on the compute stream for the next calls."""
        from . import _lib as L
        from .planner import check
        check(L.lib().dbsp_sp_set_timing(self._h, int(on)))

    def period_ms(self) -> List[float]:
        """K4 milliseconds per ring period of the last timed call (syncs on its events)."""
        import ctypes as C
        from . import _lib as L
        from .planner import check
        buf = (C.c_float * 64)()
        n = C.c_uint32()
        check(L.lib().dbsp_sp_period_ms(self._h, buf, 64, C.byref(n)))
        return [float(buf[i]) for i in range(n.value)]

    def synchronize(self, stream=None, timeout_ms: int = 60000) -> None:
        """Wait for the last call, polling NCCL's asynchronous error state; an
        error or a timeout aborts the communicator and raises CudaError."""
        import ctypes as C
        import torch
        from . import _lib as L
        from .planner import check
        st = stream if stream is not None else torch.cuda.current_stream()
        check(L.lib().dbsp_sp_synchronize(self._h, C.c_void_p(st.cuda_stream), int(timeout_ms)))


def native_sp_simulated(q, k, v, masks: AttentionMaskSet, strategy: ParallelStrategy, plan: PartitionPlan):
    """dbsp_sp_attention_simulated: all G ranks of the C++ executor on this GPU
    (device copies as the transport).  q/k/v: global [S, H, d]; returns O [S, H, d]."""
    import ctypes as C
    import torch
    from . import _lib as L
    from .planner import check
    S, H, d = q.shape
    nb = S // 64
    G = strategy.gpus()
    sl = [slice(home_range(g, G, nb)[0] * 64, home_range(g, G, nb)[1] * 64) for g in range(G)]
    qs, ks, vs = ([t[s].contiguous() for s in sl] for t in (q, k, v))
    os_ = [torch.empty_like(x) for x in qs]
    arr = lambda ts: (C.c_void_p * G)(*[t.data_ptr() for t in ts])
    check(L.lib().dbsp_sp_attention_simulated(C.byref(masks.c()), L.StrategyT(strategy.ulysses, strategy.ring),
                                              C.byref(plan.c()), arr(qs), arr(ks), arr(vs), arr(os_), S, d,
                                              C.c_void_p(torch.cuda.current_stream(q.device).cuda_stream)))
    return torch.cat(os_, 0)


# ----------------------------------------------------------------------------- per-call runtime
class SPLayerRunner:
    """One attention layer per call under db-SP, the way the paper's runtime
    runs it: every call, select() on the live masks picks
    the U x R split and its dual-balanced plan (selector.hpp:55-75, per-layer
    SelectorState with P_s head-plan reuse), then the SP executor runs it.

    Planning is pipelined: prefetch(layer', masks') computes the selection for
    the NEXT call right after this call's GPU work has been enqueued, so it
    overlaps that work instead of sitting on the critical path.  With the GPU
    selector (planner="device", dbsp_select_device) the mask integers run on a
    separate planner stream and the host only waits for that stream; with
    planner="host" the C++ selector runs on the host (the GIL is released in
    the C call).  Every rank plans the same masks with the same state, so the
    ranks agree without exchanging plans.

    executor: "native" (C++/NCCL, csrc/sp_exec.cu) or "python" (SPAttention,
    torch.distributed; takes attn_fn for CPU tests).  balance: "dbsp" runs the
    selected plan, "uniform" the selected strategy's default plan (the USP
    baseline)."""

    def __init__(self, rank: int, world: int, profile: MachineProfile, *, config: Optional[PlannerConfig] = None,
                 executor: str = "native", planner: str = "device", device=None,
                 broadcast_id: Optional[Callable[[bytes], bytes]] = None, attn_fn: Optional[AttnFn] = None,
                 group=None, balance: str = "dbsp", native_ctx: Optional["NativeSPContext"] = None):
        if executor not in ("native", "python") or planner not in ("device", "host") or \
                balance not in ("dbsp", "uniform"):
            raise ConfigError("executor must be native|python, planner device|host, balance dbsp|uniform")
        self.rank, self.world = rank, world
        self.profile, self.config = profile, config or PlannerConfig()
        self.state = SelectorState(world)
        self.executor, self.planner, self.balance = executor, planner, balance
        self.device, self.group, self.attn_fn = device, group, attn_fn
        self._native = None
        if executor == "native":
            self._native = native_ctx or NativeSPContext(rank, world, broadcast_id)
        self._py: Dict[tuple, SPAttention] = {}
        self._next: Dict[int, object] = {}
        self._plan_stream = None
        if planner == "device":
            import torch
            # high priority: the selector's small kernels take SMs at the next
            # CTA boundary of the running attention instead of queueing behind it
            self._plan_stream = torch.cuda.Stream(device, priority=-1)
        self.calls = self.prefetched = 0
        self.plan_host_ms: List[float] = []  # host time of every selection
        self.exposed_host_ms = 0.0           # selections that ran inside a call (nothing prefetched)
        self.last = None

    def _select(self, layer: int, masks: AttentionMaskSet, words=None):
        import time
        t0 = time.perf_counter()
        if self.planner == "device":
            import torch
            with torch.cuda.stream(self._plan_stream):
                if words is None:
                    words = torch.from_numpy(np.ascontiguousarray(masks.words).view(np.int64)).to(
                        self.device, non_blocking=False)
                sel = _P.select_device(layer, words, masks.num_kv_blocks, self.profile, self.config, self.state,
                                       stream=self._plan_stream)
        else:
            sel = _P.select(layer, masks, self.profile, self.config, self.state)
        self.plan_host_ms.append((time.perf_counter() - t0) * 1e3)
        return sel

    def prefetch(self, layer: int, masks: AttentionMaskSet, words=None) -> None:
        """Selection for the next call of `layer` (call right after __call__)."""
        self._next[layer] = (self._select(layer, masks, words), masks)
        self.prefetched += 1

    def __call__(self, layer: int, masks: AttentionMaskSet, q_home, k_home, v_home, out_home=None,
                 words=None, stream=None):
        nxt = self._next.pop(layer, None)
        if nxt is not None and nxt[1] is masks:
            sel = nxt[0]
        else:
            sel = self._select(layer, masks, words)
            self.exposed_host_ms += self.plan_host_ms[-1]
        st = sel.strategy
        plan = sel.outcome.plan if self.balance == "dbsp" else _P.default_plan(masks, st)
        self.calls += 1
        self.last = sel
        if self._native is not None:
            return self._native(masks, st, plan, q_home, k_home, v_home, out_home, stream=stream)
        key = (str(st), self.balance, plan.head_assignment.tobytes(), plan.q_assignment.tobytes(),
               plan.kv_assignment.tobytes(), id(masks))
        sp = self._py.get(key)
        if sp is None:
            self._py.clear()
            sp = SPAttention(masks, st, plan, masks.num_q_blocks * 64, q_home.shape[2], self.rank, self.world,
                             self.device, attn_fn=self.attn_fn, group=self.group)
            self._py[key] = sp
        return sp(q_home, k_home, v_home, out_home)

    @property
    def native(self) -> Optional[NativeSPContext]:
        return self._native
