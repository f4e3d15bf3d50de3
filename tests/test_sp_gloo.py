"""Multi-process check of the SP execution layer (paper_2511_23113_b200/sp.py)
on CPU with the gloo backend: the fused Ulysses+balancing all-to-all(v), the
ring KV exchange and the reverse all-to-all(v) reproduce single-process
attention for every U x R split, with uniform (default) and db-SP plans.

The per-period attention is the CPU oracle here (injected attn_fn, test
infrastructure); on GPUs the same executor calls the sm_100a kernel.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2511_23113_b200 as D
from paper_2511_23113_b200.sp import SPAttention, home_range

S, H, DH = 1024, 6, 16
NB = S // 64


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _words(dense):
    h, nq, nk = dense.shape
    wpr = (nk + 63) // 64
    pad = np.zeros((h, nq, wpr * 64), bool)
    pad[:, :, :nk] = dense
    return np.packbits(pad.reshape(h, nq, wpr, 64), axis=-1, bitorder="little").view(np.uint64).reshape(h, nq, wpr)


def oracle_attn_fn(dense):
    """K4 semantics on CPU: partial attention of this period + LSE merge."""
    def fn(layout, period, q_loc, k_buf, v_buf, out_loc, o_acc, lse_acc, first, last, kv_blocks):
        hq = layout.heads
        if len(hq) == 0 or len(layout.q_blocks) == 0:
            return
        local = dense[np.ix_(hq, layout.q_blocks, kv_blocks)] if len(kv_blocks) else np.zeros(
            (len(hq), len(layout.q_blocks), 1), bool)
        nk = max(len(kv_blocks), 1)
        kb = k_buf.numpy() if len(kv_blocks) else np.zeros((64, len(hq), DH), np.float32)
        vb = v_buf.numpy() if len(kv_blocks) else np.zeros((64, len(hq), DH), np.float32)
        o, l = oracle.sparse_attention(q_loc.numpy(), kb, vb, _words(local), nk)
        o, l = torch.from_numpy(o), torch.from_numpy(l)
        if layout.y == 1:
            out_loc.copy_(o)
            return
        if first:
            o_acc.zero_()
            lse_acc.fill_(-float("inf"))
        mx = torch.maximum(lse_acc, l)
        w_old = torch.where(torch.isinf(lse_acc), torch.zeros_like(mx), torch.exp(lse_acc - mx))
        w_new = torch.where(torch.isinf(l), torch.zeros_like(mx), torch.exp(l - mx))
        den = w_old + w_new
        safe = torch.where(den > 0, den, torch.ones_like(den))
        o_acc.mul_((w_old / safe).T[:, :, None]).add_(o * (w_new / safe).T[:, :, None])
        lse_acc.copy_(torch.where(den > 0, mx + torch.log(safe), mx))
        if last:
            out_loc.copy_(o_acc)
    return fn


def _worker(rank, world, port, strategy, balanced, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        masks = D.generate_mask_set(D.GeneratorSpec(H, NB, NB, 64, "clustered", 0.2, 0.6, 1.0, 5))
        dense = masks.to_dense()
        g = torch.Generator().manual_seed(0)
        q, k, v = (torch.randn(S, H, DH, generator=g) for _ in range(3))
        st = D.parse_strategy(strategy)
        plan = D.plan_dual(masks, st).plan if balanced else D.default_plan(masks, st)
        lo, hi = home_range(rank, world, NB)
        sp = SPAttention(masks, st, plan, S, DH, rank, world, torch.device("cpu"),
                         attn_fn=oracle_attn_fn(dense))
        out = sp(q[lo * 64:hi * 64].contiguous(), k[lo * 64:hi * 64].contiguous(),
                 v[lo * 64:hi * 64].contiguous())
        ref, _ = oracle.sparse_attention(q.numpy(), k.numpy(), v.numpy(), masks.words, NB)
        err = float(np.abs(out.numpy() - ref[lo * 64:hi * 64]).max())
        results[rank] = err
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,strategy,balanced", [
    (2, "U2R1", False), (2, "U1R2", False), (2, "U1R2", True), (2, "U2R1", True),
    (4, "U2R2", True), (4, "U1R4", True), (4, "U4R1", True), (4, "U2R2", False),
])
def test_sp_matches_single_process(world, strategy, balanced):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, strategy, balanced, results))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0, f"rank exited with {p.exitcode}"
    assert len(results) == world
    assert max(results.values()) < 1e-5, dict(results)


def test_rank_layouts_partition_everything():
    from paper_2511_23113_b200.sp import rank_layouts
    masks = D.generate_mask_set(D.GeneratorSpec(8, 16, 16, 64, "random", 0.3, 0.6, 1.0, 2))
    for st in D.enumerate_strategies(8):
        plan = D.plan_dual(masks, st).plan
        lays = rank_layouts(st, plan, 16, 16)
        cover = np.zeros((8, 16), int)
        for lay in lays:
            for h in lay.heads:
                cover[h, lay.q_blocks] += 1
        assert np.all(cover == 1)  # every (head, Q block) owned by exactly one GPU
        for lay in lays:  # each rank visits every KV group once over the ring
            assert sorted(lay.period_groups) == list(range(st.ring))
