"""GPU parity of the sm_100a block-sparse attention kernel (K4) against the CPU
oracle (oracle/attention_ref.c, fp32 inputs, double accumulation).

Tolerance (north_star): bf16 output within max-abs 2e-2 and rel-L2 1e-2 of the
oracle.  Inputs are the bf16-rounded Q/K/V, so the comparison measures the
kernel's arithmetic, not input quantisation.
"""
import math
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # test infrastructure: the checker
import paper_2511_23113_b200 as D
from paper_2511_23113_b200.attention import AttentionSchedule, accum_init, sparse_attention

pytestmark = pytest.mark.gpu

MAX_ABS = 2e-2
REL_L2 = 1e-2


def make_qkv(S, H, d, seed, Sk=None):
    g = torch.Generator().manual_seed(seed)
    Sk = Sk or S
    q = torch.randn(S, H, d, generator=g).to(torch.bfloat16)
    k = torch.randn(Sk, H, d, generator=g).to(torch.bfloat16)
    v = torch.randn(Sk, H, d, generator=g).to(torch.bfloat16)
    return q, k, v


def check(out, ref, what=""):
    out = out.float().cpu().numpy()
    diff = np.abs(out - ref)
    mx = float(diff.max()) if diff.size else 0.0
    rel = float(np.linalg.norm(out - ref) / max(np.linalg.norm(ref), 1e-30))
    assert np.isfinite(out).all(), f"{what}: non-finite output"
    assert mx <= MAX_ABS and rel <= REL_L2, f"{what}: max_abs={mx:.3e} rel_l2={rel:.3e} at {np.unravel_index(diff.argmax(), diff.shape)}"
    return mx, rel


def check_rows(out, q, k, v, masks, rows, what=""):
    """Sampled (head, Q-block) rows of a device output against the oracle."""
    rows = np.asarray(rows, np.int32)
    nk = masks.num_kv_blocks
    ref, _ = oracle.sparse_attention(q.float().cpu().numpy(), k.float().cpu().numpy(),
                                     v.float().cpu().numpy(), masks.words, nk, rows=rows)
    got = out.float().cpu().numpy()
    S = got.shape[0]
    idx_tok = np.concatenate([np.arange(b * 64, min(b * 64 + 64, S)) for _, b in rows])
    idx_head = np.concatenate([np.full(min(64, S - b * 64), h) for h, b in rows])
    a, r = got[idx_tok, idx_head], ref[idx_tok, idx_head]
    mx = float(np.abs(a - r).max())
    rel = float(np.linalg.norm(a - r) / max(np.linalg.norm(r), 1e-30))
    assert mx <= MAX_ABS and rel <= REL_L2, f"{what}: max_abs={mx:.3e} rel_l2={rel:.3e}"


def run_case(H, S, d, pattern, dmin, dmax, seed, Sk=None, lse=True):
    Sk = Sk or S
    nq, nk = -(-S // 64), -(-Sk // 64)
    masks = D.generate_mask_set(D.GeneratorSpec(H, nq, nk, 64, pattern, dmin, dmax, 1.0, seed))
    q, k, v = make_qkv(S, H, d, seed, Sk)
    ref, ref_lse = oracle.sparse_attention(q.float().numpy(), k.float().numpy(), v.float().numpy(),
                                           masks.words, nk)
    out, out_lse = sparse_attention(q.cuda(), k.cuda(), v.cuda(), masks, return_lse=True)
    torch.cuda.synchronize()
    mx, rel = check(out, ref, f"H{H} S{S} Sk{Sk} d{d} {pattern}")
    if lse:
        ol = out_lse.cpu().numpy()
        fin = np.isfinite(ref_lse)
        assert np.array_equal(fin, np.isfinite(ol)), "LSE -inf pattern differs"
        assert np.abs(ol[fin] - ref_lse[fin]).max() < 1e-2
    return mx, rel


def test_config_a_toy():
    # BASELINE config A: 8 heads, 4096 tokens, d=64, 50% random block mask.
    run_case(8, 4096, 64, "random", 0.5, 0.5, 1)


@pytest.mark.parametrize("pattern", ["random", "banded", "clustered"])
def test_d128_patterns(pattern):
    run_case(4, 2048, 128, pattern, 0.1, 0.6, 3)


def test_ragged_tokens_and_single_tail_block():
    run_case(3, 1000, 64, "random", 0.3, 0.7, 5)            # odd number of Q blocks, partial tail
    run_case(2, 4100, 128, "clustered", 0.2, 0.5, 6, Sk=3000)  # Sq != Sk, both ragged


def test_dense_and_empty_rows():
    H, S, d = 2, 1024, 128
    nq = nk = S // 64
    dense = np.ones((H, nq, nk), bool)
    dense[0, 3, :] = False          # a Q block with no dense tile -> O = 0, LSE = -inf
    dense[1, :, 5] = False
    masks = D.AttentionMaskSet.from_dense(dense)
    q, k, v = make_qkv(S, H, d, 9)
    ref, ref_lse = oracle.sparse_attention(q.float().numpy(), k.float().numpy(), v.float().numpy(),
                                           masks.words, nk)
    out, lse = sparse_attention(q.cuda(), k.cuda(), v.cuda(), masks, return_lse=True)
    torch.cuda.synchronize()
    check(out, ref, "dense/empty")
    assert torch.all(out[3 * 64:4 * 64, 0] == 0)
    assert torch.all(torch.isinf(lse[0, 3 * 64:4 * 64]))


def test_large_scores_rescale_path():
    # Growing score scale forces the lazy O rescale (max grows by > 2^8).
    H, S, d = 2, 2048, 64
    nq = nk = S // 64
    masks = D.generate_mask_set(D.GeneratorSpec(H, nq, nk, 64, "random", 0.6, 0.6, 1.0, 4))
    q, k, v = make_qkv(S, H, d, 10)
    ramp = torch.linspace(0.2, 6.0, S).view(S, 1, 1)
    k = (k.float() * ramp).to(torch.bfloat16)
    ref, _ = oracle.sparse_attention(q.float().numpy(), k.float().numpy(), v.float().numpy(),
                                     masks.words, nk)
    out = sparse_attention(q.cuda(), k.cuda(), v.cuda(), masks)
    torch.cuda.synchronize()
    check(out, ref, "rescale")


def test_ring_accumulate_equals_full():
    # Two "ring periods" over disjoint KV-block groups merged in the epilogue
    # reproduce the one-shot result (ring merge).
    H, S, d = 4, 2048, 128
    nq = nk = S // 64
    masks = D.generate_mask_set(D.GeneratorSpec(H, nq, nk, 64, "clustered", 0.2, 0.6, 1.0, 12))
    q, k, v = make_qkv(S, H, d, 13)
    ref, _ = oracle.sparse_attention(q.float().numpy(), k.float().numpy(), v.float().numpy(),
                                     masks.words, nk)
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    o_acc = torch.empty(S, H, d, dtype=torch.float32, device="cuda")
    l_acc = torch.empty(H, S, dtype=torch.float32, device="cuda")
    out = torch.empty_like(qd)
    accum_init(o_acc, l_acc)
    groups = [np.arange(0, nk, 2), np.arange(1, nk, 2)]
    scheds = []
    for i, g in enumerate(groups):
        kv_local = torch.cat([kd[b * 64:(b + 1) * 64] for b in g]).contiguous()
        vv_local = torch.cat([vd[b * 64:(b + 1) * 64] for b in g]).contiguous()
        sc = AttentionSchedule().build(masks, kv_block_ids=g, kv_tokens_global=S)
        sc.launch(qd, kv_local, vv_local, out, o_accum=o_acc, lse_accum=l_acc, accumulate=True,
                  finalize=(i == len(groups) - 1))
        scheds.append((sc, kv_local, vv_local))
    torch.cuda.synchronize()
    check(out, ref, "ring-accumulate")


@pytest.mark.parametrize("strategy", ["U2R2", "U1R4", "U4R1"])
def test_partitioned_execution_matches_one_shot(strategy):
    # Every rank's per-period kernels of the SP layout (accumulate + finalize
    # merge across ring periods) reproduce the single-launch output.
    from paper_2511_23113_b200.sp import simulate_on_one_gpu
    H, S, d = 8, 2048, 128
    nb = S // 64
    masks = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, "clustered", 0.15, 0.45, 1.0, 7))
    q, k, v = (t.cuda() for t in make_qkv(S, H, d, 21))
    full = sparse_attention(q, k, v, masks)
    st = D.parse_strategy(strategy)
    for plan in (D.default_plan(masks, st), D.plan_dual(masks, st).plan):
        out, times = simulate_on_one_gpu(q, k, v, masks, st, plan, time_kernels=False)
        assert float((out.float() - full.float()).abs().max()) < 1e-2


@pytest.mark.parametrize("flags", [1, 1 | 8 | 16 | 128, 1 | 256])
@pytest.mark.parametrize("pattern", ["clustered", "random", "dense"])
@pytest.mark.parametrize("case", ["identity", "rank_view", "ragged"])
def test_device_schedule_matches_host(case, pattern, flags):
    # K2 on the GPU builds exactly the host builder's list (items, order,
    # entries) for the pair layout, the CTA-pair quad layout and the d=128
    # auto choice (which resolves to the pair layout since round 2).
    from paper_2511_23113_b200.sp import rank_layouts
    H, nb = 8, 96
    if pattern == "dense":
        masks = D.AttentionMaskSet.from_dense(np.ones((H, nb, nb), bool))
    else:
        masks = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, pattern, 0.1, 0.6, 1.0, 11))
    words = torch.from_numpy(masks.words.view(np.int64)).cuda()
    kw = {}
    S = nb * 64
    if case == "rank_view":
        st = D.ParallelStrategy(2, 4)
        lay = rank_layouts(st, D.plan_dual(masks, st).plan, nb, nb)[5]
        kw = dict(head_ids=lay.heads, q_block_ids=lay.q_blocks, kv_block_ids=lay.kv_groups[2])
    if case == "ragged":
        S = nb * 64 - 37
        kw = dict(q_block_ids=list(range(nb - 3)))  # a partial quad at the end
    host = AttentionSchedule().build(masks, kv_tokens_global=S, flags=flags, **kw)
    dev = AttentionSchedule().build_device(words, nb, kv_tokens_global=S, flags=flags, **kw)
    assert host.layout() == dev.layout()
    if flags == 1 | 256:
        assert dev.layout()["kernel"] == "pair_items"
    hi, he = host.download()
    di, de = dev.download()
    assert np.array_equal(hi, di)
    assert np.array_equal(he, de)
    assert host.stats() == dev.stats()


@pytest.mark.parametrize("flags", [1 | 256, 1 | 8 | 16 | 128])
@pytest.mark.parametrize("pattern", ["clustered", "random"])
def test_device_built_schedule_launch_equals_host(pattern, flags):
    # A device-built schedule (K2) runs the same kernel over the same list as
    # the host-built one: the output is equal bit for bit.
    H, S, d = 6, 3000, 128
    nb = -(-S // 64)
    masks = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, pattern, 0.15, 0.5, 1.0, 13))
    q, k, v = (t.cuda() for t in make_qkv(S, H, d, 14))
    host = AttentionSchedule().build(masks, kv_tokens_global=S, flags=flags)
    ref = torch.empty_like(q)
    host.launch(q, k, v, ref)
    words = torch.from_numpy(masks.words.view(np.int64)).cuda()
    dev = AttentionSchedule().build_device(words, nb, kv_tokens_global=S, flags=flags)
    out = torch.full_like(q, 5.0)
    dev.launch(q, k, v, out)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_device_schedule_attention_equal():
    H, S, d = 8, 4096, 128
    nb = S // 64
    masks = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, "clustered", 0.15, 0.45, 1.0, 2))
    q, k, v = (t.cuda() for t in make_qkv(S, H, d, 3))
    a = sparse_attention(q, k, v, masks)
    b = sparse_attention(q, k, v, masks, device_schedule=True)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_host_streaming_equals_one_shot():
    # Head-chunked H2D / K4 / D2H overlap returns exactly the one-shot result.
    from paper_2511_23113_b200.e2e import HostStreamingAttention
    H, S, d = 10, 2048, 128
    nb = S // 64
    masks = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, "clustered", 0.15, 0.45, 1.0, 4))
    q, k, v = make_qkv(S, H, d, 8)
    ref = sparse_attention(q.cuda(), k.cuda(), v.cuda(), masks).cpu()
    run = HostStreamingAttention(S, H, d, chunks=3)
    qh, kh, vh = (t.pin_memory() for t in (q, k, v))
    for _ in range(2):
        out = run(qh, kh, vh, masks)
        torch.cuda.synchronize()
        assert torch.equal(out, ref)


@pytest.mark.parametrize("flags", [1 | 8 | 16 | 128, 1 | 256])
@pytest.mark.parametrize("H,S,Sk,pattern", [(4, 2048, None, "clustered"), (3, 1000, 2000, "random"),
                                             (5, 4096, None, "banded"), (2, 448, 4000, "random")])
def test_two_stage_kernel(H, S, Sk, pattern, flags):
    # quad schedule -> the CTA-pair kernel (two CTAs x two split-KV stages,
    # 128-key steps), and the auto choice; odd block counts exercise padded
    # rows of the quad and the masked second half of an odd-length step.
    d = 128
    Sk = Sk or S
    nq, nk = -(-S // 64), -(-Sk // 64)
    masks = D.generate_mask_set(D.GeneratorSpec(H, nq, nk, 64, pattern, 0.15, 0.6, 1.0, 17))
    q, k, v = make_qkv(S, H, d, 19, Sk)
    ref, ref_lse = oracle.sparse_attention(q.float().numpy(), k.float().numpy(), v.float().numpy(),
                                           masks.words, nk)
    sc = AttentionSchedule().build(masks, kv_tokens_global=Sk, flags=flags)
    out = torch.empty(S, H, d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(H, S, device="cuda", dtype=torch.float32)
    sc.launch(q.cuda(), k.cuda(), v.cuda(), out, lse=lse)
    torch.cuda.synchronize()
    check(out, ref, f"two-stage flags{flags} d{d} H{H} S{S} Sk{Sk} {pattern}")
    fin = np.isfinite(ref_lse)
    assert np.abs(lse.cpu().numpy()[fin] - ref_lse[fin]).max() < 1e-2
    assert np.all(np.isneginf(lse.cpu().numpy()[~fin]))


@pytest.mark.parametrize("flags", [1, 1 | 8 | 16 | 128])
def test_two_stage_ring_accumulate(flags):
    # Two KV periods through accumulate + finalize on the two-stage kernel
    # equal one pass over all KV (the K5 merge in its epilogue).
    H, S, d = 3, 1536, 128
    nb = S // 64
    masks = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, "clustered", 0.2, 0.5, 1.0, 5))
    q, k, v = make_qkv(S, H, d, 7)
    ref, _ = oracle.sparse_attention(q.float().numpy(), k.float().numpy(), v.float().numpy(), masks.words, nb)
    qc, kc, vc = q.cuda(), k.cuda(), v.cuda()
    o_acc = torch.empty(S, H, d, device="cuda", dtype=torch.float32)
    l_acc = torch.empty(H, S, device="cuda", dtype=torch.float32)
    accum_init(o_acc, l_acc)
    out = torch.empty(S, H, d, device="cuda", dtype=torch.bfloat16)
    half = nb // 2
    for p, ids in enumerate((list(range(half)), list(range(half, nb)))):
        sc = AttentionSchedule().build(masks, kv_block_ids=ids, kv_tokens_global=S, flags=flags)
        sl = slice(ids[0] * 64, (ids[-1] + 1) * 64)
        sc.launch(qc, kc[sl].contiguous(), vc[sl].contiguous(), out, o_accum=o_acc, lse_accum=l_acc,
                  accumulate=True, finalize=p == 1)
    torch.cuda.synchronize()
    check(out, ref, "two-stage ring accumulate")


@pytest.mark.parametrize("fuse_return", [False, True])
def test_nccl_executor_single_rank(fuse_return):
    # The NCCL-backed executor (the N>1 bench leg) on a 1-rank group: device
    # index tensors, buffers and the K4 launch path through SPAttention.
    import socket

    import torch.distributed as dist

    from paper_2511_23113_b200.sp import SPAttention
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        H, S, d = 4, 2048, 128
        nb = S // 64
        masks = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, "clustered", 0.2, 0.5, 1.0, 3))
        q, k, v = (t.cuda() for t in make_qkv(S, H, d, 5))
        st = D.ParallelStrategy(1, 1)
        sp = SPAttention(masks, st, D.plan_dual(masks, st).plan, S, d, 0, 1, torch.device("cuda"),
                         fuse_return=fuse_return)
        out = sp(q, k, v)
        ref = sparse_attention(q, k, v, masks)
        torch.cuda.synchronize()
        assert torch.equal(out, ref)
    finally:
        dist.destroy_process_group()


def test_mask_stats_device_exact():
    m = D.generate_mask_set(D.GeneratorSpec(40, 512, 512, 64, "clustered", 0.15, 0.45, 1.0, 1))
    words = torch.from_numpy(m.words.view(np.int64)).cuda()
    hc, rw, cw = D.mask_stats_device(words, 512)
    grid = D.summed_grid(m).reshape(512, 512).astype(np.int64)
    assert hc.cpu().tolist() == D.blocks_per_head(m)
    assert rw.cpu().numpy().tolist() == grid.sum(1).tolist()
    assert cw.cpu().numpy().tolist() == grid.sum(0).tolist()


def test_errors_are_loud():
    m = D.generate_mask_set(D.GeneratorSpec(2, 4, 4, 64, "random", 0.5, 0.5, 1.0, 1))
    q, k, v = make_qkv(256, 2, 96, 1)
    with pytest.raises(D.ConfigError):
        sparse_attention(q.cuda(), k.cuda(), v.cuda(), m)
    q, k, v = make_qkv(256, 2, 64, 1)
    with pytest.raises(D.ContractError):
        sparse_attention(q, k, v, m)  # CPU tensors: no fallback


@pytest.mark.parametrize("name", ["wan", "cogvideox", "hunyuan"])
def test_full_size_sampled_rows(name):
    # BASELINE configs B/C/D at full size: rows are independent, so sampled
    # (head, Q-block) rows are checked exactly against the oracle, plus the
    # LSE of those rows and a finite-output sweep over the whole layer.
    from paper_2511_23113_b200.workloads import WORKLOADS
    wl = WORKLOADS[name]
    masks = D.generate_mask_set(wl.spec())
    H, S, d = wl.heads, wl.tokens, wl.head_dim
    nb = masks.num_q_blocks
    g = torch.Generator(device="cuda").manual_seed(99)
    q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(3))
    out, lse = sparse_attention(q, k, v, masks, return_lse=True)
    torch.cuda.synchronize()
    assert bool(torch.isfinite(out).all())
    rng = np.random.default_rng(5)
    rows = np.array([(h, b) for h in range(H) for b in rng.choice(nb, 8, replace=False)], np.int32)
    ref, ref_lse = oracle.sparse_attention(q.float().cpu().numpy(), k.float().cpu().numpy(),
                                           v.float().cpu().numpy(), masks.words, nb, rows=rows)
    got, gl = out.float().cpu().numpy(), lse.cpu().numpy()
    idx_tok = np.concatenate([np.arange(b * 64, b * 64 + 64) for _, b in rows])
    idx_head = np.repeat(rows[:, 0], 64)
    a, r = got[idx_tok, idx_head], ref[idx_tok, idx_head]
    mx = float(np.abs(a - r).max())
    rel = float(np.linalg.norm(a - r) / np.linalg.norm(r))
    assert mx <= MAX_ABS and rel <= REL_L2, f"{name}: max_abs={mx:.3e} rel_l2={rel:.3e}"
    la, lr = gl[idx_head, idx_tok], ref_lse[idx_head, idx_tok]
    fin = np.isfinite(lr)
    assert np.array_equal(fin, np.isfinite(la))
    assert np.abs(la[fin] - lr[fin]).max() < 1e-2


def torch_fp32_masked_attention(q, k, v, masks, chunk=1024):
    """Plain torch fp32 block-masked attention on the GPU (TF32 off), in
    1024-row chunks: tile (q, k) is computed iff its mask bit is set
    (mask.hpp:18-20); a row with no keys gives 0.  [S, H, d] float32."""
    S, H, d = q.shape
    nq, nk = masks.num_q_blocks, masks.num_kv_blocks
    words = torch.from_numpy(np.ascontiguousarray(masks.words).view(np.int64)).cuda()  # [H, nq, wpr]
    shifts = torch.arange(64, device="cuda", dtype=torch.int64)
    ref = torch.empty(S, H, d, device="cuda", dtype=torch.float32)
    tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        scale = 1.0 / math.sqrt(d)
        for h in range(H):
            bits = ((words[h].unsqueeze(-1) >> shifts) & 1).bool().reshape(nq, -1)[:, :nk]  # [nq, nk]
            kh, vh = k[:, h].float(), v[:, h].float()
            for q0 in range(0, S, chunk):
                q1 = min(S, q0 + chunk)
                s = (q[q0:q1, h].float() @ kh.T) * scale
                m = bits[q0 // 64:(q1 + 63) // 64].repeat_interleave(64, 0)[: q1 - q0]
                s.masked_fill_(~m.repeat_interleave(64, 1)[:, :S], float("-inf"))
                ref[q0:q1, h] = torch.softmax(s, dim=-1).nan_to_num_(0.0) @ vh
    finally:
        torch.backends.cuda.matmul.allow_tf32 = tf32
    return ref


def every_row_error(out, ref):
    diff = out.float() - ref
    return float(diff.abs().max()), float(diff.norm() / ref.norm())


@pytest.mark.parametrize("name", ["wan", "wan-random", "wan-banded", "cogvideox", "hunyuan", "toy"])
def test_full_size_every_row_vs_torch_fp32(name):
    # BASELINE configs B/C/D at full size, EVERY output row, against a plain
    # torch fp32 masked attention computed on the GPU from the same block
    # masks.  The CPU oracle pins sampled rows of the same layers in
    # test_full_size_sampled_rows; this covers the rest.
    from paper_2511_23113_b200.workloads import WORKLOADS
    wl = WORKLOADS[name]
    masks = D.generate_mask_set(wl.spec())
    H, S, d = wl.heads, wl.tokens, wl.head_dim
    g = torch.Generator(device="cuda").manual_seed(7)
    q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(3))
    out = sparse_attention(q, k, v, masks)
    mx, rel = every_row_error(out, torch_fp32_masked_attention(q, k, v, masks))
    print(f"every-row parity {name}: max_abs={mx:.3e} rel_l2={rel:.3e} ({H} heads x {S} rows)")
    assert mx <= MAX_ABS and rel <= REL_L2, f"{name}: every row, max_abs={mx:.3e} rel_l2={rel:.3e}"


def test_full_size_sp_splits_every_row_vs_torch_fp32():
    # The Wan layer executed as every G=8 U x R split, uniform (USP default
    # plan) and db-SP (plan_dual), each rank's per-period kernels with the
    # ring accumulate/finalize merge, run on one GPU (simulate_on_one_gpu):
    # every output row against the torch fp32 reference.
    from paper_2511_23113_b200.sp import simulate_on_one_gpu
    from paper_2511_23113_b200.workloads import WORKLOADS
    wl = WORKLOADS["wan"]
    masks = D.generate_mask_set(wl.spec())
    H, S, d = wl.heads, wl.tokens, wl.head_dim
    g = torch.Generator(device="cuda").manual_seed(8)
    q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(3))
    ref = torch_fp32_masked_attention(q, k, v, masks)
    for strategy in ("U8R1", "U4R2", "U2R4", "U1R8"):
        st = D.parse_strategy(strategy)
        for bal, plan in (("uniform", D.default_plan(masks, st)), ("dbsp", D.plan_dual(masks, st).plan)):
            out, _ = simulate_on_one_gpu(q, k, v, masks, st, plan, time_kernels=False)
            mx, rel = every_row_error(out, ref)
            print(f"every-row parity wan {strategy}/{bal}: max_abs={mx:.3e} rel_l2={rel:.3e}")
            assert mx <= MAX_ABS and rel <= REL_L2, f"{strategy}/{bal}: max_abs={mx:.3e} rel_l2={rel:.3e}"


@pytest.mark.parametrize("strategy", ["U8R1", "U4R2", "U2R4", "U1R8"])
@pytest.mark.parametrize("balanced", [False, True])
def test_fused_o_return_matches_separate_exchange(strategy, balanced):
    # The reverse all-to-all fused into K4's epilogue (rows stored straight
    # into each home shard) gives bit-identical results to running the same
    # per-rank kernels and moving O separately.
    from paper_2511_23113_b200.sp import simulate_on_one_gpu
    H, S, d = 16, 4096, 128
    nb = S // 64
    masks = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, "clustered", 0.15, 0.45, 1.0, 21))
    st = D.parse_strategy(strategy)
    plan = D.plan_dual(masks, st).plan if balanced else D.default_plan(masks, st)
    q, k, v = (t.cuda() for t in make_qkv(S, H, d, 22))
    ref, _ = simulate_on_one_gpu(q, k, v, masks, st, plan, time_kernels=False)
    got, _ = simulate_on_one_gpu(q, k, v, masks, st, plan, time_kernels=False, fuse_return=True)
    assert torch.equal(got, ref)


@pytest.mark.parametrize("strategy", ["U8R1", "U4R2", "U2R4", "U1R8", "U2R2", "U1R1"])
@pytest.mark.parametrize("balanced", [False, True])
def test_native_sp_executor_matches_python_executor(strategy, balanced):
    # The C++ sequence-parallel call (csrc/sp_exec.cu), all ranks on this GPU
    # with device copies as the transport: layouts, packing, ring rotation and
    # the reverse exchange reproduce the Python executor bit for bit.
    from paper_2511_23113_b200.sp import native_sp_simulated, simulate_on_one_gpu
    H, S, d = 16, 4096, 128
    nb = S // 64
    masks = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, "clustered", 0.15, 0.45, 1.0, 31))
    st = D.parse_strategy(strategy)
    plan = D.plan_dual(masks, st).plan if balanced else D.default_plan(masks, st)
    q, k, v = (t.cuda() for t in make_qkv(S, H, d, 32))
    ref, _ = simulate_on_one_gpu(q, k, v, masks, st, plan, time_kernels=False)
    got = native_sp_simulated(q, k, v, masks, st, plan)
    torch.cuda.synchronize()
    assert torch.equal(got, ref)


@pytest.mark.parametrize("strategy,empty", [("U4R2", 1), ("U2R4", 3), ("U2R4", 0), ("U1R8", 7)])
def test_sp_executors_with_an_empty_ring_group(strategy, empty):
    # A plan whose KV group `empty` holds no block: that ring period exchanges
    # and computes nothing, and a rank whose LAST period it is finalises its
    # accumulator without a K4 launch.  C++ and Python executors agree bit for
    # bit and match the one-GPU kernel to bf16 rounding.
    from paper_2511_23113_b200.sp import native_sp_simulated, simulate_on_one_gpu
    H, S, d = 8, 4096, 128
    nb = S // 64
    masks = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, "clustered", 0.15, 0.45, 1.0, 33))
    st = D.parse_strategy(strategy)
    plan = D.default_plan(masks, st)
    kv = plan.kv_assignment.copy()
    kv[kv == empty] = (empty + 1) % st.ring
    plan = D.PartitionPlan(plan.head_assignment, plan.q_assignment, kv)
    q, k, v = (t.cuda() for t in make_qkv(S, H, d, 34))
    ref, _ = simulate_on_one_gpu(q, k, v, masks, st, plan, time_kernels=False)
    got = native_sp_simulated(q, k, v, masks, st, plan)
    one = sparse_attention(q, k, v, masks)
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
    assert float((got.float() - one.float()).abs().max()) <= 2e-2


def test_native_sp_context_nccl_single_rank():
    # The NCCL-backed C++ context on a 1-rank communicator.
    from paper_2511_23113_b200.sp import NativeSPContext
    H, S, d = 4, 2048, 64
    nb = S // 64
    masks = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, "clustered", 0.2, 0.5, 1.0, 3))
    q, k, v = (t.cuda() for t in make_qkv(S, H, d, 5))
    ctx = NativeSPContext(0, 1, lambda b: b)
    st = D.ParallelStrategy(1, 1)
    out = ctx(masks, st, D.plan_dual(masks, st).plan, q, k, v)
    ref = sparse_attention(q, k, v, masks)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


@pytest.mark.parametrize("mode", ["scaled_q", "ramped_k"])
@pytest.mark.parametrize("ring", [False, True])
def test_d64_rescale_mid_item_row_sum_on_tensor_core(mode, ring):
    # d=64 takes the row sum l from the tensor core (P x ones into TMEM,
    # attn_kernel.cuh KCfg::kColL): a lazy rescale in the middle of an item
    # must scale that l column with O, and the LSE (from l) must match; in
    # ring mode the merged accumulators go through the same l.
    H, S, d = 3, 2048, 64
    nb = S // 64
    masks = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, "clustered", 0.3, 0.7, 1.0, 31))
    q, k, v = make_qkv(S, H, d, 37)
    if mode == "scaled_q":
        q = (q.float() * 6.0).to(torch.bfloat16)
    else:
        ramp = torch.linspace(0.2, 4.0, S).view(S, 1, 1)
        q = (q.float().abs() + 0.5).to(torch.bfloat16)
        k = (k.float().abs() * ramp + 0.1).to(torch.bfloat16)
    ref, ref_lse = oracle.sparse_attention(q.float().numpy(), k.float().numpy(), v.float().numpy(),
                                           masks.words, nb)
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    out = torch.empty(S, H, d, device="cuda", dtype=torch.bfloat16)
    if not ring:
        lse = torch.empty(H, S, device="cuda", dtype=torch.float32)
        sc = AttentionSchedule().build(masks, kv_tokens_global=S)
        sc.launch(qd, kd, vd, out, lse=lse)
        torch.cuda.synchronize()
        fin = np.isfinite(ref_lse)
        assert np.abs(lse.cpu().numpy()[fin] - ref_lse[fin]).max() < 1e-2
    else:
        o_acc = torch.empty(S, H, d, dtype=torch.float32, device="cuda")
        l_acc = torch.empty(H, S, dtype=torch.float32, device="cuda")
        accum_init(o_acc, l_acc)
        groups = [np.arange(0, nb, 2), np.arange(1, nb, 2)]
        keep = []
        for i, g in enumerate(groups):
            kl = torch.cat([kd[b * 64:(b + 1) * 64] for b in g]).contiguous()
            vl = torch.cat([vd[b * 64:(b + 1) * 64] for b in g]).contiguous()
            sc = AttentionSchedule().build(masks, kv_block_ids=g, kv_tokens_global=S)
            sc.launch(qd, kl, vl, out, o_accum=o_acc, lse_accum=l_acc, accumulate=True,
                      finalize=(i == len(groups) - 1))
            keep.append((sc, kl, vl))
        torch.cuda.synchronize()
        fin = np.isfinite(ref_lse)
        assert np.abs(l_acc.cpu().numpy()[fin] - ref_lse[fin]).max() < 1e-2
    check(out, ref, f"d=64 rescale {mode} ring {ring}")


@pytest.mark.parametrize("flags", [1 | 8 | 16 | 128, 1])
@pytest.mark.parametrize("mode", ["scaled_q", "ramped_k"])
def test_d128_rescale_mid_item(flags, mode):
    # The lazy O rescale (running max grows by more than 2^8 inside an item):
    # with scaled Q or keys whose scores ramp up along the sequence, every
    # d=128 kernel must rescale O in the middle of its KV walk.
    H, S, d = 3, 2048, 128
    nb = S // 64
    masks = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, "clustered", 0.3, 0.7, 1.0, 23))
    q, k, v = make_qkv(S, H, d, 29)
    if mode == "scaled_q":
        q = (q.float() * 6.0).to(torch.bfloat16)
    else:
        ramp = torch.linspace(0.2, 4.0, S).view(S, 1, 1)
        q = (q.float().abs() + 0.5).to(torch.bfloat16)
        k = (k.float().abs() * ramp + 0.1).to(torch.bfloat16)
    ref, ref_lse = oracle.sparse_attention(q.float().numpy(), k.float().numpy(), v.float().numpy(),
                                           masks.words, nb)
    sc = AttentionSchedule().build(masks, kv_tokens_global=S, flags=flags)
    out = torch.empty(S, H, d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(H, S, device="cuda", dtype=torch.float32)
    sc.launch(q.cuda(), k.cuda(), v.cuda(), out, lse=lse)
    torch.cuda.synchronize()
    check(out, ref, f"rescale {mode} flags {flags}")
    fin = np.isfinite(ref_lse)
    assert np.abs(lse.cpu().numpy()[fin] - ref_lse[fin]).max() < 1e-2


def test_cta_pair_many_items_with_empty_quads():
    # Far more quad items than clusters (40 heads x 8K tokens = 1280 items for
    # 74 clusters), every fourth quad of a head empty (count 0 items).
    H, S, d = 40, 8192, 128
    nb = S // 64
    rng = np.random.default_rng(5)
    dense = rng.random((H, nb, nb)) < 0.3
    for b in range(0, nb, 16):
        dense[:, b:b + 4, :] = False
    masks = D.AttentionMaskSet.from_dense(dense)
    q, k, v = (t.cuda() for t in make_qkv(S, H, d, 31))
    sc = AttentionSchedule().build(masks, kv_tokens_global=S, flags=1 | 8 | 16 | 128)
    out = torch.full((S, H, d), 3.0, device="cuda", dtype=torch.bfloat16)
    sc.launch(q, k, v, out)
    torch.cuda.synchronize()
    rows = [(h, b) for h in range(0, H, 3) for b in range(0, nb, 7)]
    check_rows(out, q, k, v, masks, rows, "cta-pair many items")
    for b in range(0, nb, 16):
        assert torch.all(out[b * 64:(b + 4) * 64] == 0)


@pytest.mark.parametrize("flags,d", [(1, 64), (1, 128), (1 | 8 | 16 | 128, 128), (1 | 256, 128)])
def test_empty_heads_rows_and_quads_every_kernel(flags, d):
    # An all-empty head, empty Q rows, a whole empty quad (count 0 work items)
    # and a fully dense head, through every kernel family; rows without a
    # dense tile give O = 0 and LSE = -inf.
    H, S = 4, 1536
    nq = nk = S // 64
    rng = np.random.default_rng(3)
    dense = rng.random((H, nq, nk)) < 0.4
    dense[0] = False                 # empty head
    dense[1, 4:8, :] = False         # an empty quad of Q blocks in head 1
    dense[1, 10, :] = False          # one empty Q row
    dense[2] = True                  # fully dense head
    masks = D.AttentionMaskSet.from_dense(dense)
    q, k, v = make_qkv(S, H, d, 10)
    ref, ref_lse = oracle.sparse_attention(q.float().numpy(), k.float().numpy(), v.float().numpy(),
                                           masks.words, nk)
    sc = AttentionSchedule().build(masks, kv_tokens_global=S, flags=flags)
    out = torch.full((S, H, d), 7.0, device="cuda", dtype=torch.bfloat16)  # garbage must be overwritten
    lse = torch.empty(H, S, device="cuda", dtype=torch.float32)
    sc.launch(q.cuda(), k.cuda(), v.cuda(), out, lse=lse)
    torch.cuda.synchronize()
    check(out, ref, f"empty/dense flags {flags}")
    assert torch.all(out[:, 0] == 0) and torch.all(torch.isneginf(lse[0]))
    assert torch.all(out[4 * 64:8 * 64, 1] == 0) and torch.all(out[10 * 64:11 * 64, 1] == 0)
    fin = np.isfinite(ref_lse)
    assert np.array_equal(fin, np.isfinite(lse.cpu().numpy()))
    assert np.abs(lse.cpu().numpy()[fin] - ref_lse[fin]).max() < 1e-2


@pytest.mark.parametrize("flags", [1, 1 | 8 | 16 | 128])
def test_fused_scatter_every_d128_kernel(flags):
    # The fused O return through the one-CTA and the CTA-pair kernels: rows of
    # local Q block b go to "rank" b % 2 at home block b // 2, local head h to
    # home head H-1-h -- the same rows as the plain launch, permuted.
    from paper_2511_23113_b200.attention import OutScatter
    H, S, d = 6, 2048, 128
    nb = S // 64
    masks = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, "clustered", 0.2, 0.5, 1.0, 41))
    q, k, v = (t.cuda() for t in make_qkv(S, H, d, 42))
    sc = AttentionSchedule().build(masks, kv_tokens_global=S, flags=flags)
    ref = torch.empty_like(q)
    sc.launch(q, k, v, ref)
    homes = [torch.zeros(S // 2, H, d, device="cuda", dtype=torch.bfloat16) for _ in range(2)]
    qmap = np.array([[b % 2, (b // 2) * 64, 64] for b in range(nb)])
    scat = OutScatter([t.data_ptr() for t in homes], qmap, list(range(H - 1, -1, -1)), H, "cuda")
    sc.launch(q, k, v, None, scatter=scat)
    torch.cuda.synchronize()
    for b in range(nb):
        got = homes[b % 2][(b // 2) * 64:(b // 2 + 1) * 64].flip(1)
        assert torch.equal(got, ref[b * 64:(b + 1) * 64]), f"flags {flags} block {b}"


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("pattern", ["clustered", "random"])
def test_matches_flashinfer_block_sparse(d, pattern):
    # An independent implementation of the same block-sparse semantics:
    # FlashInfer's VariableBlockSparseAttentionWrapper with the per-head 64x64
    # block maps (library code, used here only as a second checker).  Rows that
    # see at least one key are compared (FlashInfer leaves empty rows undefined).
    fi = pytest.importorskip("flashinfer")
    H, S = 8, 4096
    nb = S // 64
    masks = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, pattern, 0.15, 0.45, 1.0, 5))
    g = torch.Generator(device="cuda").manual_seed(3)
    q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(3))
    out = sparse_attention(q, k, v, masks)
    words = torch.from_numpy(np.ascontiguousarray(masks.words).view(np.int64)).cuda()
    bits = ((words.unsqueeze(-1) >> torch.arange(64, device="cuda")) & 1).bool().reshape(H, nb, -1)[:, :, :nb]
    w = fi.VariableBlockSparseAttentionWrapper(torch.empty(128 << 20, dtype=torch.uint8, device="cuda"))
    w.plan(bits.contiguous(), torch.full((H, nb), 64, dtype=torch.int32, device="cuda"),
           torch.full((H, nb), 64, dtype=torch.int32, device="cuda"), H, H, d,
           q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
    ref = w.run(*(t.transpose(0, 1).contiguous() for t in (q, k, v)))
    if ref.shape[0] == H:
        ref = ref.transpose(0, 1)
    sel = bits.any(dim=-1).transpose(0, 1).repeat_interleave(64, 0)[:S]  # [S, H]
    diff = out.float()[sel] - ref.float()[sel]
    mx, rel = float(diff.abs().max()), float(diff.norm() / ref.float()[sel].norm())
    assert mx <= MAX_ABS and rel <= REL_L2, f"d={d} {pattern}: max_abs={mx:.3e} rel_l2={rel:.3e}"
