"""Small end-to-end run of every device path (K4 both head dims and every
opt-in variant, ring accumulate/finalize, K2 device schedule, K1 mask stats,
the GPU selector, K6 with and without its scatter, the fused O return, the
C++ SP executor) for
compute-sanitizer (memcheck / synccheck / racecheck) on a GPU box:
    compute-sanitizer --tool memcheck python tests/sanitize_case.py"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2511_23113_b200 as D  # noqa: E402
from paper_2511_23113_b200.attention import AttentionSchedule, accum_init, sparse_attention  # noqa: E402


def main():
    for d in (64, 128):
        H, S = 2, 640 - 17
        nb = -(-S // 64)
        m = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, "clustered", 0.2, 0.7, 1.0, 1))
        q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
        sparse_attention(q, k, v, m, return_lse=True)
        sparse_attention(q, k, v, m, device_schedule=True)
        o_acc = torch.empty(S, H, d, device="cuda", dtype=torch.float32)
        l_acc = torch.empty(H, S, device="cuda", dtype=torch.float32)
        out = torch.empty_like(q)
        accum_init(o_acc, l_acc)
        groups = [np.arange(0, nb, 2), np.arange(1, nb, 2)]
        for i, g in enumerate(groups):
            rows = torch.as_tensor((g[:, None] * 64 + np.arange(64)[None, :]).reshape(-1), device="cuda")
            rows = rows.clamp(max=S - 1)
            kl, vl = k.index_select(0, rows).contiguous(), v.index_select(0, rows).contiguous()
            sc = AttentionSchedule().build(m, kv_block_ids=g, kv_tokens_global=S)
            sc.launch(q, kl, vl, out, o_accum=o_acc, lse_accum=l_acc, accumulate=True, finalize=i == 1)
        torch.cuda.synchronize()
    words = torch.from_numpy(m.words.view(np.int64)).cuda()
    D.mask_stats_device(words, m.num_kv_blocks)
    torch.cuda.synchronize()
    # both d=128 kernels: one-CTA pair items and the CTA-pair quad items
    H, S, d = 3, 1000, 128
    nb = -(-S // 64)
    m = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, "clustered", 0.2, 0.7, 1.0, 2))
    q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    out = torch.empty_like(q)
    for fl in (1, 1 | 8 | 16 | 128):
        AttentionSchedule().build(m, kv_tokens_global=S, flags=fl).launch(q, k, v, out)
    # CTA-pair split-KV kernel through the ring accumulator (two KV periods)
    o_acc = torch.empty(S, H, d, device="cuda", dtype=torch.float32)
    l_acc = torch.empty(H, S, device="cuda", dtype=torch.float32)
    accum_init(o_acc, l_acc)
    for i, g in enumerate((np.arange(0, nb // 2), np.arange(nb // 2, nb))):
        rows = torch.as_tensor((g[:, None] * 64 + np.arange(64)[None, :]).reshape(-1), device="cuda").clamp(max=S - 1)
        kl, vl = k.index_select(0, rows).contiguous(), v.index_select(0, rows).contiguous()
        AttentionSchedule().build(m, kv_block_ids=g, kv_tokens_global=S, flags=1 | 8 | 16 | 128).launch(
            q, kl, vl, out, o_accum=o_acc, lse_accum=l_acc, accumulate=True, finalize=i == 1)
    torch.cuda.synchronize()
    # GPU selector, SP paths (fused O return, C++ executor), K6
    from paper_2511_23113_b200.qkv import QkvScatter, qkv_project
    from paper_2511_23113_b200.sp import native_sp_simulated, rank_layouts, simulate_on_one_gpu
    H, S, d, C = 8, 1024, 128, 256
    nb = S // 64
    m = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, "clustered", 0.2, 0.6, 1.0, 3))
    prof = D.MachineProfile.from_json(__import__("json").loads(
        (Path(__file__).resolve().parents[1] / "paper_2511_23113_b200" / "profiles" / "b200_nominal.json").read_text()))
    w64 = torch.from_numpy(m.words.view(np.int64)).cuda()
    D.select_device(0, w64, nb, prof, D.PlannerConfig(), D.SelectorState(4))
    q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    st = D.parse_strategy("U2R2")
    plan = D.plan_dual(m, st).plan
    simulate_on_one_gpu(q, k, v, m, st, plan, time_kernels=False, fuse_return=True)
    native_sp_simulated(q, k, v, m, st, plan)
    x = torch.randn(S, C, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(3 * H * d, C, device="cuda", dtype=torch.bfloat16)
    qkv_project(x, w, H, d)
    lays = rank_layouts(st, plan, nb, nb)
    qb = [torch.empty(len(l.q_blocks) * 64, len(l.heads), d, device="cuda", dtype=torch.bfloat16) for l in lays]
    kb = [torch.empty(len(l.kv_groups[l.r]) * 64, len(l.heads), d, device="cuda", dtype=torch.bfloat16) for l in lays]
    vb = [torch.empty_like(t) for t in kb]
    sc = QkvScatter(lays, 0, nb, [t.data_ptr() for t in qb], [t.data_ptr() for t in kb], [t.data_ptr() for t in vb],
                    "cuda")
    qkv_project(x[:S // 4].contiguous(), w, H, d, scatter=sc)
    torch.cuda.synchronize()
    print("sanitize case done")


if __name__ == "__main__":
    main()
