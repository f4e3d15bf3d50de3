"""Small end-to-end run of every device path (K4 both head dims, ring
accumulate/finalize, K2 device schedule, K1 mask stats) for
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
    print("sanitize case done")


if __name__ == "__main__":
    main()
