"""K4 against FlashInfer's block-sparse attention (VariableBlockSparseAttentionWrapper,
per-head 64x64 block masks) on the same layer: an independent third-party
implementation of the same block-sparse semantics (mask.hpp:18-20) for
parity, and a library timing beside K4's.  FlashInfer is library code here:
the comparison point, never the product path.  GPU-box tool (FlashInfer
JIT-compiles its kernels on first use):
    python tests/flashinfer_compare.py [workload ...] > out.json"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_23113_b200 as D  # noqa: E402
from paper_2511_23113_b200.attention import AttentionSchedule  # noqa: E402
from paper_2511_23113_b200.workloads import WORKLOADS  # noqa: E402


def timed(fn, n=10):
    ts = []
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    from flashinfer import VariableBlockSparseAttentionWrapper
    names = sys.argv[1:] or ["cogvideox", "wan"]
    res = {}
    for name in names:
        wl = WORKLOADS[name]
        masks = D.generate_mask_set(wl.spec())
        H, S, d = wl.heads, wl.tokens, wl.head_dim
        nq, nk = masks.num_q_blocks, masks.num_kv_blocks
        g = torch.Generator(device="cuda").manual_seed(11)
        q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(3))
        # K4
        sc = AttentionSchedule().build(masks, kv_tokens_global=S, head_dim=d)
        sc.upload()
        out = torch.empty_like(q)
        k4_ms = timed(lambda: sc.launch(q, k, v, out))
        # FlashInfer, head-major inputs, the same per-head block map
        words = torch.from_numpy(np.ascontiguousarray(masks.words).view(np.int64)).cuda()  # [H, nq, wpr]
        bits = ((words.unsqueeze(-1) >> torch.arange(64, device="cuda")) & 1).bool().reshape(H, nq, -1)[:, :, :nk]
        rows = torch.full((H, nq), 64, dtype=torch.int32, device="cuda")
        cols = torch.full((H, nk), 64, dtype=torch.int32, device="cuda")
        ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        w = VariableBlockSparseAttentionWrapper(ws)
        w.plan(bits.contiguous(), rows, cols, H, H, d, q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
        qh, kh, vh = (t.transpose(0, 1).contiguous() for t in (q, k, v))
        o_fi = w.run(qh, kh, vh)
        fi_ms = timed(lambda: w.run(qh, kh, vh))
        if o_fi.shape[0] == H:  # (H, S, d) -> (S, H, d)
            o_fi = o_fi.transpose(0, 1)
        # rows that see at least one key (FlashInfer's empty-row output is not defined)
        has = bits.any(dim=-1)  # [H, nq]
        tok_has = has.transpose(0, 1).repeat_interleave(64, 0)[:S]  # [S, H]
        a, b = out.float()[tok_has], o_fi.float()[tok_has]
        diff = (a - b)
        flop = 4.0 * 64 * 64 * d * D.total_blocks(masks)
        res[wl.name] = {
            "max_abs_k4_vs_flashinfer": float(diff.abs().max()),
            "rel_l2_k4_vs_flashinfer": float(diff.norm() / b.norm()),
            "rows_compared": int(tok_has.sum()),
            "k4_ms": round(k4_ms, 4), "flashinfer_ms": round(fi_ms, 4),
            "k4_tflops": round(flop / k4_ms / 1e9, 1), "flashinfer_tflops": round(flop / fi_ms / 1e9, 1),
            "speedup_k4_vs_flashinfer": round(fi_ms / k4_ms, 3),
        }
        print(json.dumps({wl.name: res[wl.name]}), flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
