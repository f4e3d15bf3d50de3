"""Diagnostic run of K4 on a GPU: prints per-case error breakdowns (by head,
row half, column chunk) instead of asserting, plus timing for a Wan-shaped
layer.  Test infrastructure; uses the oracle as the checker."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
import paper_2511_23113_b200 as D  # noqa: E402
from paper_2511_23113_b200.attention import AttentionSchedule, sparse_attention  # noqa: E402


def case(H, S, d, pattern, dmin, dmax, seed, Sk=None):
    Sk = Sk or S
    nq, nk = -(-S // 64), -(-Sk // 64)
    m = D.generate_mask_set(D.GeneratorSpec(H, nq, nk, 64, pattern, dmin, dmax, 1.0, seed))
    g = torch.Generator().manual_seed(seed)
    q = torch.randn(S, H, d, generator=g).to(torch.bfloat16)
    k = torch.randn(Sk, H, d, generator=g).to(torch.bfloat16)
    v = torch.randn(Sk, H, d, generator=g).to(torch.bfloat16)
    ref, rl = oracle.sparse_attention(q.float().numpy(), k.float().numpy(), v.float().numpy(), m.words, nk)
    t0 = time.time()
    out, lse = sparse_attention(q.cuda(), k.cuda(), v.cuda(), m, return_lse=True)
    torch.cuda.synchronize()
    o = out.float().cpu().numpy()
    diff = np.abs(o - ref)
    rel = np.linalg.norm(o - ref) / np.linalg.norm(ref)
    print(f"H{H} S{S} Sk{Sk} d{d} {pattern}: max_abs={np.nanmax(diff):.3e} rel_l2={rel:.3e} "
          f"nan={int(np.isnan(o).sum())} t={time.time()-t0:.2f}s")
    if not (np.nanmax(diff) < 2e-2):
        per_head = [float(np.nanmax(diff[:, h])) for h in range(H)]
        print("   per-head max:", " ".join(f"{x:.2e}" for x in per_head))
        rows = diff.max(axis=(1, 2))
        blk = rows[: (S // 64) * 64].reshape(-1, 64)
        print("   rows 0-31 / 32-63 max per first 4 blocks:",
              [(float(b[:32].max()), float(b[32:].max())) for b in blk[:4]])
        print("   block max (first 8):", [f"{x:.2e}" for x in blk.max(1)[:8]])
        cols = diff.max(axis=(0, 1))
        print("   col chunk max:", [f"{float(cols[c:c+32].max()):.2e}" for c in range(0, d, 32)])
        print("   sample out/ref row0 h0:", o[0, 0, :6], ref[0, 0, :6])
        print("   ratio out/ref (row0,h0):", (o[0, 0, :6] / ref[0, 0, :6]))
        ol = lse.cpu().numpy()
        fin = np.isfinite(rl)
        print("   lse max diff:", float(np.abs(ol[fin] - rl[fin]).max()))


def timing(H=40, S=32768, d=128, pattern="clustered", dmin=0.15, dmax=0.45, reps=10):
    nb = S // 64
    m = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, pattern, dmin, dmax, 1.0, 1))
    q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    sc = AttentionSchedule().build(m, kv_tokens_global=S)
    st = sc.stats()
    out = torch.empty_like(q)
    for _ in range(3):
        sc.launch(q, k, v, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        sc.launch(q, k, v, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    flops = 4 * 64 * 64 * d * D.total_blocks(m)
    mma_flops = 4 * 128 * 64 * d * st["tile_visits"]
    print(f"timing {H}x{S}x{d} {pattern}: {ms:.3f} ms/launch (incl. schedule upload), "
          f"{flops/ms/1e9:.1f} TFLOP/s algorithmic, {mma_flops/ms/1e9:.1f} TFLOP/s issued; {st}")


if __name__ == "__main__":
    print(torch.cuda.get_device_name(0))
    case(1, 128, 64, "random", 1.0, 1.0, 1)
    case(1, 256, 128, "random", 1.0, 1.0, 2)
    case(8, 4096, 64, "random", 0.5, 0.5, 1)
    case(4, 2048, 128, "clustered", 0.1, 0.6, 3)
    case(3, 1000, 64, "random", 0.3, 0.7, 5)
    if "--time" in sys.argv:
        timing()
        timing(48, 17792, 64, "clustered", 0.317, 0.317)
