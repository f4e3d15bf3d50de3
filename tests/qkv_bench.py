"""K6 timing on one B200 (GPU-box tool): the tcgen05 QKV projection against
cuBLAS (torch.nn.functional.linear) at Wan2.1-14B shapes, and the fused
scatter against projection + a separate gather into the ranks' buffers (all
ranks' buffers on this GPU, so the NVLink leg is not in the number)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_23113_b200 as D  # noqa: E402
from paper_2511_23113_b200.qkv import QkvScatter, qkv_project  # noqa: E402
from paper_2511_23113_b200.sp import home_range, rank_layouts  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    H, d, C = 40, 128, 5120
    N = 3 * H * d
    res = {}
    g = torch.Generator(device="cuda").manual_seed(0)
    w = (torch.randn(N, C, device="cuda", generator=g) / C ** 0.5).to(torch.bfloat16)
    b = (torch.randn(N, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    for T in (4096, 32768):
        x = torch.randn(T, C, device="cuda", generator=g).to(torch.bfloat16)
        out = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
        flop = 2.0 * T * N * C
        ours = timed(lambda: qkv_project(x, w, H, d, bias=b, out=out))
        cub = timed(lambda: torch.nn.functional.linear(x, w, b))
        res[f"T{T}"] = {"k6_ms": round(ours, 4), "k6_tflops": round(flop / ours / 1e9, 1),
                        "cublas_ms": round(cub, 4), "cublas_tflops": round(flop / cub / 1e9, 1)}
    # fused scatter for home rank 0 of an 8-GPU U8R1 db-SP plan on the Wan masks
    S, G = 32768, 8
    nb = S // 64
    masks = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, "clustered", 0.15, 0.45, 1.0, 1))
    for sname in ("U8R1", "U4R2"):
        st = D.parse_strategy(sname)
        plan = D.plan_dual(masks, st).plan
        lays = rank_layouts(st, plan, nb, nb)
        qb = [torch.empty(len(l.q_blocks) * 64, len(l.heads), d, device="cuda", dtype=torch.bfloat16) for l in lays]
        kb = [torch.empty(len(l.kv_groups[l.r]) * 64, len(l.heads), d, device="cuda", dtype=torch.bfloat16)
              for l in lays]
        vb = [torch.empty_like(t) for t in kb]
        lo, hi = home_range(0, G, nb)
        xh = torch.randn((hi - lo) * 64, C, device="cuda", generator=g).to(torch.bfloat16)
        sc = QkvScatter(lays, 0, nb, [t.data_ptr() for t in qb], [t.data_ptr() for t in kb],
                        [t.data_ptr() for t in vb], "cuda")
        fused = timed(lambda: qkv_project(xh, w, H, d, bias=b, scatter=sc))
        yh = torch.empty(xh.shape[0], N, device="cuda", dtype=torch.bfloat16)
        # projection home, then the exchange's gather of every destination piece
        pieces = []
        for l in lays:
            hs = torch.as_tensor(l.heads, device="cuda")
            qr = [bb - lo for bb in l.q_blocks if lo <= bb < hi]
            kr = [bb - lo for bb in l.kv_groups[l.r] if lo <= bb < hi]
            rr = lambda bl: torch.as_tensor(np.concatenate([np.arange(x * 64, x * 64 + 64) for x in bl])
                                            if bl else np.zeros(0, np.int64), device="cuda")
            pieces.append((rr(qr), rr(kr), hs))

        def separate():
            qkv_project(xh, w, H, d, bias=b, out=yh)
            y4 = yh.view(-1, 3, H, d)
            for q_rows, kv_rows, hs in pieces:
                y4[q_rows][:, 0][:, hs].contiguous()
                y4[kv_rows][:, 1][:, hs].contiguous()
                y4[kv_rows][:, 2][:, hs].contiguous()
        sep = timed(separate)
        res[f"scatter_{sname}_rank0"] = {"fused_ms": round(fused, 4), "project_then_gather_ms": round(sep, 4)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
