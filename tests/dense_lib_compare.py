"""Library dense attention on the same B200, same shape as config C (Wan: 40
heads, d=128, 32768 tokens), next to K4 on an all-dense mask and on the 30%
clustered benchmark mask.  It answers "what does a tuned tcgen05 dense FMHA
reach on this box, power cap included", the context for K4's roofline
fraction.  Libraries: torch SDPA with the cuDNN backend (cuDNN's Blackwell
FMHA) and with the flash backend (FlashAttention-2, mma.sync).  FLOPs =
4 * S_q * S_k * d * H (QK^T + PV), as for K4's dense tiles.
GPU-box tool: python tests/dense_lib_compare.py [workload] > out.json (default wan; the
sparse line uses the workload's own benchmark masks)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
from torch.nn.attention import SDPBackend, sdpa_kernel  # noqa: E402

import paper_2511_23113_b200 as D  # noqa: E402
from paper_2511_23113_b200.attention import AttentionSchedule  # noqa: E402


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return {"ms_median": round(ts[len(ts) // 2], 4), "ms_min": round(ts[0], 4)}


def main():
    from paper_2511_23113_b200.workloads import WORKLOADS
    wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "wan"]
    S, H, d = wl.tokens, wl.heads, wl.head_dim
    g = torch.Generator(device="cuda").manual_seed(1234)
    q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(3))
    out = {"workload": wl.name, "shape": {"tokens": S, "heads": H, "head_dim": d}}
    dense_flop = 4.0 * S * S * d * H
    # libraries want [B, H, S, d]; the transposed views are what they read
    qt, kt, vt = (t.permute(1, 0, 2).unsqueeze(0) for t in (q, k, v))
    for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash2", SDPBackend.FLASH_ATTENTION)):
        try:
            with sdpa_kernel(be):
                r = timed(lambda: torch.nn.functional.scaled_dot_product_attention(qt, kt, vt))
            r["tflops_median"] = round(dense_flop / r["ms_median"] / 1e9, 1)
            r["tflops_best"] = round(dense_flop / r["ms_min"] / 1e9, 1)
        except Exception as e:  # backend not available for this layout / build
            r = {"error": str(e).splitlines()[0][:200]}
        out[f"sdpa_{name}_dense"] = r
    nb = -(-S // 64)
    for label, spec in (("k4_dense", D.GeneratorSpec(H, nb, nb, 64, "random", 1.0, 1.0, 1.0, 1)),
                        ("k4_benchmark_masks", wl.spec())):
        masks = D.generate_mask_set(spec)
        flop = 4.0 * 64 * 64 * d * D.total_blocks(masks)
        sc = AttentionSchedule().build(masks, kv_tokens_global=S)
        sc.upload()
        o = torch.empty_like(q)
        r = timed(lambda: sc.launch(q, k, v, o))
        r["tflops_median"] = round(flop / r["ms_median"] / 1e9, 1)
        r["tflops_best"] = round(flop / r["ms_min"] / 1e9, 1)
        r["density"] = round(D.density(masks), 4)
        out[label] = r
        del sc
    print(json.dumps(out))


if __name__ == "__main__":
    main()
