"""Rebuild K4 with each compile-time variant and time it on the Wan layer
(plus a quick parity check).  GPU-box tool: python tests/kernel_sweep.py
"FLAGS1" "FLAGS2" ...  (flags go to nvcc, e.g. -DDBSP_POLY_EVERY=3)."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

CHILD = r"""
import os, sys, json, numpy as np, torch
sys.path.insert(0, %r)
import oracle, paper_2511_23113_b200 as D
from paper_2511_23113_b200.attention import AttentionSchedule, sparse_attention
res = {}
fl = int(os.environ.get("DBSP_SWEEP_FLAGS", "1"))
flags_for = lambda d: fl if d == 128 else fl & ~(8 | 16 | 128)  # the CTA-pair kernel is d=128 only
# parity (toy + d128 clustered) with the swept schedule flags
for (H, S, d, pat, lo, hi, seed) in [(8, 4096, 64, "random", .5, .5, 1), (4, 2048, 128, "clustered", .1, .6, 3)]:
    nb = S // 64
    m = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, pat, lo, hi, 1.0, seed))
    g = torch.Generator().manual_seed(seed)
    q, k, v = (torch.randn(S, H, d, generator=g).to(torch.bfloat16) for _ in range(3))
    ref, _ = oracle.sparse_attention(q.float().numpy(), k.float().numpy(), v.float().numpy(), m.words, nb)
    sc = AttentionSchedule().build(m, kv_tokens_global=S, flags=flags_for(d))
    o = torch.empty(S, H, d, device="cuda", dtype=torch.bfloat16)
    sc.launch(q.cuda(), k.cuda(), v.cuda(), o)
    out = o.float().cpu().numpy()
    res[f"maxabs_d{d}"] = float(np.abs(out - ref).max())
for name, (H, S, d, pat, lo, hi) in {"wan": (40, 32768, 128, "clustered", .15, .45),
                                     "cog": (48, 17792, 64, "clustered", .317, .317)}.items():
    nb = S // 64
    m = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, pat, lo, hi, 1.0, 1))
    q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    sc = AttentionSchedule().build(m, kv_tokens_global=S, flags=flags_for(d)); sc.upload()
    out = torch.empty_like(q)
    for _ in range(3): sc.launch(q, k, v, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): sc.launch(q, k, v, out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    res[name + "_ms"] = round(ms, 4)
    res[name + "_tflops"] = round(4 * 64 * 64 * d * D.total_blocks(m) / ms / 1e9, 1)
print("RESULT", json.dumps(res))
""" % str(ROOT)


def main():
    if sys.argv[1:] == ["--no-build"]:  # time the in-tree build as is
        out = subprocess.run([sys.executable, "-c", CHILD], capture_output=True, text=True, timeout=600)
        print(out.stdout.strip() or out.stderr[-800:], flush=True)
        return
    variants = sys.argv[1:] or [""]
    for flags in variants:
        env = dict(os.environ, DBSP_NVCC_FLAGS=flags)
        subprocess.run([sys.executable, str(ROOT / "paper_2511_23113_b200" / "build.py"), "-f"], env=env,
                       check=True, capture_output=True)
        out = subprocess.run([sys.executable, "-c", CHILD], capture_output=True, text=True, timeout=600)
        line = [l for l in out.stdout.splitlines() if l.startswith("RESULT")]
        print(json.dumps({"flags": flags, **(json.loads(line[0][7:]) if line else {"error": out.stderr[-800:]})}),
              flush=True)
    # leave the default build in place
    subprocess.run([sys.executable, str(ROOT / "paper_2511_23113_b200" / "build.py"), "-f"], check=True,
                   capture_output=True)


if __name__ == "__main__":
    main()
