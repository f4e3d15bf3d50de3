"""Measure the dense-attention term of a B200 MachineProfile (latency.hpp:45-67)
for a workload shape: K4 latency at mask densities 0.1 .. 1.0 on one GPU,
least-squares fitted by fit_profile (latency.hpp:114-169) into
`dense_attn_seconds` (slope) and `launch_seconds` (intercept).  The
communication curves need >= 2 GPUs; until measured they are the nominal
NVLink 5 figures (B200_PROFILING.md: 725 GB/s all-reduce bus bw, 770 GB/s
peer copy).  GPU-box tool:  python tests/measure_profile.py [workload]
writes paper_2511_23113_b200/profiles/b200_<workload>_measured.json."""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2511_23113_b200 as D  # noqa: E402
from paper_2511_23113_b200.attention import AttentionSchedule  # noqa: E402
from paper_2511_23113_b200.workloads import WORKLOADS  # noqa: E402


def main():
    wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "wan"]
    H, S, d, nb = wl.heads, wl.tokens, wl.head_dim, wl.blocks
    q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    out = torch.empty_like(q)
    samples = []
    for dens in (0.1, 0.2, 0.3, 0.45, 0.6, 0.8, 1.0):
        m = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, wl.pattern, dens, dens, 1.0, 3))
        sc = AttentionSchedule().build(m, kv_tokens_global=S, head_dim=d)
        sc.upload()
        for _ in range(3):
            sc.launch(q, k, v, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            sc.launch(q, k, v, out)
        e1.record()
        torch.cuda.synchronize()
        sec = e0.elapsed_time(e1) / 10 / 1e3
        samples.append(D.ProfileSample("dense", 1, D.density(m), sec))
        print(f"density {D.density(m):.3f}: {sec * 1e3:.3f} ms", flush=True)
    nominal = json.loads((ROOT / "paper_2511_23113_b200" / "profiles" / "b200_nominal.json").read_text())
    for e in nominal["all2all"]:
        samples.append(D.ProfileSample("all2all", e["degree"], e["payload_bytes"], e["seconds"]))
    for e in nominal["p2p"]:
        samples.append(D.ProfileSample("p2p", e["degree"], e["payload_bytes"], e["seconds"]))
    prof = D.fit_profile(samples, D.FitOptions(nominal["exchange_overlap"], nominal["replan_seconds"],
                                               nominal["bytes_per_token_per_head"]))
    j = prof.to_json()
    j["dense"] = [{"density": s.x, "seconds": s.seconds} for s in samples if s.primitive == "dense"]
    j["_comment"] = (f"B200 profile for the {wl.name} shape: dense samples measured with K4 on one B200 "
                     "(fit: dense_attn_seconds=%.6g, launch_seconds=%.6g); all2all/p2p nominal NVLink 5 "
                     "until measured on >= 2 GPUs." % (prof.dense_attn_seconds, prof.launch_seconds))
    dst = ROOT / "paper_2511_23113_b200" / "profiles" / f"b200_{sys.argv[1] if len(sys.argv) > 1 else 'wan'}_measured.json"
    dst.write_text(json.dumps(j, indent=1) + "\n")
    Path(ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / dst.name).write_text(json.dumps(j, indent=1) + "\n")
    print("wrote", dst, "dense_attn_seconds", prof.dense_attn_seconds, "launch", prof.launch_seconds)


if __name__ == "__main__":
    main()
