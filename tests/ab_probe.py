"""Interleaved A/B timing of K4 schedule-flag variants on one workload: the
B200's power cap moves the clock by +-10% between runs, so variants are timed
round-robin (R rounds x N launches each, the order rotated every round) and
compared by median of round medians.  GPU-box tool: python tests/ab_probe.py workload flagsA flagsB ... [--rounds R]
(a flags entry 'F:ENV=V' sets nothing -- env is per process; use one process per env)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_23113_b200 as D  # noqa: E402
from paper_2511_23113_b200.attention import AttentionSchedule  # noqa: E402
from paper_2511_23113_b200.workloads import WORKLOADS  # noqa: E402


def main():
    args = sys.argv[1:]
    rounds = 5
    per_round = 8
    if "--sustained" in args:  # 30 back-to-back launches per variant and round, median of the last 20
        i = args.index("--sustained")
        args = args[:i] + args[i + 1:]
        per_round = 30
    if "--rounds" in args:
        i = args.index("--rounds")
        rounds = int(args[i + 1])
        args = args[:i] + args[i + 2:]
    wl = WORKLOADS[args[0]]
    flag_list = [int(x) for x in args[1:]] or [1, 153]
    masks = D.generate_mask_set(wl.spec())
    S, H, d = wl.tokens, wl.heads, wl.head_dim
    g = torch.Generator(device="cuda").manual_seed(1234)
    q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(3))
    flop = 4.0 * 64 * 64 * d * D.total_blocks(masks)
    scheds = []
    for f in flag_list:
        sc = AttentionSchedule().build(masks, kv_tokens_global=S, flags=f)
        sc.upload()
        scheds.append(sc)
    o = torch.empty_like(q)
    for sc in scheds:
        for _ in range(3):
            sc.launch(q, k, v, o)
    torch.cuda.synchronize()
    res = {f: [] for f in flag_list}
    for r in range(rounds):
        # rotate the order every round: a variant's position in the round biases it
        rot = r % len(flag_list)
        for f, sc in list(zip(flag_list, scheds))[rot:] + list(zip(flag_list, scheds))[:rot]:
            ts = []
            for _ in range(per_round):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                sc.launch(q, k, v, o)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[f].append(float(np.median(ts[-20:] if per_round > 20 else ts)))
    out = {"workload": wl.name}
    for f in flag_list:
        r = np.array(res[f])
        out[str(f)] = {"ms_median": round(float(np.median(r)), 4), "ms_min_round": round(float(r.min()), 4),
                       "tflops": round(flop / float(np.median(r)) / 1e9, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
