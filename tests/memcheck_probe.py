"""compute-sanitizer target for the K4 kernels: one small launch per
schedule-flag set given on the command line (GPU-box tool):
    compute-sanitizer --tool memcheck python tests/memcheck_probe.py 153 1"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2511_23113_b200 as D  # noqa: E402
from paper_2511_23113_b200.attention import AttentionSchedule  # noqa: E402

for fl in [int(x) for x in sys.argv[1:]] or [153]:
    for d in (64, 128):
        if fl & 128 and d != 128:
            continue
        H, S = 3, 1000
        nb = -(-S // 64)
        m = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, "clustered", 0.2, 0.7, 1.0, 2))
        q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
        out = torch.empty_like(q)
        AttentionSchedule().build(m, kv_tokens_global=S, flags=fl).launch(q, k, v, out)
torch.cuda.synchronize()
print("memcheck probe done")
