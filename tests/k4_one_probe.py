"""One workload, a few K4 launches with given schedule flags -- a target for
ncu captures (GPU-box tool): python tests/k4_one_probe.py [flags] [workload]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2511_23113_b200 as D  # noqa: E402
from paper_2511_23113_b200.attention import AttentionSchedule  # noqa: E402
from paper_2511_23113_b200.workloads import WORKLOADS  # noqa: E402

flags = int(sys.argv[1]) if len(sys.argv) > 1 else 1
wl = WORKLOADS[sys.argv[2] if len(sys.argv) > 2 else "wan"]
masks = D.generate_mask_set(wl.spec())
S, H, d = wl.tokens, wl.heads, wl.head_dim
g = torch.Generator(device="cuda").manual_seed(1234)
q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(3))
sc = AttentionSchedule().build(masks, kv_tokens_global=S, flags=flags)
sc.upload()
o = torch.empty_like(q)
import os  # noqa: E402
for _ in range(int(os.environ.get("DBSP_PROBE_N", "3"))):
    sc.launch(q, k, v, o)
torch.cuda.synchronize()
