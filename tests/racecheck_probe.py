import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2511_23113_b200 as D
from paper_2511_23113_b200.attention import AttentionSchedule
H, S, d = 3, 1000, 128
nb = -(-S // 64)
m = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, "clustered", 0.2, 0.7, 1.0, 2))
q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
AttentionSchedule().build(m, kv_tokens_global=S, flags=int(sys.argv[1])).launch(q, k, v, out)
torch.cuda.synchronize()
print("done")
