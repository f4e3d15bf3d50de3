import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2511_23113_b200 as D
from paper_2511_23113_b200.attention import AttentionSchedule
for name, (H, S) in {"wan": (40, 32768), "hunyuan": (24, 118848), "cog": (48, 17792)}.items():
    nb = -(-S // 64)
    m = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, "clustered", .15, .45, 1.0, 1))
    w = torch.from_numpy(np.ascontiguousarray(m.words).view(np.int64)).cuda()
    sc = AttentionSchedule()
    d = 64 if name == "cog" else 128
    for _ in range(3): sc.build_device(w, nb, kv_tokens_global=S, head_dim=d)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): sc.build_device(w, nb, kv_tokens_global=S, head_dim=d)
    e1.record(); torch.cuda.synchronize()
    host = AttentionSchedule().build(m, kv_tokens_global=S, head_dim=d)
    hi, he = host.download(); di, de = sc.download()
    print(name, "K2 ms", round(e0.elapsed_time(e1) / 20, 4), "equal", np.array_equal(hi, di) and np.array_equal(he, de), sc.layout()["kernel"])
