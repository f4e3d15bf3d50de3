import torch, time, json, sys
sys.path.insert(0, "/root/repo")
x = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
y = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
for _ in range(2): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); y.copy_(x, non_blocking=True); e1.record(); torch.cuda.synchronize()
h2d = (1 << 30) / e0.elapsed_time(e1) / 1e6
e0.record(); x.copy_(y, non_blocking=True); e1.record(); torch.cuda.synchronize()
d2h = (1 << 30) / e0.elapsed_time(e1) / 1e6
# both directions at once on two streams
x2 = torch.empty(1 << 29, dtype=torch.uint8).pin_memory(); y2 = torch.empty(1 << 29, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(s1): y.copy_(x, non_blocking=True)
with torch.cuda.stream(s2): x2.copy_(y2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
print(json.dumps({"h2d_GBps": round(h2d, 1), "d2h_GBps": round(d2h, 1), "duplex_1GB_h2d_plus_0.5GB_d2h_ms": round(dt * 1e3, 2)}))
from paper_2511_23113_b200.workloads import WORKLOADS
import paper_2511_23113_b200 as D
from paper_2511_23113_b200.e2e import HostStreamingAttention
wl = WORKLOADS["wan"]; m = D.generate_mask_set(wl.spec()); S, H, d = wl.tokens, wl.heads, wl.head_dim
qh, kh, vh = (torch.randn(S, H, d, dtype=torch.bfloat16).pin_memory() for _ in range(3)); oh = torch.empty_like(qh).pin_memory()
for ch in (4, 8, 10, 20, 40):
    run = HostStreamingAttention(S, H, d, chunks=ch)
    for _ in range(2): run(qh, kh, vh, m, oh)
    torch.cuda.synchronize(); e0.record()
    for _ in range(3): run(qh, kh, vh, m, oh)
    e1.record(); torch.cuda.synchronize()
    print("chunks", ch, round(e0.elapsed_time(e1) / 3, 3), "ms")
