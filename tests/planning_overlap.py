"""Per-layer U x R selection kept off the critical path (GPU-box tool).

A stand-in denoising loop on one B200: for every (step, layer) the GPU
selector (dbsp_select_device, G=8) plans the layer from its live masks, and
the layer's attention (K4 over the Wan layer) runs.  Sequential: plan, then
launch.  Overlapped: a host thread plans layer l+1 on its own CUDA stream while
layer l's attention runs.  Prints wall time per layer for both."""
import json
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_23113_b200 as D  # noqa: E402
from paper_2511_23113_b200.attention import AttentionSchedule  # noqa: E402


def main():
    steps, layers = 3, 20
    H, S, d = 40, 32768, 128
    nb = S // 64
    prof = D.MachineProfile.from_json(json.loads(
        (ROOT / "paper_2511_23113_b200" / "profiles" / "b200_wan_measured.json").read_text()))
    base = D.GeneratorSpec(H, nb, nb, 64, "clustered", 0.15, 0.45, 1.0, 1)
    masks = [D.generate_mask_set(D.GeneratorSpec(**{**base.__dict__, "seed": D.mix_seed(1, l)}))
             for l in range(layers)]
    words = [torch.from_numpy(np.ascontiguousarray(m.words).view(np.int64)).cuda() for m in masks]
    scheds = [AttentionSchedule().build(m, kv_tokens_global=S) for m in masks]
    for sc in scheds:
        sc.upload()
    q, k, v = (torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    out = torch.empty_like(q)
    plan_stream = torch.cuda.Stream(priority=-1)  # high priority: its small kernels take the next free SM slots
    state = D.SelectorState(8)

    def plan(layer):
        with torch.cuda.stream(plan_stream):
            return D.select_device(layer, words[layer], nb, prof, D.PlannerConfig(), state, stream=plan_stream)

    def run(overlap: bool) -> float:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        nxt = plan(0)
        for step in range(steps):
            for layer in range(layers):
                sel = nxt
                holder = {}
                th = None
                last = step == steps - 1 and layer == layers - 1
                if not last:
                    ln = (layer + 1) % layers
                    if overlap:
                        th = threading.Thread(target=lambda: holder.setdefault("s", plan(ln)))
                        th.start()
                scheds[layer].launch(q, k, v, out)  # the layer's attention under `sel`
                if not last:
                    if overlap:
                        th.join()
                        nxt = holder["s"]
                    else:
                        torch.cuda.current_stream().synchronize()
                        nxt = plan(ln)
                torch.cuda.current_stream().synchronize()
        return (time.perf_counter() - t0) / (steps * layers) * 1e3

    run(False)
    seq = run(False)
    ovl = run(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        scheds[0].launch(q, k, v, out)
    e1.record()
    torch.cuda.synchronize()
    attn = e0.elapsed_time(e1) / 10
    print(json.dumps({"layers_per_run": steps * layers, "attention_ms": round(attn, 3),
                      "wall_ms_per_layer_sequential": round(seq, 3),
                      "wall_ms_per_layer_overlapped": round(ovl, 3),
                      "planning_exposed_ms_sequential": round(seq - attn, 3),
                      "planning_exposed_ms_overlapped": round(ovl - attn, 3)}))


if __name__ == "__main__":
    main()
