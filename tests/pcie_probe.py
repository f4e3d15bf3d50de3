"""PCIe copy rates on the GPU box for the e2e path's copy shapes: 1D pinned
H2D / D2H, and the head-chunk 2D copies of HostStreamingAttention (row width
= heads_in_chunk x d x 2 B, pitch = H x d x 2 B), plus simultaneous H2D + D2H.
GPU-box tool: python tests/pcie_probe.py"""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2511_23113_b200 import _lib as L  # noqa: E402


def timed(fn, n=5):
    fn()
    torch.cuda.synchronize()
    best = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best.append(e0.elapsed_time(e1))
    best.sort()
    return best[len(best) // 2]


def main():
    S, H, d = 32768, 40, 128  # Wan layer
    nbytes = S * H * d * 2
    host = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    host2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    dev2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    res = {"bytes": nbytes}
    res["h2d_1d_GBps"] = nbytes / timed(lambda: dev.copy_(host, non_blocking=True)) / 1e6
    res["d2h_1d_GBps"] = nbytes / timed(lambda: host.copy_(dev, non_blocking=True)) / 1e6
    for hc in (1, 5, 10, 20):
        width = hc * d * 2
        chunks = H // hc

        def run():
            for c in range(chunks):
                L.lib().dbsp_copy_2d(C.c_void_p(dev.data_ptr() + c * S * width), width,
                                     C.c_void_p(host.data_ptr() + c * width), H * d * 2, width, S, 1,
                                     C.c_void_p(st.cuda_stream))
        res[f"h2d_2d_{hc}heads_GBps"] = nbytes / timed(run) / 1e6
    s2 = torch.cuda.Stream()

    def both():
        dev.copy_(host, non_blocking=True)
        with torch.cuda.stream(s2):
            host2.copy_(dev2, non_blocking=True)
        st.wait_stream(s2)
    res["h2d_plus_d2h_concurrent_GBps_each"] = nbytes / timed(both) / 1e6
    print(json.dumps({k: round(v, 2) if isinstance(v, float) else v for k, v in res.items()}))


if __name__ == "__main__":
    main()
