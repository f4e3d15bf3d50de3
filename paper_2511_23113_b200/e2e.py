"""Host-resident layer -> GPU -> host, with the transfers hidden behind K4.

A layer whose Q/K/V live in pinned host memory ([S, H, d] bf16, token-major)
is streamed through the GPU in head chunks on three CUDA streams:

    copy-in  : strided H2D of chunk c's head slice (cudaMemcpy2DAsync)
    compute  : K2 work-list build for chunk c's heads + K4 on chunk c
    copy-out : strided D2H of chunk c's output slice

so PCIe traffic of chunk c+1 overlaps the kernel on chunk c and the
read-back of chunk c-1 (double-buffered device chunks).  Heads are
independent in attention, so the chunked result equals the one-shot one
bit for bit (tested).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

import numpy as np
import torch

from . import _lib as L
from .attention import AttentionSchedule
from .planner import AttentionMaskSet, ContractError, check


def _copy2d(dst: int, dst_pitch: int, src: int, src_pitch: int, width: int, rows: int, to_device: bool,
            stream: torch.cuda.Stream) -> None:
    check(L.lib().dbsp_copy_2d(C.c_void_p(dst), dst_pitch, C.c_void_p(src), src_pitch, width, rows,
                               int(to_device), C.c_void_p(stream.cuda_stream)))


class HostStreamingAttention:
    def __init__(self, tokens: int, heads: int, head_dim: int, chunks: int = 4, device=None):
        self.S, self.H, self.d = tokens, heads, head_dim
        self.device = torch.device(device or "cuda")
        self.chunks = max(1, min(chunks, heads))
        bounds = np.linspace(0, heads, self.chunks + 1).round().astype(int)
        self.ranges = [(int(a), int(b)) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
        hc = max(b - a for a, b in self.ranges)
        mk = lambda: torch.empty(tokens, hc, head_dim, device=self.device, dtype=torch.bfloat16)
        self.bufs = [{"q": mk(), "k": mk(), "v": mk(), "o": mk()} for _ in range(2)]
        self.scheds = [AttentionSchedule() for _ in self.ranges]
        self.s_in = torch.cuda.Stream(self.device)
        self.s_comp = torch.cuda.Stream(self.device)
        self.s_out = torch.cuda.Stream(self.device)

    def __call__(self, q_h: torch.Tensor, k_h: torch.Tensor, v_h: torch.Tensor, masks: AttentionMaskSet,
                 o_h: Optional[torch.Tensor] = None) -> torch.Tensor:
        S, H, d = self.S, self.H, self.d
        for t, n in ((q_h, "q"), (k_h, "k"), (v_h, "v")):
            if t.is_cuda or not t.is_pinned() or t.dtype != torch.bfloat16 or tuple(t.shape) != (S, H, d):
                raise ContractError(f"{n} must be pinned host bf16 [{S}, {H}, {d}]")
        if o_h is None:
            o_h = torch.empty_like(q_h).pin_memory()
        cur = torch.cuda.current_stream(self.device)
        for s in (self.s_in, self.s_comp, self.s_out):
            s.wait_stream(cur)
        with torch.cuda.stream(self.s_comp):
            words = torch.from_numpy(masks.words.view(np.int64)).to(self.device, non_blocking=True)
        row_b = H * d * 2
        free: List[Optional[torch.cuda.Event]] = [None, None]
        done_out = []
        for c, (h0, h1) in enumerate(self.ranges):
            b = self.bufs[c % 2]
            hc = h1 - h0
            width = hc * d * 2
            if free[c % 2] is not None:  # chunk c-2's output must have left the buffer
                self.s_in.wait_event(free[c % 2])
            for key, src in (("q", q_h), ("k", k_h), ("v", v_h)):
                _copy2d(b[key].data_ptr(), width, src.data_ptr() + h0 * d * 2, row_b, width, S, True, self.s_in)
            ev_in = torch.cuda.Event()
            ev_in.record(self.s_in)
            self.s_comp.wait_event(ev_in)
            # chunks are packed [S, hc, d] at the front of the (widest-chunk) buffers
            qv, kv, vv, ov = (b[x].view(-1)[: S * hc * d].view(S, hc, d) for x in ("q", "k", "v", "o"))
            sc = self.scheds[c]
            with torch.cuda.stream(self.s_comp):
                sc.build_device(words, masks.num_kv_blocks, head_ids=np.arange(h0, h1), kv_tokens_global=S,
                                head_dim=d, stream=self.s_comp)
                sc.launch(qv, kv, vv, ov, stream=self.s_comp)
            ev_c = torch.cuda.Event()
            ev_c.record(self.s_comp)
            self.s_out.wait_event(ev_c)
            _copy2d(o_h.data_ptr() + h0 * d * 2, row_b, ov.data_ptr(), width, width, S, False, self.s_out)
            ev_o = torch.cuda.Event()
            ev_o.record(self.s_out)
            free[c % 2] = ev_o
            done_out.append((ev_o, ov))
        for s in (self.s_in, self.s_comp, self.s_out):
            cur.wait_stream(s)
        self._keep = (words, done_out)
        return o_h
