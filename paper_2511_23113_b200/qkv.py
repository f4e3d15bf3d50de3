"""K6: the DiT QKV projection on sm_100a with the sequence-parallel
all-to-all(v) fused into its epilogue (csrc/qkv_proj.cu; SURVEY.md §8(f)
item 4).  Without a scatter it is a plain bf16 GEMM Y = X W^T (+ b)."""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _lib as L
from .planner import ContractError, check
from .sp import RankLayout, home_range


def _cuda_bf16(t: torch.Tensor, name: str) -> None:
    if not t.is_cuda or t.dtype != torch.bfloat16 or not t.is_contiguous():
        raise ContractError(f"{name} must be a contiguous bf16 CUDA tensor (no CPU fallback exists)")


class QkvScatter:
    """Device tables of one home rank's fused QKV scatter: per home block
    {Q ring rank, Q local block, KV group, KV local block}, per head {u, local
    head}, per rank its local head count, and the destination pointers."""

    def __init__(self, layouts: List[RankLayout], rank: int, nb: int, q_ptrs: Sequence[int],
                 k_ptrs: Sequence[int], v_ptrs: Sequence[int], device):
        G = len(layouts)
        y = layouts[0].y
        lo, hi = home_range(rank, G, nb)
        qa = np.zeros(nb, np.int64)
        qpos = np.zeros(nb, np.int64)
        for lay in layouts[:y]:  # u = 0 row of ranks: q sets are shared across u
            for i, b in enumerate(lay.q_blocks):
                qa[b], qpos[b] = lay.r, i
        ka = np.zeros(nb, np.int64)
        kpos = np.zeros(nb, np.int64)
        for g, blocks in enumerate(layouts[0].kv_groups):
            for i, b in enumerate(blocks):
                ka[b], kpos[b] = g, i
        bm = np.stack([qa[lo:hi], qpos[lo:hi], ka[lo:hi], kpos[lo:hi]], axis=1).astype(np.int32)
        H = sum(len(l.heads) for l in layouts[::y])
        hm = np.zeros((H, 2), np.int32)
        for lay in layouts[::y]:
            for i, h in enumerate(lay.heads):
                hm[h] = (lay.u, i)
        t = lambda a, dt=torch.int32: torch.as_tensor(np.ascontiguousarray(a).reshape(-1), dtype=dt, device=device)
        self.block_map = t(bm)
        self.head_map = t(hm)
        self.heads_of = t(np.array([len(l.heads) for l in layouts], np.int32))
        self.q = t(np.array(q_ptrs, np.int64), torch.int64)
        self.k = t(np.array(k_ptrs, np.int64), torch.int64)
        self.v = t(np.array(v_ptrs, np.int64), torch.int64)
        self.ring = y

    def c(self):
        return L.QkvScatterT(self.q.data_ptr(), self.k.data_ptr(), self.v.data_ptr(), self.block_map.data_ptr(),
                             self.head_map.data_ptr(), self.heads_of.data_ptr(), self.ring)


def qkv_project(x: torch.Tensor, w: torch.Tensor, heads: int, head_dim: int, bias: Optional[torch.Tensor] = None,
                out: Optional[torch.Tensor] = None, scatter: Optional[QkvScatter] = None, stream=None):
    """Y = x w^T (+ bias): x [T, C], w [3*heads*head_dim, C] bf16.  Returns Y
    [T, 3*heads*head_dim], or None when `scatter` sends the rows to their ranks."""
    _cuda_bf16(x, "x")
    _cuda_bf16(w, "w")
    T, Cdim = x.shape
    N = 3 * heads * head_dim
    if w.shape != (N, Cdim):
        raise ContractError("w must be [3*heads*head_dim, hidden]")
    if bias is not None:
        _cuda_bf16(bias, "bias")
    if scatter is None and out is None:
        out = torch.empty(T, N, device=x.device, dtype=torch.bfloat16)
    a = L.QkvArgsT(x.data_ptr(), w.data_ptr(), bias.data_ptr() if bias is not None else None,
                   out.data_ptr() if out is not None else None, T, Cdim, heads, head_dim)
    s = stream if stream is not None else torch.cuda.current_stream(x.device)
    sc = scatter.c() if scatter is not None else None
    check(L.lib().dbsp_qkv_project(C.byref(a), C.byref(sc) if sc is not None else None, C.c_void_p(s.cuda_stream)))
    return out
