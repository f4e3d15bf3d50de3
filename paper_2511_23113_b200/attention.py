"""Block-sparse attention call (K4 on sm_100a) over torch CUDA tensors.

torch supplies device memory and the current stream only; the schedule is
built by the C++ host code and the math runs in libdbsp_b200.so's tcgen05
kernel.  Requires a CUDA device: there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import math
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib as L
from .planner import AttentionMaskSet, ConfigError, ContractError, check


def _require_cuda(t: torch.Tensor, name: str, dtype=torch.bfloat16) -> None:
    if not t.is_cuda:
        raise ContractError(f"{name} must be a CUDA tensor (no CPU fallback exists)")
    if t.dtype != dtype:
        raise ContractError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ContractError(f"{name} must be contiguous")


def _u32arr(seq) -> Optional[np.ndarray]:
    if seq is None:
        return None
    return np.ascontiguousarray(np.asarray(seq, dtype=np.uint32))


class AttentionSchedule:
    """Work list of one kernel launch (dbsp_schedule): which (head, Q tile)
    items exist and which KV blocks each visits.  Reusable across launches
    while the masks and the local view do not change."""

    def __init__(self):
        h = C.c_void_p()
        check(L.lib().dbsp_schedule_create(C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and L is not None:  # modules may be gone at interpreter exit
            L.lib().dbsp_schedule_destroy(h)
            self._h = None

    def build(self, masks: AttentionMaskSet, *, head_ids: Sequence[int] = None,
              q_block_ids: Sequence[int] = None, kv_block_ids: Sequence[int] = None,
              kv_tokens_global: int = 0, pair_q: bool = True, flags: Optional[int] = None,
              head_dim: Optional[int] = None) -> "AttentionSchedule":
        """flags: DBSP_SCHED_* bits (1 pair, 2 global LPT, 4 head order, 128 the d=128 CTA-pair
        kernel's quad items (adds the layout bits 8|16), 256 the automatic d=128 layout choice, which
        resolves to the pair layout since round 2 (schedule.hpp)).  Default: pair_q, plus the auto
        choice when head_dim is 128 (DBSP_SCHED_AUTO_D128)."""
        hid, qid, kid = _u32arr(head_ids), _u32arr(q_block_ids), _u32arr(kv_block_ids)
        if flags is None:
            flags = (1 | 256 if head_dim == 128 else 1) if pair_q else 0
        self._keep = (hid, qid, kid)
        ptr = lambda a: a.ctypes.data_as(C.POINTER(C.c_uint32)) if a is not None else None
        view = L.LocalViewT(
            len(hid) if hid is not None else masks.num_heads, ptr(hid),
            len(qid) if qid is not None else masks.num_q_blocks, ptr(qid),
            len(kid) if kid is not None else masks.num_kv_blocks, ptr(kid),
            kv_tokens_global)
        check(L.lib().dbsp_schedule_build(self._h, C.byref(masks.c()), C.byref(view), int(flags)))
        return self

    def build_device(self, words: torch.Tensor, num_kv_blocks: int, *, head_ids=None, q_block_ids=None,
                     kv_block_ids=None, kv_tokens_global: int = 0, flags: Optional[int] = None,
                     head_dim: Optional[int] = None,
                     stream: Optional[torch.cuda.Stream] = None) -> "AttentionSchedule":
        """K2: build the work list on the GPU from device mask words (int64
        [H, Nq, ceil(Nk/64)], the BlockMask row layout).  flags as in build();
        default: pair items, and for head_dim 128 the auto choice, made on the
        device (both layouts are built, both kernels launched, the kernel not
        chosen returns at once)."""
        if flags is None:
            flags = 1 | 256 if head_dim == 128 else 1
        if not words.is_cuda or words.dtype != torch.int64 or words.dim() != 3 or not words.is_contiguous():
            raise ContractError("device mask words must be a contiguous CUDA int64 [H, Nq, words] tensor")
        H, nq, _ = words.shape
        hid, qid, kid = _u32arr(head_ids), _u32arr(q_block_ids), _u32arr(kv_block_ids)
        self._keep = (hid, qid, kid, words)
        ptr = lambda a: a.ctypes.data_as(C.POINTER(C.c_uint32)) if a is not None else None
        view = L.LocalViewT(len(hid) if hid is not None else H, ptr(hid),
                            len(qid) if qid is not None else nq, ptr(qid),
                            len(kid) if kid is not None else num_kv_blocks, ptr(kid), kv_tokens_global)
        s = stream if stream is not None else torch.cuda.current_stream(words.device)
        check(L.lib().dbsp_schedule_build_device(self._h, C.c_void_p(words.data_ptr()), H, nq, num_kv_blocks,
                                                 C.byref(view), int(flags), C.c_void_p(s.cuda_stream)))
        return self

    def download(self):
        """(items [n, 8] uint32, entries uint32) of the built list."""
        st = self.stats()
        items = np.zeros((st["items"], 8), np.uint32)
        entries = np.zeros(max(st["tile_visits"], 1), np.uint32)
        check(L.lib().dbsp_schedule_download(self._h, C.c_void_p(items.ctypes.data),
                                             entries.ctypes.data_as(C.POINTER(C.c_uint32)), entries.size))
        return items, entries[:st["tile_visits"]]

    def stats(self) -> dict:
        items, visits, dense = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(L.lib().dbsp_schedule_stats(self._h, C.byref(items), C.byref(visits), C.byref(dense)))
        return {"items": items.value, "tile_visits": visits.value, "dense_tiles": dense.value}

    def layout(self) -> dict:
        """Schedule flags actually built (an auto build reports its choice) and the 64-row Q
        blocks each work item covers (its M per tile visit)."""
        f = C.c_uint32()
        check(L.lib().dbsp_schedule_layout(self._h, C.byref(f)))
        rows = 4 if f.value & 8 else 2 if f.value & 1 else 1
        return {"flags": f.value, "q_blocks_per_item": rows,
                "kernel": "cta_pair_split_kv" if f.value & 128 else "pair_items"}

    def upload(self, stream: Optional[torch.cuda.Stream] = None) -> int:
        """Make the schedule device-resident (no-op if already); returns bytes moved."""
        s = stream if stream is not None else torch.cuda.current_stream()
        n = C.c_uint64()
        check(L.lib().dbsp_schedule_upload_bytes(self._h, C.byref(n)))
        check(L.lib().dbsp_schedule_upload(self._h, C.c_void_p(s.cuda_stream)))
        return n.value

    def launch(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out: Optional[torch.Tensor],
               *, lse: Optional[torch.Tensor] = None, o_accum: Optional[torch.Tensor] = None,
               lse_accum: Optional[torch.Tensor] = None, accumulate: bool = False,
               finalize: bool = False, softmax_scale: Optional[float] = None,
               stream: Optional[torch.cuda.Stream] = None, scatter: Optional["OutScatter"] = None) -> None:
        """scatter: fused O return -- bf16 rows go to their home ranks' buffers
        (dbsp_attention_launch_scatter) instead of `out`."""
        for t, n in ((q, "q"), (k, "k"), (v, "v")):
            _require_cuda(t, n)
        if out is not None:
            _require_cuda(out, "out")
        if lse is not None:
            _require_cuda(lse, "lse", torch.float32)
        if accumulate:
            _require_cuda(o_accum, "o_accum", torch.float32)
            _require_cuda(lse_accum, "lse_accum", torch.float32)
        Sq, H, d = q.shape
        Sk = k.shape[0]
        if k.shape != (Sk, H, d) or v.shape != (Sk, H, d):
            raise ContractError("k/v must be [kv_tokens, heads, head_dim] matching q")
        args = L.AttnArgsT(q.data_ptr(), k.data_ptr(), v.data_ptr(),
                           out.data_ptr() if out is not None else None,
                           lse.data_ptr() if lse is not None else None,
                           o_accum.data_ptr() if o_accum is not None else None,
                           lse_accum.data_ptr() if lse_accum is not None else None,
                           Sq, Sk, H, d, float(softmax_scale or 0.0), int(accumulate), int(finalize))
        s = stream if stream is not None else torch.cuda.current_stream(q.device)
        if scatter is not None:
            if len(scatter.head_map) != H:
                raise ContractError("scatter head map must cover the local heads")
            sc = scatter.c()
            check(L.lib().dbsp_attention_launch_scatter(self._h, C.byref(args), C.byref(sc),
                                                        C.c_void_p(s.cuda_stream)))
            return
        check(L.lib().dbsp_attention_launch(self._h, C.byref(args), C.c_void_p(s.cuda_stream)))


class OutScatter:
    """Device tables of the fused O return (include/dbsp_b200.h dbsp_out_scatter):
    peer output pointers per rank, per local Q block (home rank, first home
    row, valid rows) and local -> global heads."""

    def __init__(self, peer_ptrs: Sequence[int], q_block_map: np.ndarray, head_map: Sequence[int],
                 out_heads: int, device):
        qm = np.ascontiguousarray(np.asarray(q_block_map, np.int64).reshape(-1, 3))
        if (qm[:, 0] >= len(peer_ptrs)).any() or (qm < 0).any():
            raise ContractError("scatter block map addresses past the peer table")
        hm = np.asarray(head_map, np.int64)
        if len(hm) and (hm.min() < 0 or hm.max() >= out_heads):
            raise ContractError("scatter head map addresses past the home heads")
        self.peers = torch.tensor([int(p) for p in peer_ptrs], dtype=torch.int64, device=device)
        self.q_map = torch.as_tensor(qm.astype(np.int32).reshape(-1), device=device)
        self.head_map = torch.as_tensor(hm.astype(np.int32), device=device)
        self.out_heads = int(out_heads)

    def c(self):
        return L.OutScatterT(self.peers.data_ptr(), self.q_map.data_ptr(), self.head_map.data_ptr(),
                             self.out_heads)


def accum_init(o_accum: torch.Tensor, lse_accum: torch.Tensor, stream=None) -> None:
    _require_cuda(o_accum, "o_accum", torch.float32)
    _require_cuda(lse_accum, "lse_accum", torch.float32)
    Sq, H, d = o_accum.shape
    s = stream if stream is not None else torch.cuda.current_stream(o_accum.device)
    check(L.lib().dbsp_accum_init(C.c_void_p(o_accum.data_ptr()), C.c_void_p(lse_accum.data_ptr()),
                                  Sq, H, d, C.c_void_p(s.cuda_stream)))


def sparse_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, masks: AttentionMaskSet, *,
                     softmax_scale: Optional[float] = None, out: Optional[torch.Tensor] = None,
                     return_lse: bool = False, schedule: Optional[AttentionSchedule] = None,
                     device_schedule: bool = True):
    """O = softmax(Q K^T * scale) V restricted to the dense 64x64 tiles of
    `masks` (bit (q, k) of head h set => tile computed; reference
    mask.hpp:18-20).  q: [Sq, H, d], k/v: [Sk, H, d], bf16 CUDA, d in {64, 128}.
    Rows with no dense tile return 0 (LSE -inf)."""
    Sq, H, d = q.shape
    Sk = k.shape[0]
    bs = masks.block_size
    if bs != 64:
        raise ConfigError("the sm_100a kernel tiles 64-token blocks; block_size must be 64")
    if masks.num_heads != H or masks.num_q_blocks != -(-Sq // bs) or masks.num_kv_blocks != -(-Sk // bs):
        raise ContractError("mask grid does not match q/k shapes")
    if out is None:
        out = torch.empty_like(q)
    lse = torch.empty((H, Sq), dtype=torch.float32, device=q.device) if return_lse else None
    sched = schedule
    if sched is None and device_schedule:
        # K2: masks go to the device (1.3 MB for the Wan layer) and the work
        # list is built there; no host pass over the masks, no list upload.
        words = torch.from_numpy(masks.words.view(np.int64)).to(q.device, non_blocking=True)
        sched = AttentionSchedule().build_device(words, masks.num_kv_blocks, kv_tokens_global=Sk,
                                                 head_dim=q.shape[-1])
    elif sched is None:
        sched = AttentionSchedule().build(masks, kv_tokens_global=Sk, head_dim=q.shape[-1])
    sched.launch(q, k, v, out, lse=lse, softmax_scale=softmax_scale)
    if schedule is None:
        # keep the schedule (and its pinned staging buffer) alive until the
        # asynchronous upload has been consumed by the launch
        out._dbsp_schedule = sched
    return (out, lse) if return_lse else out


def mask_stats_device(words: torch.Tensor, num_kv_blocks: int):
    """K1: exact per-head counts and Q/KV marginals from device mask words."""
    if not words.is_cuda or words.dtype != torch.int64 or words.dim() != 3:
        raise ContractError("mask words must be a CUDA int64 tensor [heads, q_blocks, words]")
    H, nq, _ = words.shape
    dev = words.device
    hc = torch.empty(H, dtype=torch.int64, device=dev)
    rw = torch.empty(nq, dtype=torch.int64, device=dev)
    cw = torch.empty(num_kv_blocks, dtype=torch.int64, device=dev)
    s = torch.cuda.current_stream(dev)
    check(L.lib().dbsp_mask_stats_device(C.c_void_p(words.data_ptr()), H, nq, num_kv_blocks,
                                         C.c_void_p(hc.data_ptr()), C.c_void_p(rw.data_ptr()),
                                         C.c_void_p(cw.data_ptr()), C.c_void_p(s.cuda_stream)))
    return hc, rw, cw
