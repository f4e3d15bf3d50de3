"""ORACLE package — test infrastructure only.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
`--impl reference`) may import this package, and only as the checker or as
the timed CPU baseline.  The product (paper_2511_23113_b200) never imports it.

Contents
  attention_ref.c   fp32-in / double-accumulate block-sparse attention (OpenMP)
  planner_ref.py    pure-Python restatement of the reference planner
  Makefile          builds liboracle_attn.so and, when /root/reference is
                    present, the compiled reference tools into oracle/_ref/
  ref_tools/        our drivers compiled against the reference headers
                    (golden_dump: planner golden vectors; ref_bench: timing)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ATTN_LIB = HERE / "liboracle_attn.so"
REF_DIR = HERE / "_ref"
REFERENCE_ROOT = Path("/root/reference/proj/include")

_attn = None


def build(reference: bool = True) -> None:
    """Compile the C oracle (always) and the reference tools (when the
    reference tree is present, i.e. in the build container)."""
    targets = ["attn"]
    if reference and REFERENCE_ROOT.exists():
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", str(HERE)] + targets, check=True)


def _lib():
    global _attn
    if _attn is None:
        if not ATTN_LIB.exists():
            build(reference=False)
        lib = C.CDLL(str(ATTN_LIB))
        lib.oracle_sparse_attention.restype = C.c_int
        lib.oracle_sparse_attention.argtypes = [
            C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
            C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_float, C.c_void_p, C.c_void_p,
            C.c_int64, C.c_void_p, C.c_void_p]
        lib.oracle_num_threads.restype = C.c_int
        lib.oracle_fnv1a.restype = C.c_uint64
        lib.oracle_fnv1a.argtypes = [C.c_void_p, C.c_uint64]
        _attn = lib
    return _attn


def fnv1a(words: np.ndarray) -> str:
    a = np.ascontiguousarray(words)
    return str(_lib().oracle_fnv1a(a.ctypes.data, a.nbytes))


def num_threads() -> int:
    return int(_lib().oracle_num_threads())


def sparse_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, words: np.ndarray, nk: int,
                     scale: float = None, rows: np.ndarray = None, kv_allow: np.ndarray = None,
                     block: int = 64):
    """q [Sq,H,d], k/v [Sk,H,d] float32; words [H,Nq,wpr] uint64.
    rows: optional int32 [(head, q_block), ...]; only those rows are written.
    Returns (out [Sq,H,d] float32, lse [H,Sq] float32)."""
    q = np.ascontiguousarray(q, np.float32)
    k = np.ascontiguousarray(k, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    words = np.ascontiguousarray(words, np.uint64)
    Sq, H, d = q.shape
    Sk = k.shape[0]
    nq = words.shape[1]
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    out = np.zeros_like(q)
    lse = np.full((H, Sq), -np.inf, np.float32)
    rp, nrows = None, 0
    if rows is not None:
        rows = np.ascontiguousarray(rows, np.int32).reshape(-1, 2)
        rp, nrows = rows.ctypes.data, rows.shape[0]
    ka = None
    if kv_allow is not None:
        kv_allow = np.ascontiguousarray(kv_allow, np.uint64)
        ka = kv_allow.ctypes.data
    rc = _lib().oracle_sparse_attention(q.ctypes.data, k.ctypes.data, v.ctypes.data, Sq, Sk, H, d,
                                        words.ctypes.data, nq, nk, block, float(scale), ka, rp,
                                        nrows, out.ctypes.data, lse.ctypes.data)
    if rc:
        raise ValueError("oracle: mask grid smaller than the token counts")
    return out, lse


def load_mask_words(path) -> tuple:
    """DBSPMSK1 file (reference mask_io.hpp:17-28: 28-byte header, then
    heads*q_blocks rows of ceil(kv_blocks/8) bytes, key k at byte k/8 bit k%8)
    -> (words uint64 [H, Nq, ceil(Nk/64)] in the BlockMask row layout, Nk)."""
    data = np.fromfile(str(path), np.uint8)
    if data[:8].tobytes() != b"DBSPMSK1":
        raise ValueError(f"{path}: not a DBSPMSK1 file")
    H, nq, nk, _bs = (int(x) for x in data[12:28].view("<u4"))
    rb, wpr = (nk + 7) // 8, (nk + 63) // 64
    rows = data[28:28 + H * nq * rb].reshape(H * nq, rb)
    padded = np.zeros((H * nq, wpr * 8), np.uint8)
    padded[:, :rb] = rows
    return padded.view("<u8").reshape(H, nq, wpr).astype(np.uint64), nk


def ref_tool(name: str) -> Path:
    """Path of a compiled reference tool in oracle/_ref (built here, shipped
    to the GPU box with the snapshot)."""
    return REF_DIR / name
