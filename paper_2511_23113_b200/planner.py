"""Python face of the db-SP planner API (reference proj/include/dbsp/*.hpp).

Names, argument meaning and error behaviour mirror the reference C++ API so
parity tests read like the reference's own; all computation happens in the
C ABI of libdbsp_b200.so (host C++ planner), never in Python.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Dict, Iterable, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib as L

# ---------------------------------------------------------------------------
# Errors (reference error.hpp:10-44)


class DbspError(RuntimeError):
    """dbsp::error"""


class ConfigError(DbspError):
    """dbsp::config_error"""


class IoError(DbspError):
    """dbsp::io_error"""


class ParseError(IoError):
    """dbsp::parse_error"""


class ContractError(DbspError):
    """dbsp::contract_error"""


class SearchSpaceError(ConfigError):
    """dbsp::search_space_error"""


class CudaError(DbspError):
    """CUDA runtime/driver failure inside the library."""


_CODES = {1: DbspError, 2: ConfigError, 3: IoError, 4: ContractError, 5: ParseError,
          6: SearchSpaceError, 7: CudaError}


def check(rc: int) -> None:
    if rc != 0:
        msg = L.lib().dbsp_last_error().decode(errors="replace")
        raise _CODES.get(rc, DbspError)(msg)


def _u64p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def _u32p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def _f64p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


# ---------------------------------------------------------------------------
# Mask model (mask.hpp)

PATTERNS = {"random": 0, "uniform-random": 0, "banded": 1, "banded-diagonal": 1, "clustered": 2}


class AttentionMaskSet:
    """Per-head block masks: words[h, q, w] bit k%64 of word k//64 (mask.hpp:18-28)."""

    def __init__(self, words: np.ndarray, num_kv_blocks: int, block_size: int = 64):
        words = np.ascontiguousarray(words, dtype=np.uint64)
        if words.ndim != 3:
            raise ConfigError("mask words must be [heads, q_blocks, words_per_row]")
        H, nq, wpr = words.shape
        if nq == 0 or num_kv_blocks == 0:
            raise ConfigError("BlockMask dimensions must be positive")
        if H == 0:
            raise ConfigError("mask set needs at least one head")
        if block_size == 0:
            raise ConfigError("block_size must be positive")
        if wpr != (num_kv_blocks + 63) // 64:
            raise ContractError("words_per_row does not match num_kv_blocks")
        tail = num_kv_blocks % 64
        if tail and np.any(words[:, :, -1] >> np.uint64(tail)):
            raise ContractError("padding bits past num_kv_blocks must be zero")
        self.words = words
        self.nk = int(num_kv_blocks)
        self.block_size = int(block_size)
        self._c = None

    # -- shape
    @property
    def num_heads(self) -> int:
        return self.words.shape[0]

    @property
    def num_q_blocks(self) -> int:
        return self.words.shape[1]

    @property
    def num_kv_blocks(self) -> int:
        return self.nk

    @property
    def words_per_row(self) -> int:
        return self.words.shape[2]

    def grid_cells(self) -> int:
        return self.num_heads * self.num_q_blocks * self.nk

    # -- conversion
    @classmethod
    def from_dense(cls, dense: np.ndarray, block_size: int = 64) -> "AttentionMaskSet":
        dense = np.asarray(dense, dtype=bool)
        H, nq, nk = dense.shape
        wpr = (nk + 63) // 64
        padded = np.zeros((H, nq, wpr * 64), dtype=bool)
        padded[:, :, :nk] = dense
        bits = np.packbits(padded.reshape(H, nq, wpr, 64), axis=-1, bitorder="little")
        words = bits.view(np.uint64).reshape(H, nq, wpr)
        return cls(words, nk, block_size)

    def to_dense(self) -> np.ndarray:
        H, nq, wpr = self.words.shape
        bits = np.unpackbits(self.words.view(np.uint8).reshape(H, nq, wpr * 8), axis=-1,
                             bitorder="little")
        return bits[:, :, : self.nk].astype(bool)

    def get(self, h: int, q: int, k: int) -> bool:
        return bool((int(self.words[h, q, k // 64]) >> (k % 64)) & 1)

    def set(self, h: int, q: int, k: int, value: bool = True) -> None:
        w = int(self.words[h, q, k // 64])
        bit = 1 << (k % 64)
        self.words[h, q, k // 64] = np.uint64((w | bit) if value else (w & ~bit))
        self._c = None

    def __eq__(self, other) -> bool:
        return (isinstance(other, AttentionMaskSet) and self.nk == other.nk
                and self.block_size == other.block_size and np.array_equal(self.words, other.words))

    # -- C view (per-head pointers into the contiguous buffer)
    def c(self) -> L.MaskSetT:
        if self._c is None:
            H = self.num_heads
            stride = self.num_q_blocks * self.words_per_row * 8
            base = self.words.ctypes.data
            ptrs = (C.POINTER(C.c_uint64) * H)(
                *[C.cast(C.c_void_p(base + h * stride), C.POINTER(C.c_uint64)) for h in range(H)])
            self._ptrs = ptrs
            self._c = L.MaskSetT(ptrs, H, self.num_q_blocks, self.nk, self.block_size)
        return self._c


@dataclass
class GeneratorSpec:
    """mask.hpp:137-162."""
    num_heads: int = 1
    num_q_blocks: int = 1
    num_kv_blocks: int = 1
    block_size: int = 64
    pattern: str = "random"
    min_density: float = 0.5
    max_density: float = 0.5
    skew: float = 1.0
    seed: int = 0


def generate_mask_set(spec: GeneratorSpec) -> AttentionMaskSet:
    if spec.pattern not in PATTERNS:
        raise ConfigError(f"unknown mask pattern '{spec.pattern}' (expected random|banded|clustered)")
    wpr = (spec.num_kv_blocks + 63) // 64
    words = np.zeros((max(spec.num_heads, 0), max(spec.num_q_blocks, 0), wpr), dtype=np.uint64)
    cs = L.GeneratorSpecT(spec.num_heads, spec.num_q_blocks, spec.num_kv_blocks, spec.block_size,
                          PATTERNS[spec.pattern], spec.min_density, spec.max_density, spec.skew,
                          spec.seed & 0xFFFFFFFFFFFFFFFF)
    check(L.lib().dbsp_generate_mask_set(C.byref(cs), _u64p(words)))
    return AttentionMaskSet(words, spec.num_kv_blocks, spec.block_size)


def perturb_mask_set(mset: AttentionMaskSet, flip_rate: float, seed: int) -> AttentionMaskSet:
    out = np.empty_like(mset.words)
    check(L.lib().dbsp_perturb_mask_set(C.byref(mset.c()), flip_rate, seed & 0xFFFFFFFFFFFFFFFF,
                                        _u64p(out)))
    return AttentionMaskSet(out, mset.nk, mset.block_size)


def save_mask_set(mset: AttentionMaskSet, path) -> None:
    """DBSPMSK1 binary file, written atomically (mask_io.hpp:131-147)."""
    check(L.lib().dbsp_save_mask_set(C.byref(mset.c()), str(path).encode()))


def load_mask_set(path) -> AttentionMaskSet:
    """DBSPMSK1 binary file, or the JSON hex sidecar accepted for fixtures
    (mask_io.hpp:80-127,149-207)."""
    p = str(path)
    try:
        with open(p, "rb") as f:
            head = f.read(64)
    except OSError:
        raise IoError(f"cannot open '{p}'") from None
    if not head.startswith(b"DBSPMSK1") and head.lstrip()[:1] == b"{":
        return _mask_set_from_sidecar(p)
    dims = [C.c_uint32() for _ in range(4)]
    check(L.lib().dbsp_load_mask_set_header(p.encode(), *[C.byref(d) for d in dims]))
    H, nq, nk, bs = (d.value for d in dims)
    words = np.zeros((H, nq, (nk + 63) // 64), np.uint64)
    check(L.lib().dbsp_load_mask_set(p.encode(), _u64p(words)))
    return AttentionMaskSet(words, nk, bs)


def _mask_set_from_sidecar(path: str) -> AttentionMaskSet:
    import json
    try:
        with open(path) as f:
            j = json.load(f)
    except json.JSONDecodeError as e:
        raise ParseError(f"{path}: invalid JSON sidecar: {e}") from None
    try:
        H, nq, nk, bs = (int(j[k]) for k in ("heads", "q_blocks", "kv_blocks", "block_size"))
        rows = j["rows"]
    except KeyError as e:
        raise ParseError(f"{path}: sidecar is missing a required key: {e}") from None
    if min(H, nq, nk, bs) <= 0:
        raise ParseError(f"{path}: sidecar dimensions must be positive")
    if len(rows) != H * nq:
        raise ParseError(f"{path}: sidecar needs heads*q_blocks row strings, got {len(rows)}")
    nbytes = (nk + 7) // 8
    dense = np.zeros((H * nq, nbytes * 8), bool)
    for r, hx in enumerate(rows):
        if len(hx) != 2 * nbytes:
            raise ParseError(f"{path}: row {r} needs {2 * nbytes} hex chars")
        try:
            b = bytes.fromhex(hx)
        except ValueError:
            raise ParseError(f"{path}: row {r} has a non-hex character") from None
        dense[r] = np.unpackbits(np.frombuffer(b, np.uint8), bitorder="little").astype(bool)
    return AttentionMaskSet.from_dense(dense[:, :nk].reshape(H, nq, nk), bs)


def mix_seed(base: int, a: int, b: int = 0) -> int:
    m = 0xFFFFFFFFFFFFFFFF
    return int(L.lib().dbsp_mix_seed(base & m, a & m, b & m))


def total_blocks(mset: AttentionMaskSet) -> int:
    out = C.c_uint64()
    check(L.lib().dbsp_total_blocks(C.byref(mset.c()), C.byref(out)))
    return out.value


def density(mset: AttentionMaskSet) -> float:
    out = C.c_double()
    check(L.lib().dbsp_density(C.byref(mset.c()), C.byref(out)))
    return out.value


def blocks_per_head(mset: AttentionMaskSet) -> List[int]:
    out = np.zeros(mset.num_heads, dtype=np.uint64)
    check(L.lib().dbsp_blocks_per_head(C.byref(mset.c()), _u64p(out)))
    return [int(v) for v in out]


# ---------------------------------------------------------------------------
# Strategy / plan / rho_s (metrics.hpp)


@dataclass(frozen=True, order=True)
class ParallelStrategy:
    ulysses: int = 1
    ring: int = 1

    def gpus(self) -> int:
        return self.ulysses * self.ring

    def __str__(self) -> str:
        return f"U{self.ulysses}R{self.ring}"

    def c(self) -> L.StrategyT:
        return L.StrategyT(self.ulysses, self.ring)


def parse_strategy(text: str) -> ParallelStrategy:
    """metrics.hpp:32-51."""
    def fail():
        raise ConfigError(f"invalid strategy '{text}' (expected UxRy)")
    if len(text) < 4 or text[0] != "U":
        fail()
    r = text.find("R", 1)
    if r < 0 or r == 1 or r + 1 >= len(text):
        fail()
    a, b = text[1:r], text[r + 1:]
    if not (a.isdigit() and b.isdigit()):
        fail()
    s = ParallelStrategy(int(a), int(b))
    if s.ulysses < 1 or s.ring < 1:
        fail()
    return s


def enumerate_strategies(total_gpus: int) -> List[ParallelStrategy]:
    buf = (L.StrategyT * 33)()
    n = C.c_uint32()
    check(L.lib().dbsp_enumerate_strategies(total_gpus, buf, C.byref(n)))
    return [ParallelStrategy(buf[i].ulysses, buf[i].ring) for i in range(n.value)]


@dataclass
class PartitionPlan:
    head_assignment: np.ndarray
    q_assignment: np.ndarray
    kv_assignment: np.ndarray

    @classmethod
    def empty(cls, mset: AttentionMaskSet) -> "PartitionPlan":
        return cls(np.zeros(mset.num_heads, np.uint32), np.zeros(mset.num_q_blocks, np.uint32),
                   np.zeros(mset.num_kv_blocks, np.uint32))

    @classmethod
    def of(cls, head, q, kv) -> "PartitionPlan":
        return cls(np.ascontiguousarray(head, np.uint32), np.ascontiguousarray(q, np.uint32),
                   np.ascontiguousarray(kv, np.uint32))

    def c(self) -> L.PlanT:
        for a in (self.head_assignment, self.q_assignment, self.kv_assignment):
            assert a.dtype == np.uint32 and a.flags.c_contiguous
        return L.PlanT(_u32p(self.head_assignment), _u32p(self.q_assignment),
                       _u32p(self.kv_assignment))

    def __eq__(self, o) -> bool:
        return (isinstance(o, PartitionPlan) and np.array_equal(self.head_assignment, o.head_assignment)
                and np.array_equal(self.q_assignment, o.q_assignment)
                and np.array_equal(self.kv_assignment, o.kv_assignment))

    def to_json(self, strategy: ParallelStrategy) -> dict:
        """plan_to_json (metrics.hpp:222-229)."""
        return {"strategy": {"x": strategy.ulysses, "y": strategy.ring},
                "head_assignment": self.head_assignment.tolist(),
                "q_assignment": self.q_assignment.tolist(),
                "kv_assignment": self.kv_assignment.tolist()}


def _plan_dims_ok(mset: AttentionMaskSet, plan: PartitionPlan) -> None:
    if (len(plan.head_assignment) != mset.num_heads or len(plan.q_assignment) != mset.num_q_blocks
            or len(plan.kv_assignment) != mset.num_kv_blocks):
        raise ContractError("plan dimensions do not match the mask set")


def validate_plan(mset: AttentionMaskSet, strategy: ParallelStrategy, plan: PartitionPlan) -> None:
    _plan_dims_ok(mset, plan)
    check(L.lib().dbsp_validate_plan(C.byref(mset.c()), strategy.c(), C.byref(plan.c())))


def default_plan(mset: AttentionMaskSet, strategy: ParallelStrategy) -> PartitionPlan:
    out = PartitionPlan.empty(mset)
    check(L.lib().dbsp_default_plan(C.byref(mset.c()), strategy.c(), C.byref(out.c())))
    return out


@dataclass
class WorkloadTable:
    gpus: int
    counts: np.ndarray  # periods x gpus, uint64

    @property
    def periods(self) -> int:
        return self.counts.shape[0]

    def total(self) -> int:
        return int(self.counts.sum())


def workload_table(mset: AttentionMaskSet, strategy: ParallelStrategy,
                   plan: PartitionPlan) -> WorkloadTable:
    _plan_dims_ok(mset, plan)
    x, y = strategy.ulysses, strategy.ring
    counts = np.zeros((max(1, y), max(1, x * y)), dtype=np.uint64)
    periods = C.c_uint32()
    check(L.lib().dbsp_workload_table(C.byref(mset.c()), strategy.c(), C.byref(plan.c()),
                                      _u64p(counts), C.byref(periods)))
    return WorkloadTable(x * y, counts[: periods.value].copy())


def imbalance_ratio(table) -> float:
    if isinstance(table, WorkloadTable):
        counts, gpus = np.ascontiguousarray(table.counts, np.uint64), table.gpus
    else:
        counts = np.ascontiguousarray(np.asarray(table[0], dtype=np.uint64))
        gpus = int(table[1])
    counts = counts.reshape(-1, gpus) if counts.size else counts.reshape(0, max(gpus, 1))
    out = C.c_double()
    check(L.lib().dbsp_imbalance_ratio(_u64p(counts), counts.shape[0], gpus, C.byref(out)))
    return out.value


@dataclass
class ExchangeVolume:
    q_blocks_moved: int = 0
    kv_blocks_moved: int = 0
    token_payload: int = 0


def exchange_volume(mset: AttentionMaskSet, strategy: ParallelStrategy,
                    plan: PartitionPlan) -> ExchangeVolume:
    _plan_dims_ok(mset, plan)
    e = L.ExchangeT()
    check(L.lib().dbsp_exchange_volume(C.byref(mset.c()), strategy.c(), C.byref(plan.c()),
                                       C.byref(e)))
    return ExchangeVolume(e.q_blocks_moved, e.kv_blocks_moved, e.token_payload)


# ---------------------------------------------------------------------------
# Partitioner (planner.hpp)

kInfiniteReward = math.inf


@dataclass
class PlannerConfig:
    reuse_threshold: float = 1.10  # P_s
    exchange_reward: float = 0.0   # R_b

    def c(self) -> L.PlannerConfigT:
        return L.PlannerConfigT(self.reuse_threshold, self.exchange_reward)


@dataclass
class PlanOutcome:
    plan: PartitionPlan
    head_replanned: bool = False
    rho_pre: float = 1.0
    rho_post: float = 1.0


def summed_grid(mset: AttentionMaskSet) -> np.ndarray:
    out = np.zeros(mset.num_q_blocks * mset.num_kv_blocks, dtype=np.uint64)
    check(L.lib().dbsp_summed_grid(C.byref(mset.c()), _u64p(out)))
    return out


def head_level_imbalance(weights: Sequence[int], assignment: Sequence[int], x: int) -> float:
    w = np.ascontiguousarray(weights, np.uint64)
    a = np.ascontiguousarray(assignment, np.uint32)
    out = C.c_double()
    check(L.lib().dbsp_head_level_imbalance(_u64p(w), _u32p(a), len(w), x, C.byref(out)))
    return out.value


def partition_heads(mset: AttentionMaskSet, x: int) -> np.ndarray:
    out = np.zeros(mset.num_heads, np.uint32)
    check(L.lib().dbsp_partition_heads(C.byref(mset.c()), x, _u32p(out)))
    return out


def partition_blocks(mset: AttentionMaskSet, y: int, reward: float) -> Tuple[np.ndarray, np.ndarray]:
    q = np.zeros(mset.num_q_blocks, np.uint32)
    kv = np.zeros(mset.num_kv_blocks, np.uint32)
    check(L.lib().dbsp_partition_blocks(C.byref(mset.c()), y, reward, _u32p(q), _u32p(kv)))
    return q, kv


def biased_greedy(weights: Sequence[int], y: int, reward: float) -> np.ndarray:
    w = np.ascontiguousarray(weights, np.uint64)
    out = np.zeros(len(w), np.uint32)
    check(L.lib().dbsp_biased_greedy(_u64p(w), len(w), y, reward, _u32p(out)))
    return out


def plan_dual(mset: AttentionMaskSet, strategy: ParallelStrategy, config: PlannerConfig = None,
              prev: Optional[PartitionPlan] = None) -> PlanOutcome:
    config = config or PlannerConfig()
    if prev is not None:
        _plan_dims_ok(mset, prev)
    out = PartitionPlan.empty(mset)
    oc = L.PlanOutcomeT()
    prev_c = C.byref(prev.c()) if prev is not None else None
    check(L.lib().dbsp_plan_dual(C.byref(mset.c()), strategy.c(), C.byref(config.c()), prev_c,
                                 C.byref(out.c()), C.byref(oc)))
    return PlanOutcome(out, bool(oc.head_replanned), oc.rho_pre, oc.rho_post)


def brute_force_heads(mset: AttentionMaskSet, x: int) -> np.ndarray:
    out = np.zeros(mset.num_heads, np.uint32)
    check(L.lib().dbsp_brute_force_heads(C.byref(mset.c()), x, _u32p(out)))
    return out


def brute_force_blocks(grid: Sequence[int], nq: int, nk: int, y: int):
    g = np.ascontiguousarray(grid, np.uint64)
    if g.size != nq * nk:
        raise ContractError("summed grid size does not match its dimensions")
    q = np.zeros(nq, np.uint32)
    kv = np.zeros(nk, np.uint32)
    rho = C.c_double()
    check(L.lib().dbsp_brute_force_blocks(_u64p(g), nq, nk, y, _u32p(q), _u32p(kv), C.byref(rho)))
    return q, kv, rho.value


# ---------------------------------------------------------------------------
# Latency model (latency.hpp)


@dataclass
class PiecewiseLinear:
    xs: List[float] = field(default_factory=list)
    ys: List[float] = field(default_factory=list)

    def eval(self, x: float) -> float:
        xs = np.ascontiguousarray(self.xs, np.float64)
        ys = np.ascontiguousarray(self.ys, np.float64)
        out = C.c_double()
        check(L.lib().dbsp_pwl_eval(_f64p(xs), _f64p(ys), len(xs), x, C.byref(out)))
        return out.value


@dataclass
class MachineProfile:
    all2all: Dict[int, PiecewiseLinear] = field(default_factory=dict)
    p2p: Dict[int, PiecewiseLinear] = field(default_factory=dict)
    dense_attn_seconds: float = 0.0
    launch_seconds: float = 0.0
    exchange_overlap: float = 1.0
    replan_seconds: float = 0.0
    bytes_per_token_per_head: float = 256.0

    def c(self) -> L.ProfileT:
        keep = []

        def flat(curves: Dict[int, PiecewiseLinear]):
            degs = sorted(curves)
            d = np.array(degs, np.uint32)
            off = np.zeros(len(degs) + 1, np.uint32)
            xs, ys = [], []
            for i, k in enumerate(degs):
                xs += list(curves[k].xs)
                ys += list(curves[k].ys)
                off[i + 1] = len(xs)
            x = np.array(xs, np.float64)
            y = np.array(ys, np.float64)
            keep.extend([d, off, x, y])
            return len(degs), _u32p(d), _u32p(off), _f64p(x), _f64p(y)

        a = flat(self.all2all)
        p = flat(self.p2p)
        st = L.ProfileT(*a, *p, self.dense_attn_seconds, self.launch_seconds,
                        self.exchange_overlap, self.replan_seconds, self.bytes_per_token_per_head)
        st._keep = keep
        return st

    def all2all_at(self, degree: int, payload: float) -> float:
        if degree not in self.all2all:
            raise ConfigError(f"profile missing all2all degree {degree}")
        return self.all2all[degree].eval(payload)

    def p2p_at(self, degree: int, payload: float) -> float:
        if degree not in self.p2p:
            raise ConfigError(f"profile missing p2p degree {degree}")
        return self.p2p[degree].eval(payload)

    # profile JSON (latency.hpp:318-379): stored as samples, re-fitted on load.
    def to_json(self) -> dict:
        def curves(t):
            return [{"degree": d, "payload_bytes": x, "seconds": y}
                    for d in sorted(t) for x, y in zip(t[d].xs, t[d].ys)]
        return {"all2all": curves(self.all2all), "p2p": curves(self.p2p),
                "dense": [{"density": 0.0, "seconds": self.launch_seconds},
                          {"density": 1.0, "seconds": self.launch_seconds + self.dense_attn_seconds}],
                "exchange_overlap": self.exchange_overlap, "replan_seconds": self.replan_seconds,
                "bytes_per_token_per_head": self.bytes_per_token_per_head}

    @classmethod
    def from_json(cls, j: dict) -> "MachineProfile":
        samples = []
        for prim in ("all2all", "p2p"):
            for e in j.get(prim, []):
                samples.append(ProfileSample(prim, int(e["degree"]), float(e["payload_bytes"]),
                                             float(e["seconds"])))
        for e in j["dense"]:
            samples.append(ProfileSample("dense", 1, float(e["density"]), float(e["seconds"])))
        return fit_profile(samples, FitOptions(j.get("exchange_overlap", 1.0),
                                               j.get("replan_seconds", 0.0),
                                               j.get("bytes_per_token_per_head", 256.0)))


@dataclass
class ProfileSample:
    primitive: str
    degree: int = 1
    x: float = 0.0
    seconds: float = 0.0


@dataclass
class FitOptions:
    exchange_overlap: float = 1.0
    replan_seconds: float = 0.0
    bytes_per_token_per_head: float = 256.0


_PRIM = {"all2all": 0, "p2p": 1, "dense": 2}


def fit_profile(samples: Iterable[ProfileSample], options: FitOptions = None) -> MachineProfile:
    samples = list(samples)
    options = options or FitOptions()
    for s in samples:
        if s.primitive not in _PRIM:
            raise ConfigError(f"unknown profile primitive '{s.primitive}'")
    n = len(samples)
    arr = (L.ProfileSampleT * max(n, 1))(*[L.ProfileSampleT(_PRIM[s.primitive], s.degree, s.x, s.seconds)
                                           for s in samples])
    deg = np.zeros(n + 1, np.uint32), np.zeros(n + 1, np.uint32)
    off = np.zeros(n + 2, np.uint32), np.zeros(n + 2, np.uint32)
    xs = np.zeros(n + 1, np.float64), np.zeros(n + 1, np.float64)
    ys = np.zeros(n + 1, np.float64), np.zeros(n + 1, np.float64)
    st = L.ProfileStorageT(_u32p(deg[0]), _u32p(off[0]), _f64p(xs[0]), _f64p(ys[0]),
                           _u32p(deg[1]), _u32p(off[1]), _f64p(xs[1]), _f64p(ys[1]))
    out = L.ProfileT()
    opt = L.FitOptionsT(options.exchange_overlap, options.replan_seconds,
                        options.bytes_per_token_per_head)
    check(L.lib().dbsp_fit_profile(arr, n, C.byref(opt), C.byref(st), C.byref(out)))

    def curves(i, count):
        res = {}
        for c in range(count):
            a, b = int(off[i][c]), int(off[i][c + 1])
            res[int(deg[i][c])] = PiecewiseLinear(xs[i][a:b].tolist(), ys[i][a:b].tolist())
        return res

    return MachineProfile(curves(0, out.num_all2all), curves(1, out.num_p2p), out.dense_attn_seconds,
                          out.launch_seconds, out.exchange_overlap, out.replan_seconds,
                          out.bytes_per_token_per_head)


@dataclass
class LatencyBreakdown:
    all2all_s: float = 0.0
    attn_compute_s: float = 0.0
    ring_p2p_exposed_s: float = 0.0
    imbalance_penalty_s: float = 0.0
    exchange_s: float = 0.0
    replan_s: float = 0.0
    total_s: float = 0.0

    def attn_seconds(self) -> float:
        return self.attn_compute_s + self.ring_p2p_exposed_s + self.imbalance_penalty_s

    @classmethod
    def of(cls, t: L.LatencyT) -> "LatencyBreakdown":
        return cls(t.all2all_s, t.attn_compute_s, t.ring_p2p_exposed_s, t.imbalance_penalty_s,
                   t.exchange_s, t.replan_s, t.total_s)


@dataclass
class MaskShape:
    heads: int = 1
    q_blocks: int = 1
    kv_blocks: int = 1
    block_size: int = 1


@dataclass
class CallInputs:
    shape: MaskShape = field(default_factory=MaskShape)
    strategy: ParallelStrategy = field(default_factory=ParallelStrategy)
    density: float = 0.0
    rho: float = 1.0
    exchange: ExchangeVolume = field(default_factory=ExchangeVolume)
    charge_replan: bool = False


def predict_from_inputs(inp: CallInputs, profile: MachineProfile) -> LatencyBreakdown:
    ci = L.CallInputsT(inp.shape.heads, inp.shape.q_blocks, inp.shape.kv_blocks,
                       inp.shape.block_size, inp.strategy.c(), inp.density, inp.rho,
                       L.ExchangeT(inp.exchange.q_blocks_moved, inp.exchange.kv_blocks_moved,
                                   inp.exchange.token_payload), int(inp.charge_replan))
    out = L.LatencyT()
    pc = profile.c()
    check(L.lib().dbsp_predict_from_inputs(C.byref(ci), C.byref(pc), C.byref(out)))
    return LatencyBreakdown.of(out)


def predict_latency(mset: AttentionMaskSet, strategy: ParallelStrategy, plan: PartitionPlan,
                    profile: MachineProfile, charge_replan: bool = False) -> LatencyBreakdown:
    _plan_dims_ok(mset, plan)
    out = L.LatencyT()
    pc = profile.c()
    check(L.lib().dbsp_predict_latency(C.byref(mset.c()), strategy.c(), C.byref(plan.c()),
                                       C.byref(pc), int(charge_replan), C.byref(out)))
    return LatencyBreakdown.of(out)


@dataclass
class StrategyPrediction:
    strategy: ParallelStrategy
    outcome: PlanOutcome
    latency: LatencyBreakdown


def predict_all(mset: AttentionMaskSet, profile: MachineProfile, total_gpus: int,
                config: PlannerConfig = None,
                prev_plans: Optional[Dict[ParallelStrategy, PartitionPlan]] = None
                ) -> List[StrategyPrediction]:
    config = config or PlannerConfig()
    prev_plans = prev_plans or {}
    n_prev = len(prev_plans)
    ps = (L.StrategyT * max(n_prev, 1))(*[s.c() for s in prev_plans])
    pp = (L.PlanT * max(n_prev, 1))(*[p.c() for p in prev_plans.values()])
    out = (L.PredictionT * 33)()
    plans = [PartitionPlan.empty(mset) for _ in range(33)]
    plans_c = (L.PlanT * 33)(*[p.c() for p in plans])
    n = C.c_uint32()
    pc = profile.c()
    check(L.lib().dbsp_predict_all(C.byref(mset.c()), C.byref(pc), total_gpus, C.byref(config.c()),
                                   ps, pp, n_prev, out, plans_c, C.byref(n)))
    res = []
    for i in range(n.value):
        o = out[i]
        res.append(StrategyPrediction(
            ParallelStrategy(o.strategy.ulysses, o.strategy.ring),
            PlanOutcome(plans[i], bool(o.outcome.head_replanned), o.outcome.rho_pre, o.outcome.rho_post),
            LatencyBreakdown.of(o.latency)))
    return res


# ---------------------------------------------------------------------------
# Selector (selector.hpp)


class SelectorState:
    """Per-layer memory of the last (strategy, plan); internally locked."""

    def __init__(self, total_gpus: int):
        h = C.c_void_p()
        check(L.lib().dbsp_selector_create(total_gpus, C.byref(h)))
        self._h = h
        self._gpus = total_gpus

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            L.lib().dbsp_selector_destroy(h)
            self._h = None

    def total_gpus(self) -> int:
        return self._gpus

    def prebuilt_groups(self) -> List[ParallelStrategy]:
        return enumerate_strategies(self._gpus)

    def stored(self, layer: int):
        found = C.c_int32()
        s = L.StrategyT()
        sizes = np.zeros(3, np.uint32)
        check(L.lib().dbsp_selector_stored(self._h, layer, C.byref(found), C.byref(s), _u32p(sizes), None))
        if not found.value:
            return None
        plan = PartitionPlan(np.zeros(sizes[0], np.uint32), np.zeros(sizes[1], np.uint32),
                             np.zeros(sizes[2], np.uint32))
        check(L.lib().dbsp_selector_stored(self._h, layer, C.byref(found), C.byref(s), _u32p(sizes),
                                           C.byref(plan.c())))
        return ParallelStrategy(s.ulysses, s.ring), plan

    def store(self, layer: int, strategy: ParallelStrategy, plan: PartitionPlan) -> None:
        sizes = np.array([len(plan.head_assignment), len(plan.q_assignment), len(plan.kv_assignment)],
                         np.uint32)
        check(L.lib().dbsp_selector_store(self._h, layer, strategy.c(), C.byref(plan.c()), _u32p(sizes)))


@dataclass
class Selection:
    strategy: ParallelStrategy
    outcome: PlanOutcome
    latency: LatencyBreakdown


def select(layer_id: int, mset: AttentionMaskSet, profile: MachineProfile,
           config: PlannerConfig, state: SelectorState) -> Selection:
    s = L.StrategyT()
    plan = PartitionPlan.empty(mset)
    oc = L.PlanOutcomeT()
    lat = L.LatencyT()
    pc = profile.c()
    check(L.lib().dbsp_select(state._h, layer_id, C.byref(mset.c()), C.byref(pc),
                              C.byref(config.c()), C.byref(s), C.byref(plan.c()), C.byref(oc),
                              C.byref(lat)))
    return Selection(ParallelStrategy(s.ulysses, s.ring),
                     PlanOutcome(plan, bool(oc.head_replanned), oc.rho_pre, oc.rho_post),
                     LatencyBreakdown.of(lat))


def select_two_phase(layer_id: int, mset: AttentionMaskSet, profile: MachineProfile,
                     config: PlannerConfig, state: SelectorState) -> Selection:
    """select() through the two-phase path of select_device (assignments, then
    one batch of workload tables), tables on the host.  Same result as select()."""
    s = L.StrategyT()
    plan = PartitionPlan.empty(mset)
    oc = L.PlanOutcomeT()
    lat = L.LatencyT()
    pc = profile.c()
    check(L.lib().dbsp_select_two_phase(state._h, layer_id, C.byref(mset.c()), C.byref(pc),
                                        C.byref(config.c()), C.byref(s), C.byref(plan.c()), C.byref(oc),
                                        C.byref(lat)))
    return Selection(ParallelStrategy(s.ulysses, s.ring),
                     PlanOutcome(plan, bool(oc.head_replanned), oc.rho_pre, oc.rho_post),
                     LatencyBreakdown.of(lat))


def select_device(layer_id: int, words, num_kv_blocks: int, profile: MachineProfile, config: PlannerConfig,
                  state: SelectorState, block_size: int = 64, stream=None) -> Selection:
    """select() with the mask integers computed on the GPU (dbsp_select_device).
    words: contiguous CUDA int64 tensor [H, Nq, ceil(Nk/64)] of BlockMask rows."""
    import torch
    if not words.is_cuda or words.dtype != torch.int64 or words.dim() != 3 or not words.is_contiguous():
        raise ContractError("device mask words must be a contiguous CUDA int64 [H, Nq, words] tensor")
    H, nq, _ = words.shape
    s = L.StrategyT()
    plan = PartitionPlan(np.zeros(H, np.uint32), np.zeros(nq, np.uint32), np.zeros(num_kv_blocks, np.uint32))
    oc = L.PlanOutcomeT()
    lat = L.LatencyT()
    pc = profile.c()
    st = stream if stream is not None else torch.cuda.current_stream(words.device)
    check(L.lib().dbsp_select_device(state._h, layer_id, C.c_void_p(words.data_ptr()), H, nq, num_kv_blocks,
                                     block_size, C.byref(pc), C.byref(config.c()), C.byref(s),
                                     C.byref(plan.c()), C.byref(oc), C.byref(lat), C.c_void_p(st.cuda_stream)))
    return Selection(ParallelStrategy(s.ulysses, s.ring),
                     PlanOutcome(plan, bool(oc.head_replanned), oc.rho_pre, oc.rho_post),
                     LatencyBreakdown.of(lat))
