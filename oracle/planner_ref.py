"""ORACLE — test infrastructure only (never imported by the product path).

Pure-Python restatement of the reference db-SP planner, function by function,
for small cases.  Each function cites the reference it restates
(paths under /root/reference/proj/include/dbsp/).  It is pinned against the
golden vectors dumped by the compiled reference (oracle/_ref/golden_dump,
tests/golden/planner_golden.json) in tests/test_oracle.py, and the product
planner (C++ in libdbsp_b200.so) is checked against both.

Masks here are numpy bool arrays [H, Nq, Nk] (dense) for clarity.
"""
from __future__ import annotations

import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

M64 = (1 << 64) - 1


# rng.hpp:10-35 (splitmix64) -------------------------------------------------
class Rng:
    def __init__(self, seed: int):
        self.s = seed & M64

    def next_u64(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & M64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def next_double(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def bernoulli(self, p: float) -> bool:
        return self.next_double() < p

    def next_below(self, n: int) -> int:
        return (self.next_u64() * n) >> 64


# rng.hpp:37-40
def mix_seed(base: int, a: int, b: int = 0) -> int:
    return Rng(base ^ ((a * 0x9E3779B97F4A7C15) & M64) ^ ((b * 0xC2B2AE3D27D4EB4F) & M64)).next_u64()


# mask.hpp:157-161
def head_density(h: int, H: int, dmin: float, dmax: float, skew: float) -> float:
    t = math.pow(float(h) / float(H - 1), skew) if H > 1 else 0.0
    return dmin + (dmax - dmin) * t


def _llround(x: float) -> int:
    # std::llround: half away from zero (x - floor(x) is exact in binary64)
    if x < 0:
        return -_llround(-x)
    r = math.floor(x)
    return int(r) + (1 if x - r >= 0.5 else 0)


# mask.hpp:166-228
def gen_head(pattern: str, nq: int, nk: int, p: float, rng: Rng) -> np.ndarray:
    m = np.zeros((nq, nk), dtype=bool)
    if pattern == "random":
        for q in range(nq):
            for k in range(nk):
                if rng.bernoulli(p):
                    m[q, k] = True
        return m
    cells = nq * nk
    target = _llround(p * float(cells))
    if pattern == "banded":
        if target == 0:
            return m
        order = sorted((abs(float(q) - float(k) * nq / nk), q * nk + k)
                       for q in range(nq) for k in range(nk))
        for _, c in order[:target]:
            m[c // nk, c % nk] = True
        return m
    # clustered
    count, stalled = 0, 0
    while count < target and stalled < 256:
        h = 1 + rng.next_below(max(1, nq // 4))
        w = 1 + rng.next_below(max(1, nk // 4))
        q0 = rng.next_below(nq - h + 1)
        k0 = rng.next_below(nk - w + 1)
        added = 0
        for q in range(q0, q0 + h):
            if count >= target:
                break
            for k in range(k0, k0 + w):
                if count >= target:
                    break
                if not m[q, k]:
                    m[q, k] = True
                    count += 1
                    added += 1
        stalled = 0 if added else stalled + 1
    for q in range(nq):
        for k in range(nk):
            if count >= target:
                break
            if not m[q, k]:
                m[q, k] = True
                count += 1
    return m


# mask.hpp:233-256
def generate_mask_set(H, nq, nk, pattern="random", dmin=0.5, dmax=0.5, skew=1.0, seed=0):
    return np.stack([gen_head(pattern, nq, nk, head_density(h, H, dmin, dmax, skew),
                              Rng(mix_seed(seed, h))) for h in range(H)])


# mask.hpp:260-273
def perturb_mask_set(masks: np.ndarray, flip: float, seed: int) -> np.ndarray:
    out = masks.copy()
    if flip == 0.0:
        return out
    H, nq, nk = masks.shape
    for h in range(H):
        rng = Rng(mix_seed(seed, h))
        for q in range(nq):
            for k in range(nk):
                if rng.bernoulli(flip):
                    out[h, q, k] = not out[h, q, k]
    return out


def blocks_per_head(masks) -> List[int]:
    return [int(m.sum()) for m in masks]


def density(masks) -> float:
    return float(int(masks.sum())) / float(masks.size)


# metrics.hpp:56-66
def enumerate_strategies(G: int) -> List[Tuple[int, int]]:
    out, x = [], G
    while True:
        out.append((x, G // x))
        if x == 1:
            break
        x //= 2
    return out


# metrics.hpp:94-113
def default_plan(H, nq, nk, x, y):
    return ([h * x // H for h in range(H)], [q * y // nq for q in range(nq)],
            [k * y // nk for k in range(nk)])


# metrics.hpp:133-168
def workload_table(masks, x, y, plan) -> List[List[int]]:
    head, qa, ka = plan
    H, nq, nk = masks.shape
    G = x * y
    if y == 1:
        row = [0] * G
        for h in range(H):
            row[head[h]] += int(masks[h].sum())
        return [row]
    t = [[0] * G for _ in range(y)]
    ka = np.asarray(ka)
    for h in range(H):
        u = head[h]
        for q in range(nq):
            r = qa[q]
            for g in range(y):
                c = int(masks[h, q, ka == g].sum())
                if c:
                    t[(g + y - r) % y][u * y + r] += c
    return t


# metrics.hpp:173-186
def imbalance_ratio(counts, gpus) -> float:
    total = sum(sum(r) for r in counts)
    if total == 0:
        return 1.0
    return float(sum(max(r) for r in counts)) * float(gpus) / float(total)


# metrics.hpp:198-211
def exchange_volume(nq, nk, y, q_assign, kv_assign, block_size):
    qm = sum(1 for q in range(nq) if q_assign[q] != q * y // nq)
    km = sum(1 for k in range(nk) if kv_assign[k] != k * y // nk)
    return qm, km, (qm + 2 * km) * block_size


# planner.hpp:65-76
def head_level_imbalance(w, a, x) -> float:
    loads = [0] * x
    for i, wi in enumerate(w):
        loads[a[i]] += wi
    total = sum(w)
    if total == 0:
        return 1.0
    return float(max(loads)) * x / float(total)


# planner.hpp:82-90
def descending_order(w) -> List[int]:
    return sorted(range(len(w)), key=lambda i: (-w[i], i))


# planner.hpp:96-112
def partition_heads(w, x) -> List[int]:
    a, loads = [0] * len(w), [0] * x
    for h in descending_order(w):
        best = 0
        for r in range(1, x):
            if loads[r] < loads[best]:
                best = r
        a[h] = best
        loads[best] += w[h]
    return a


# planner.hpp:119-145
def biased_greedy(w, y, reward) -> List[int]:
    n = len(w)
    if math.isinf(reward):
        return [i * y // n for i in range(n)]
    a, loads = [0] * n, [0] * y
    for i in descending_order(w):
        home = i * y // n
        bias = reward * float(w[i])
        best, best_load = 0, float(loads[0]) - (bias if home == 0 else 0.0)
        for r in range(1, y):
            l = float(loads[r]) - (bias if home == r else 0.0)
            if l < best_load:
                best, best_load = r, l
        a[i] = best
        loads[best] += w[i]
    return a


# planner.hpp:47-61 + 151-170
def partition_blocks(masks, y, reward):
    grid = masks.sum(axis=0).astype(np.int64)
    qw = [int(v) for v in grid.sum(axis=1)]
    kw = [int(v) for v in grid.sum(axis=0)]
    return biased_greedy(qw, y, reward), biased_greedy(kw, y, reward)


# planner.hpp:175-217
def plan_dual(masks, x, y, ps=1.10, rb=0.0, prev=None):
    H, nq, nk = masks.shape
    pre = prev if prev is not None else default_plan(H, nq, nk, x, y)
    rho_pre = imbalance_ratio(workload_table(masks, x, y, pre), x * y)
    replanned = False
    if x > 1:
        reuse = prev is not None and head_level_imbalance(blocks_per_head(masks), prev[0], x) <= ps
        if reuse:
            head = list(prev[0])
        else:
            head = partition_heads(blocks_per_head(masks), x)
            replanned = True
    else:
        head = [0] * H
    if y > 1:
        qa, ka = partition_blocks(masks, y, rb)
    else:
        qa, ka = [0] * nq, [0] * nk
    plan = (head, qa, ka)
    rho_post = imbalance_ratio(workload_table(masks, x, y, plan), x * y)
    return plan, replanned, rho_pre, rho_post


# latency.hpp:27-40
def pwl_eval(xs, ys, x) -> float:
    import bisect
    if len(xs) == 1:
        return ys[0]
    hi = bisect.bisect_right(xs, x)
    hi = max(hi, 1)
    if hi == len(xs):
        hi = len(xs) - 1
    lo = hi - 1
    if x == xs[lo]:
        return ys[lo]
    if x == xs[hi]:
        return ys[hi]
    if ys[lo] == ys[hi]:
        return ys[lo]
    t = (x - xs[lo]) / (xs[hi] - xs[lo])
    return max(0.0, ys[lo] + t * (ys[hi] - ys[lo]))


# latency.hpp:225-268 ; profile = dict(all2all={deg:(xs,ys)}, p2p=..., dense, launch, overlap,
# replan, bpt)
def predict_from_inputs(H, nq, nk, bs, x, y, dens, rho, payload, charge_replan, prof) -> Dict:
    gpus = float(x) * y
    q_tok = float(nq) * bs
    kv_tok = float(nk) * bs
    heads = float(H)
    bpt = prof["bpt"]
    it = prof["dense"] * dens / (gpus * y) + prof["launch"]
    a2a = 0.0
    if x > 1:
        qkv = (q_tok + 2.0 * kv_tok) * heads * bpt
        a2a = pwl_eval(*prof["all2all"][x], qkv / gpus)
    exp_it = 0.0
    if y > 1:
        kvb = 2.0 * (kv_tok / y) * (heads / x) * bpt
        exp_it = max(0.0, pwl_eval(*prof["p2p"][y], kvb) - it)
    comp = it * y
    exposed = exp_it * (y - 1)
    body = comp + exposed
    imb = body * (rho - 1.0) if rho > 1.0 else 0.0
    exch = 0.0
    if payload > 0 and prof["overlap"] < 1.0:
        b = float(payload) * (float(H) / x) * bpt
        exch = (1.0 - prof["overlap"]) * pwl_eval(*prof["all2all"][y], b / y)
    rep = prof["replan"] if charge_replan else 0.0
    total = a2a + comp + exposed + imb + exch + rep
    return dict(all2all=a2a, compute=comp, exposed=exposed, imbalance=imb, exchange=exch,
                replan=rep, total=total)


# latency.hpp:295-315 + selector.hpp:55-75 (one call; prev = {(x,y): plan})
def select(masks, G, prof, ps=1.10, rb=0.0, prev: Optional[dict] = None):
    H, nq, nk = masks.shape
    prev = prev or {}
    preds = []
    for x, y in enumerate_strategies(G):
        if x > H or y > min(nq, nk):
            continue
        plan, rep, pre, post = plan_dual(masks, x, y, ps, rb, prev.get((x, y)))
        _, _, payload = exchange_volume(nq, nk, y, plan[1], plan[2], 64)
        lat = predict_from_inputs(H, nq, nk, 64, x, y, density(masks), post, payload, False, prof)
        preds.append(((x, y), plan, rep, pre, post, lat))
    best = 0
    for i in range(1, len(preds)):
        if preds[i][5]["total"] < preds[best][5]["total"]:
            best = i
    return preds[best], preds
