"""Pin the oracles before trusting them.

* The pure-Python planner restatement (oracle/planner_ref.py) against the
  golden vectors dumped by the compiled reference.
* The C attention oracle (oracle/attention_ref.c) against torch's SDPA with
  the block mask expanded to tokens (fp64), including ragged tails, empty
  rows and the ring-period (kv_allow) merge identity.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from oracle import planner_ref as R
from conftest import f64, fnv_words

SMALL = lambda c: not c["large"] and c["spec"]["heads"] * c["spec"]["q_blocks"] * c["spec"]["kv_blocks"] <= 40 * 64 * 64


def dense_of(case):
    s = case["spec"]
    return R.generate_mask_set(s["heads"], s["q_blocks"], s["kv_blocks"], s["pattern"],
                               s["min_density"], s["max_density"], s["skew"], int(s["seed"]))


def words_of(dense):
    H, nq, nk = dense.shape
    wpr = (nk + 63) // 64
    pad = np.zeros((H, nq, wpr * 64), bool)
    pad[:, :, :nk] = dense
    return np.packbits(pad.reshape(H, nq, wpr, 64), axis=-1, bitorder="little").view(np.uint64).reshape(H, nq, wpr)


def test_python_oracle_generator_and_plans_match_reference(golden):
    checked = 0
    for case in golden["cases"]:
        if not SMALL(case):
            continue
        d = dense_of(case)
        assert fnv_words(words_of(d)) == case["mask"]["fnv"], case["spec"]
        for p in case["plans"]:
            x, y = (int(t) for t in p["strategy"][1:].split("R"))
            rb = math.inf if p["rb"] == "inf" else float(p["rb"])
            plan, rep, pre, post = R.plan_dual(d, x, y, 1.10, rb)
            assert list(plan[0]) == p["plan"]["head"]
            assert list(plan[1]) == p["plan"]["q"]
            assert list(plan[2]) == p["plan"]["kv"]
            assert rep == p["replanned"]
            assert pre == f64(p["rho_pre"]) and post == f64(p["rho_post"])
            assert R.workload_table(d, x, y, plan) == p["post_counts"]
            checked += 1
    assert checked > 100


def test_python_oracle_select_matches_reference(golden):
    pj = golden["profiles"]["node"]
    prof = {"all2all": {int(k): ([f64(v) for v in c["xs"]], [f64(v) for v in c["ys"]])
                        for k, c in pj["all2all"].items()},
            "p2p": {int(k): ([f64(v) for v in c["xs"]], [f64(v) for v in c["ys"]])
                    for k, c in pj["p2p"].items()},
            "dense": f64(pj["dense_attn_seconds"]), "launch": f64(pj["launch_seconds"]),
            "overlap": f64(pj["exchange_overlap"]), "replan": f64(pj["replan_seconds"]),
            "bpt": f64(pj["bytes_per_token_per_head"])}
    for case in golden["cases"]:
        if not SMALL(case) or "error" in case["select"]["node"]:
            continue
        best, _ = R.select(dense_of(case), 8, prof)
        (x, y), plan, _, _, post, lat = best
        ref = case["select"]["node"]
        assert f"U{x}R{y}" == ref["strategy"]
        assert post == f64(ref["rho_post"])
        assert lat["total"] == f64(ref["latency"]["total"])


def sdpa_ref(q, k, v, dense, Sq, Sk):
    # Expand the block mask to tokens; fully-masked rows produce NaN in SDPA,
    # which we map to the oracle's defined O = 0.
    H = q.shape[1]
    tok = np.repeat(np.repeat(dense, 64, axis=1), 64, axis=2)[:, :Sq, :Sk]
    qt = torch.from_numpy(q).double().permute(1, 0, 2)
    kt = torch.from_numpy(k).double().permute(1, 0, 2)
    vt = torch.from_numpy(v).double().permute(1, 0, 2)
    out = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, attn_mask=torch.from_numpy(tok))
    out = torch.nan_to_num(out, nan=0.0)
    return out.permute(1, 0, 2).numpy()


@pytest.mark.parametrize("Sq,Sk,H,d,dens", [(256, 256, 2, 64, 0.5), (200, 330, 3, 32, 0.4),
                                            (128, 64, 1, 16, 1.0)])
def test_attention_oracle_vs_sdpa(Sq, Sk, H, d, dens):
    rng = np.random.default_rng(0)
    nq, nk = -(-Sq // 64), -(-Sk // 64)
    dense = rng.random((H, nq, nk)) < dens
    dense[0, 0, :] = False  # an empty row block
    q = rng.standard_normal((Sq, H, d)).astype(np.float32)
    k = rng.standard_normal((Sk, H, d)).astype(np.float32)
    v = rng.standard_normal((Sk, H, d)).astype(np.float32)
    out, lse = oracle.sparse_attention(q, k, v, words_of(dense), nk)
    ref = sdpa_ref(q, k, v, dense, Sq, Sk)
    assert np.abs(out - ref).max() < 1e-5
    assert np.all(out[:64, 0] == 0) and np.all(np.isinf(lse[0, :64]))


def test_attention_oracle_ring_merge_identity():
    rng = np.random.default_rng(1)
    Sq = Sk = 512
    H, d, nk = 2, 32, 8
    dense = rng.random((H, 8, nk)) < 0.5
    w = words_of(dense)
    q, k, v = (rng.standard_normal((Sq, H, d)).astype(np.float32) for _ in range(3))
    full, full_lse = oracle.sparse_attention(q, k, v, w, nk)
    parts = []
    for g in range(2):
        allow = np.array([sum(1 << b for b in range(nk) if b % 2 == g)], np.uint64)
        parts.append(oracle.sparse_attention(q, k, v, w, nk, kv_allow=allow))
    l0, l1 = parts[0][1], parts[1][1]
    mx = np.maximum(l0, l1)
    with np.errstate(invalid="ignore"):
        w0 = np.where(np.isinf(l0), 0.0, np.exp(l0 - mx))
        w1 = np.where(np.isinf(l1), 0.0, np.exp(l1 - mx))
    den = w0 + w1
    den[den == 0] = 1
    merged = (parts[0][0] * (w0 / den).T[:, :, None] + parts[1][0] * (w1 / den).T[:, :, None])
    assert np.abs(merged - full).max() < 1e-5


def test_attention_oracle_sampled_rows_equal_full():
    rng = np.random.default_rng(2)
    S, H, d = 640, 3, 16
    dense = rng.random((H, 10, 10)) < 0.3
    q, k, v = (rng.standard_normal((S, H, d)).astype(np.float32) for _ in range(3))
    full, _ = oracle.sparse_attention(q, k, v, words_of(dense), 10)
    rows = np.array([(1, 3), (2, 9), (0, 0)], np.int32)
    part, _ = oracle.sparse_attention(q, k, v, words_of(dense), 10, rows=rows)
    for h, b in rows:
        assert np.array_equal(part[b * 64:(b + 1) * 64, h], full[b * 64:(b + 1) * 64, h])
