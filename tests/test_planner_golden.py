"""Bit-exact parity of the product planner (C++ in libdbsp_b200.so, via the C
ABI) against golden vectors dumped by the compiled reference
(oracle/ref_tools/golden_dump.cpp -> tests/golden/planner_golden.json).

Assignments must match exactly and every double must match to the bit.
"""
import math

import numpy as np
import pytest

import paper_2511_23113_b200 as D
from conftest import bits_of, f64, fnv_words, profile_from_bits, spec_of

CACHE = {}


def mask_of(case):
    key = tuple(sorted((k, str(v)) for k, v in case["spec"].items()))
    if key not in CACHE:
        CACHE[key] = D.generate_mask_set(spec_of(case["spec"]))
    return CACHE[key]


def rb_of(s):
    return math.inf if s == "inf" else float(s)


def lat_bits(l: D.LatencyBreakdown):
    return {"all2all": bits_of(l.all2all_s), "compute": bits_of(l.attn_compute_s),
            "exposed": bits_of(l.ring_p2p_exposed_s), "imbalance": bits_of(l.imbalance_penalty_s),
            "exchange": bits_of(l.exchange_s), "replan": bits_of(l.replan_s),
            "total": bits_of(l.total_s)}


def test_generator_matches_reference(golden):
    for case in golden["cases"]:
        m = mask_of(case)
        g = case["mask"]
        assert fnv_words(m.words) == g["fnv"], case["spec"]
        assert D.blocks_per_head(m) == g["head_counts"]
        assert D.total_blocks(m) == g["total"]
        assert bits_of(D.density(m)) == g["density_bits"]
        if "words" in g:
            assert [str(int(w)) for w in m.words.reshape(-1)] == g["words"]


def test_summed_grid(golden):
    for case in golden["cases"]:
        if "summed_grid" in case:
            assert D.summed_grid(mask_of(case)).tolist() == case["summed_grid"]


def test_plan_dual_workload_exchange_latency(golden):
    node = profile_from_bits(golden["profiles"]["node"])
    n = 0
    for case in golden["cases"]:
        m = mask_of(case)
        for p in case["plans"]:
            s = D.parse_strategy(p["strategy"])
            cfg = D.PlannerConfig(exchange_reward=rb_of(p["rb"]))
            oc = D.plan_dual(m, s, cfg)
            assert oc.plan.head_assignment.tolist() == p["plan"]["head"], (case["spec"], p["strategy"])
            assert oc.plan.q_assignment.tolist() == p["plan"]["q"], (case["spec"], p["strategy"], p["rb"])
            assert oc.plan.kv_assignment.tolist() == p["plan"]["kv"]
            assert oc.head_replanned == p["replanned"]
            assert bits_of(oc.rho_pre) == p["rho_pre"]
            assert bits_of(oc.rho_post) == p["rho_post"]
            assert D.workload_table(m, s, oc.plan).counts.tolist() == p["post_counts"]
            assert D.workload_table(m, s, D.default_plan(m, s)).counts.tolist() == p["default_counts"]
            ev = D.exchange_volume(m, s, oc.plan)
            assert [ev.q_blocks_moved, ev.kv_blocks_moved, ev.token_payload] == p["exchange"]
            assert lat_bits(D.predict_latency(m, s, oc.plan, node)) == p["latency_node"]
            n += 1
    assert n > 300


def test_select_matches_reference(golden):
    profiles = {k: profile_from_bits(v) for k, v in golden["profiles"].items()}
    for case in golden["cases"]:
        m = mask_of(case)
        for name, ref in case["select"].items():
            st = D.SelectorState(8)
            if "error" in ref:
                with pytest.raises(D.DbspError):
                    D.select(0, m, profiles[name], D.PlannerConfig(), st)
                continue
            sel = D.select(0, m, profiles[name], D.PlannerConfig(), st)
            assert str(sel.strategy) == ref["strategy"], (case["spec"], name)
            assert sel.outcome.plan.head_assignment.tolist() == ref["plan"]["head"]
            assert sel.outcome.plan.q_assignment.tolist() == ref["plan"]["q"]
            assert sel.outcome.plan.kv_assignment.tolist() == ref["plan"]["kv"]
            assert bits_of(sel.outcome.rho_post) == ref["rho_post"]
            assert lat_bits(sel.latency) == ref["latency"]


def test_reuse_chains_and_dynamic_selection(golden):
    a800 = profile_from_bits(golden["profiles"]["a800"])
    for ch in golden["chains"]:
        base = spec_of(ch["spec"])
        # ScheduleMasks chain (simulator.hpp:53-113): per-layer seeds, per-step flips.
        cur = []
        for layer in range(ch["layers"]):
            sp = spec_of(ch["spec"])
            sp.seed = D.mix_seed(base.seed, layer)
            cur.append(D.generate_mask_set(sp))
        masks = {}
        for step in range(ch["steps"]):
            for layer in range(ch["layers"]):
                if step > 0:
                    cur[layer] = D.perturb_mask_set(cur[layer], ch["flip"],
                                                    D.mix_seed(base.seed, layer, step))
                masks[(step, layer)] = cur[layer]
        prev = {}
        for rec in ch["plans"]:
            s = D.parse_strategy(rec["strategy"])
            m = masks[(rec["step"], rec["layer"])]
            assert fnv_words(m.words) == rec["mask_fnv"]
            key = (rec["strategy"], rec["layer"])
            oc = D.plan_dual(m, s, D.PlannerConfig(), prev.get(key) if rec["step"] > 0 else None)
            assert oc.head_replanned == rec["replanned"], rec
            assert oc.plan.head_assignment.tolist() == rec["plan"]["head"]
            assert oc.plan.q_assignment.tolist() == rec["plan"]["q"]
            assert bits_of(oc.rho_pre) == rec["rho_pre"]
            assert bits_of(oc.rho_post) == rec["rho_post"]
            prev[key] = oc.plan
        st = D.SelectorState(8)
        for rec in ch["dynamic"]:
            sel = D.select(rec["layer"], masks[(rec["step"], rec["layer"])], a800, D.PlannerConfig(), st)
            assert str(sel.strategy) == rec["strategy"], rec
            assert sel.outcome.head_replanned == rec["replanned"]
            assert bits_of(sel.outcome.rho_post) == rec["rho_post"]
            assert bits_of(sel.latency.total_s) == rec["total"]
            assert sel.outcome.plan.head_assignment.tolist() == rec["plan"]["head"]


def test_predict_from_inputs(golden):
    node = profile_from_bits(golden["profiles"]["node"])
    for r in golden["predict_from_inputs"]:
        ci = D.CallInputs(D.MaskShape(r["heads"], r["q_blocks"], r["kv_blocks"], r["block_size"]),
                          D.ParallelStrategy(r["x"], r["y"]), f64(r["density"]), f64(r["rho"]),
                          D.ExchangeVolume(*r["exchange"]), r["charge_replan"])
        if "error" in r["latency"]:
            with pytest.raises(D.ConfigError, match="all2all degree"):
                D.predict_from_inputs(ci, node)
        else:
            assert lat_bits(D.predict_from_inputs(ci, node)) == r["latency"]


def test_fit_profile(golden):
    samples = [D.ProfileSample("all2all", 8, 1048576, 0.001), D.ProfileSample("all2all", 8, 2097152, 0.002),
               D.ProfileSample("all2all", 2, 1048576, 0.0006), D.ProfileSample("all2all", 2, 2097152, 0.0011),
               D.ProfileSample("p2p", 8, 1048576, 0.0008), D.ProfileSample("p2p", 8, 2097152, 0.0016),
               D.ProfileSample("p2p", 2, 1048576, 0.0005), D.ProfileSample("p2p", 2, 2097152, 0.0009),
               D.ProfileSample("dense", 1, 0.5, 0.0055), D.ProfileSample("dense", 1, 1.0, 0.010),
               D.ProfileSample("dense", 1, 0.25, 0.0031), D.ProfileSample("dense", 1, 0.25, 0.0029)]
    p = D.fit_profile(samples, D.FitOptions(0.9, 1e-4, 128.0))
    assert bits_of(p.dense_attn_seconds) == golden["fit"]["dense_attn_seconds"]
    assert bits_of(p.launch_seconds) == golden["fit"]["launch_seconds"]
    ref = profile_from_bits(golden["fit"]["profile"])
    for d, c in ref.all2all.items():
        assert [bits_of(v) for v in p.all2all[d].xs] == [bits_of(v) for v in c.xs]
        assert [bits_of(v) for v in p.all2all[d].ys] == [bits_of(v) for v in c.ys]
