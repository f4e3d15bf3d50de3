"""Reference unit-test fixtures (proj/tests/test_{metrics,planner,latency,selector}.cpp)
restated against the product planner through the Python face of the C ABI,
plus error-class behaviour (error.hpp) and the C ABI surface itself."""
import ctypes
import json
import math
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2511_23113_b200 as D
from paper_2511_23113_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]


def set_from_weights(weights, capacity=0):
    cap = capacity or max(1, max(weights))
    dense = np.zeros((len(weights), 1, cap), bool)
    for h, w in enumerate(weights):
        dense[h, 0, :w] = True
    return D.AttentionMaskSet.from_dense(dense)


def set_from_row_weights(rows, nk):
    dense = np.zeros((1, len(rows), nk), bool)
    for q, w in enumerate(rows):
        dense[0, q, :w] = True
    return D.AttentionMaskSet.from_dense(dense)


def max_load(w, a, x):
    loads = [0] * x
    for i, wi in enumerate(w):
        loads[a[i]] += wi
    return max(loads)


# ---------------------------------------------------------------- C ABI surface
def test_library_exports_every_declared_symbol():
    header = (ROOT / "include" / "dbsp_b200.h").read_text()
    declared = set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(dbsp_\w+)\s*\(", header, re.M))
    declared = {d for d in declared if not d.endswith("_t")}
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_lib.EXPORTED) <= declared
    assert len(declared) >= 40


def test_version_string():
    assert b"sm_100a" in _lib.lib().dbsp_version()


# ---------------------------------------------------------------- metrics.hpp
def test_strategy_parse_and_enumeration():
    assert str(D.ParallelStrategy(8, 1)) == "U8R1"
    assert D.parse_strategy("U4R2") == D.ParallelStrategy(4, 2)
    assert D.parse_strategy("U1R16") == D.ParallelStrategy(1, 16)
    for bad in ("8x1", "U0R4", "UxRy"):
        with pytest.raises(D.ConfigError):
            D.parse_strategy(bad)
    assert D.enumerate_strategies(8) == [D.ParallelStrategy(8, 1), D.ParallelStrategy(4, 2),
                                         D.ParallelStrategy(2, 4), D.ParallelStrategy(1, 8)]
    assert D.enumerate_strategies(1) == [D.ParallelStrategy(1, 1)]
    for bad in (6, 0):
        with pytest.raises(D.ConfigError):
            D.enumerate_strategies(bad)


def test_default_plan_contiguous():
    s = D.AttentionMaskSet.from_dense(np.ones((4, 4, 6), bool))
    p = D.default_plan(s, D.ParallelStrategy(2, 2))
    assert p.head_assignment.tolist() == [0, 0, 1, 1]
    assert p.q_assignment.tolist() == [0, 0, 1, 1]
    assert p.kv_assignment.tolist() == [0, 0, 0, 1, 1, 1]
    with pytest.raises(D.ConfigError):
        D.default_plan(s, D.ParallelStrategy(8, 1))


def test_ring_schedule_fixture():
    dense = np.zeros((1, 2, 2), bool)
    dense[0, 0, 0] = dense[0, 0, 1] = dense[0, 1, 1] = True
    s = D.AttentionMaskSet.from_dense(dense)
    t = D.workload_table(s, D.ParallelStrategy(1, 2), D.default_plan(s, D.ParallelStrategy(1, 2)))
    assert t.counts.tolist() == [[1, 1], [1, 0]]
    assert abs(D.imbalance_ratio(t) - 4 / 3) < 1e-12
    t1 = D.workload_table(s, D.ParallelStrategy(1, 1), D.default_plan(s, D.ParallelStrategy(1, 1)))
    assert t1.counts.tolist() == [[3]]


def test_rho_fixtures():
    assert D.imbalance_ratio(([[3, 1], [2, 2]], 2)) == 1.25
    assert D.imbalance_ratio(([[4, 0]], 2)) == 2.0
    assert D.imbalance_ratio(([[5, 5], [7, 7]], 2)) == 1.0
    assert D.imbalance_ratio(([[0, 0]], 2)) == 1.0


def test_counts_3122_fixture():
    # proj/tests/fixtures/counts_3122.json: 4 heads, 2x2, popcounts {4,3,1,0};
    # U1R2 gives [[3,1],[2,2]] and rho 1.25.
    rows = [0x03, 0x03, 0x03, 0x01, 0x01, 0x00, 0x00, 0x00]
    words = np.array(rows, np.uint64).reshape(4, 2, 1)
    s = D.AttentionMaskSet(words, 2, 64)
    assert D.blocks_per_head(s) == [4, 3, 1, 0]
    st = D.ParallelStrategy(1, 2)
    t = D.workload_table(s, st, D.default_plan(s, st))
    assert t.counts.tolist() == [[3, 1], [2, 2]]
    assert D.imbalance_ratio(t) == 1.25


def test_plan_contract_errors():
    s = D.AttentionMaskSet.from_dense(np.ones((2, 4, 4), bool))
    bad = D.PartitionPlan.of([0, 2], [0, 0, 0, 0], [0, 0, 0, 0])
    with pytest.raises(D.ContractError):
        D.workload_table(s, D.ParallelStrategy(2, 1), bad)
    short = D.PartitionPlan.of([0], [0, 0, 0, 0], [0, 0, 0, 0])
    with pytest.raises(D.ContractError):
        D.validate_plan(s, D.ParallelStrategy(2, 1), short)


def test_exchange_volume_fixture():
    s = D.AttentionMaskSet.from_dense(np.ones((1, 4, 4), bool))
    p = D.PartitionPlan.of([0], [1, 1, 0, 0], [0, 0, 1, 0])
    e = D.exchange_volume(s, D.ParallelStrategy(1, 2), p)
    assert (e.q_blocks_moved, e.kv_blocks_moved, e.token_payload) == (4, 1, (4 + 2) * 64)


# ---------------------------------------------------------------- planner.hpp
def test_lpt_fixtures():
    s = set_from_weights([7, 5, 3, 1])
    a = D.partition_heads(s, 2)
    assert max_load([7, 5, 3, 1], a, 2) == 8
    assert D.head_level_imbalance([7, 5, 3, 1], a, 2) == 1.0
    assert max_load([7, 5, 3, 1], D.brute_force_heads(s, 2), 2) == 8
    s = set_from_weights([5, 4, 3])
    a = D.partition_heads(s, 2)
    assert max_load([5, 4, 3], a, 2) == 7
    assert abs(D.head_level_imbalance([5, 4, 3], a, 2) - 7 / 6) < 1e-12


def test_lpt_edge_cases():
    s = set_from_weights([3, 2, 1])
    assert D.partition_heads(s, 1).tolist() == [0, 0, 0]
    with pytest.raises(D.ConfigError):
        D.partition_heads(s, 4)
    assert D.partition_heads(set_from_weights([2, 2, 2, 2]), 2).tolist() == [0, 1, 0, 1]
    a = D.partition_heads(set_from_weights([0, 0, 5], 5), 2)
    assert a.tolist() == [1, 1, 0]


def test_block_fixtures_and_rewards():
    s = set_from_row_weights([4, 3, 2, 1], 4)
    qa, _ = D.partition_blocks(s, 2, 0.0)
    assert qa.tolist() == [0, 1, 1, 0]
    qa, _ = D.partition_blocks(s, 2, 10.0)
    assert qa.tolist() == [0, 0, 1, 1]
    qa1, ka1 = D.partition_blocks(s, 1, 0.0)
    assert qa1.tolist() == [0] * 4 and ka1.tolist() == [0] * 4
    with pytest.raises(D.ConfigError):
        D.partition_blocks(s, 5, 0.0)
    with pytest.raises(D.ConfigError):
        D.partition_blocks(s, 2, -1.0)
    with pytest.raises(D.ConfigError):
        D.partition_blocks(s, 2, float("nan"))


def test_infinite_reward_moves_nothing():
    rng = np.random.default_rng(31)
    for _ in range(10):
        s = D.AttentionMaskSet.from_dense(rng.random((3, 8, 12)) < rng.random())
        qa, ka = D.partition_blocks(s, 4, D.kInfiniteReward)
        p = D.PartitionPlan.of([0, 0, 0], qa, ka)
        e = D.exchange_volume(s, D.ParallelStrategy(1, 4), p)
        assert (e.q_blocks_moved, e.kv_blocks_moved, e.token_payload) == (0, 0, 0)


def test_plan_dual_reuse_threshold():
    st = D.ParallelStrategy(2, 1)
    first = set_from_weights([7, 5, 3, 1], 9)
    fresh = D.plan_dual(first, st)
    assert fresh.head_replanned and fresh.rho_post == 1.0
    reused = D.plan_dual(first, st, D.PlannerConfig(), fresh.plan)
    assert not reused.head_replanned and reused.rho_pre == 1.0
    assert reused.plan.head_assignment.tolist() == fresh.plan.head_assignment.tolist()
    prev = D.plan_dual(set_from_weights([9, 1], 9), st)
    rep = D.plan_dual(set_from_weights([1, 9], 9), st, D.PlannerConfig(), prev.plan)
    assert rep.head_replanned
    assert abs(rep.rho_pre - 9 / 5) < 1e-12 and abs(rep.rho_post - 9 / 5) < 1e-12


def test_planner_config_validation():
    s = set_from_weights([1, 2])
    for cfg in (D.PlannerConfig(reuse_threshold=0.9), D.PlannerConfig(exchange_reward=-1.0),
                D.PlannerConfig(exchange_reward=float("nan"))):
        with pytest.raises(D.ConfigError):
            D.plan_dual(s, D.ParallelStrategy(2, 1), cfg)


def test_brute_force_guards():
    s = set_from_weights([1] * 30)
    with pytest.raises(D.SearchSpaceError):
        D.brute_force_heads(s, 2)
    with pytest.raises(D.ConfigError):  # search_space_error is a config_error
        D.brute_force_heads(s, 2)
    g = np.ones(64, np.uint64)
    with pytest.raises(D.SearchSpaceError):
        D.brute_force_blocks(g, 8, 8, 4)
    q, kv, rho = D.brute_force_blocks(np.array([4, 0, 0, 4], np.uint64), 2, 2, 2)
    assert rho == 1.0


def test_generator_validation():
    for kw in (dict(min_density=0.6, max_density=0.5), dict(skew=0.0), dict(max_density=1.5)):
        spec = D.GeneratorSpec(2, 4, 4, 64, "random", **{**dict(min_density=0.1, max_density=0.5), **kw})
        with pytest.raises(D.ConfigError):
            D.generate_mask_set(spec)
    with pytest.raises(D.ConfigError):
        D.generate_mask_set(D.GeneratorSpec(0, 4, 4))
    with pytest.raises(D.ConfigError):
        D.generate_mask_set(D.GeneratorSpec(1, 4, 4, pattern="spiral"))


def test_perturb_laws():
    m = D.generate_mask_set(D.GeneratorSpec(3, 10, 70, 64, "random", 0.3, 0.6, 1.0, 3))
    assert D.perturb_mask_set(m, 0.0, 5) == m
    comp = D.perturb_mask_set(m, 1.0, 5)
    assert np.array_equal(comp.to_dense(), ~m.to_dense())
    twice = D.perturb_mask_set(D.perturb_mask_set(m, 0.3, 9), 0.3, 9)
    assert twice == m  # same substreams flip the same bits: involution
    with pytest.raises(D.ConfigError):
        D.perturb_mask_set(m, 1.5, 1)


# ---------------------------------------------------------------- latency.hpp
def flat_profile(a2a=1e-4, p2p=1e-4):
    c = lambda v: D.PiecewiseLinear([0.0, 1e12], [v, v])
    return D.MachineProfile({2: c(a2a), 4: c(a2a), 8: c(a2a)}, {2: c(p2p), 4: c(p2p), 8: c(p2p)},
                            0.5, 1e-5, 1.0, 0.0, 256.0)


def test_pwl_interpolation():
    c = D.PiecewiseLinear([1.0, 3.0], [10.0, 30.0])
    assert c.eval(1.0) == 10.0 and c.eval(3.0) == 30.0 and c.eval(2.0) == 20.0
    assert c.eval(5.0) == 50.0 and c.eval(-100.0) == 0.0
    inf = D.PiecewiseLinear([0.0, 1.0], [math.inf, math.inf])
    assert inf.eval(0.5) == math.inf
    with pytest.raises(D.ContractError):
        D.PiecewiseLinear([], []).eval(1.0)


def test_fit_errors():
    with pytest.raises(D.ConfigError, match="all2all degree 4"):
        D.fit_profile([D.ProfileSample("all2all", 4, 1.0, 1.0), D.ProfileSample("dense", 1, 0.5, 1.0),
                       D.ProfileSample("dense", 1, 1.0, 2.0)])
    with pytest.raises(D.ConfigError, match="dense"):
        D.fit_profile([D.ProfileSample("dense", 1, 0.5, 1.0)])
    with pytest.raises(D.ConfigError, match="dense"):
        D.fit_profile([D.ProfileSample("dense", 1, 0.5, 2.0), D.ProfileSample("dense", 1, 1.0, 1.0)])


def test_eq4_reductions():
    p = flat_profile()
    shape = D.MaskShape(8, 64, 64, 64)
    u = D.predict_from_inputs(D.CallInputs(shape, D.ParallelStrategy(8, 1), 0.5, 1.0), p)
    assert u.ring_p2p_exposed_s == 0.0 and u.all2all_s > 0
    r = D.predict_from_inputs(D.CallInputs(shape, D.ParallelStrategy(1, 8), 0.5, 1.0), p)
    assert r.all2all_s == 0.0
    r2 = D.predict_from_inputs(D.CallInputs(shape, D.ParallelStrategy(1, 8), 0.5, 1.5), p)
    assert abs(r2.imbalance_penalty_s - 0.5 * (r.attn_compute_s + r.ring_p2p_exposed_s)) < 1e-15
    with pytest.raises(D.ContractError):
        D.predict_from_inputs(D.CallInputs(shape, D.ParallelStrategy(1, 8), 0.5, 0.9), p)
    with pytest.raises(D.ConfigError, match="p2p degree 8"):
        q = flat_profile()
        q.p2p.pop(8)
        D.predict_from_inputs(D.CallInputs(shape, D.ParallelStrategy(1, 8), 0.5, 1.0), q)


def test_profile_json_roundtrip():
    p = flat_profile()
    q = D.MachineProfile.from_json(p.to_json())
    assert q.all2all[2].xs == p.all2all[2].xs and q.p2p[8].ys == p.p2p[8].ys
    assert abs(q.dense_attn_seconds - p.dense_attn_seconds) < 1e-15


# ---------------------------------------------------------------- selector.hpp
def test_selector_ties_and_state():
    m = D.generate_mask_set(D.GeneratorSpec(8, 16, 16, 64, "random", 0.5, 0.5, 1.0, 3))
    p = flat_profile()
    p.dense_attn_seconds = 0.0
    p.launch_seconds = 0.0
    for c in list(p.all2all.values()) + list(p.p2p.values()):
        c.ys = [0.0, 0.0]
    # all-zero costs: every strategy ties at 0 -> largest Ulysses degree wins
    st = D.SelectorState(8)
    sel = D.select(3, m, p, D.PlannerConfig(), st)
    assert sel.strategy == D.ParallelStrategy(8, 1)
    got = st.stored(3)
    assert got is not None and got[0] == sel.strategy
    assert st.stored(4) is None
    inf = flat_profile(p2p=math.inf)
    assert D.select(0, m, inf, D.PlannerConfig(), D.SelectorState(8)).strategy == D.ParallelStrategy(8, 1)


def test_selector_feasibility():
    # x <= heads and y <= min(Nq, Nk) (latency.hpp:301-302): only U4R2 fits 4 heads x 2x2.
    m = D.generate_mask_set(D.GeneratorSpec(4, 2, 2, 64, "random", 0.5, 0.5, 1.0, 3))
    preds = D.predict_all(m, flat_profile(), 8)
    assert [str(p.strategy) for p in preds] == ["U4R2"]


def test_selector_no_feasible_strategy():
    m = D.generate_mask_set(D.GeneratorSpec(1, 1, 1, 64, "random", 0.5, 0.5, 1.0, 3))
    with pytest.raises(D.ConfigError, match="no feasible strategy"):
        D.predict_all(m, flat_profile(), 8)


def _same_selection(a, b):
    assert (a.strategy.ulysses, a.strategy.ring) == (b.strategy.ulysses, b.strategy.ring)
    for x, y in ((a.outcome.plan.head_assignment, b.outcome.plan.head_assignment),
                 (a.outcome.plan.q_assignment, b.outcome.plan.q_assignment),
                 (a.outcome.plan.kv_assignment, b.outcome.plan.kv_assignment)):
        assert np.array_equal(x, y)
    assert a.outcome.head_replanned == b.outcome.head_replanned
    # doubles compared exactly (selector.hpp:67-69 argmin on exact totals)
    assert a.outcome.rho_pre == b.outcome.rho_pre and a.outcome.rho_post == b.outcome.rho_post
    assert a.latency == b.latency


@pytest.mark.parametrize("shape", [(8, 64, 64, "random", 0.5, 0.5), (40, 512, 512, "clustered", 0.15, 0.45),
                                   (48, 278, 278, "clustered", 0.15, 0.484), (12, 100, 37, "banded", 0.2, 0.7)])
def test_two_phase_select_equals_select(shape):
    # The planning code of the device selector (assignments first, then one
    # batch of workload tables) reproduces select() bit for bit, including
    # the P_s head-plan reuse across a perturbed chain of calls.
    H, nq, nk, pat, lo, hi = shape
    prof = D.MachineProfile.from_json(json.loads(
        (ROOT / "paper_2511_23113_b200" / "profiles" / "b200_wan_measured.json").read_text()))
    m = D.generate_mask_set(D.GeneratorSpec(H, nq, nk, 64, pat, lo, hi, 1.0, 3))
    for gpus in (2, 4, 8):
        s_host, s_two = D.SelectorState(gpus), D.SelectorState(gpus)
        cur = m
        for step in range(4):
            if step:
                cur = D.perturb_mask_set(cur, 0.02, D.mix_seed(3, gpus, step))
            for layer in (0, 1):
                _same_selection(D.select(layer, cur, prof, D.PlannerConfig(), s_host),
                                D.select_two_phase(layer, cur, prof, D.PlannerConfig(), s_two))


def test_new_entry_points_validate_before_touching_the_gpu():
    # The C ABI of the GPU paths checks its arguments on the host and fails
    # with the reference's error classes (error.hpp:10-44) before any CUDA call.
    L = _lib.lib()
    C = ctypes
    # K6: head_dim 96, then 3*H*d not a multiple of 256, then a null input
    a = _lib.QkvArgsT(1, 1, None, 1, 128, 512, 4, 96)
    assert L.dbsp_qkv_project(C.byref(a), None, None) == 2
    a = _lib.QkvArgsT(1, 1, None, 1, 128, 512, 1, 64)
    assert L.dbsp_qkv_project(C.byref(a), None, None) == 2
    a = _lib.QkvArgsT(None, 1, None, 1, 128, 512, 4, 64)
    assert L.dbsp_qkv_project(C.byref(a), None, None) == 4
    # the fused scatter needs whole 64-token blocks and a complete table set
    a = _lib.QkvArgsT(1, 1, None, None, 100, 512, 4, 64)
    sc = _lib.QkvScatterT(1, 1, 1, 1, 1, 1, 1)
    assert L.dbsp_qkv_project(C.byref(a), C.byref(sc), None) == 4
    # GPU selector: null words / zero dims
    st = D.SelectorState(4)
    prof = D.MachineProfile.from_json(json.loads(
        (ROOT / "paper_2511_23113_b200" / "profiles" / "b200_nominal.json").read_text()))
    out = [_lib.StrategyT(), None, _lib.PlanOutcomeT(), _lib.LatencyT()]
    rc = L.dbsp_select_device(st._h, 0, None, 4, 8, 8, 64, C.byref(prof.c()), C.byref(D.PlannerConfig().c()),
                              C.byref(out[0]), None, C.byref(out[2]), C.byref(out[3]), None)
    assert rc == 4
    rc = L.dbsp_select_device(st._h, 0, C.c_void_p(8), 4, 0, 8, 64, C.byref(prof.c()),
                              C.byref(D.PlannerConfig().c()), C.byref(out[0]), None, C.byref(out[2]),
                              C.byref(out[3]), None)
    assert rc == 2
    # C++ SP call: strategy / rank-count mismatch and bad plans, before any NCCL or CUDA work
    m = D.generate_mask_set(D.GeneratorSpec(4, 8, 8, 64, "random", 0.5, 0.5, 1.0, 1))
    plan = D.default_plan(m, D.ParallelStrategy(2, 2))
    ptrs = (C.c_void_p * 4)(1, 1, 1, 1)
    rc = L.dbsp_sp_attention_simulated(C.byref(m.c()), _lib.StrategyT(2, 2), C.byref(plan.c()), ptrs, ptrs, ptrs,
                                       ptrs, 8 * 64, 96, None)
    assert rc == 2  # head_dim
    rc = L.dbsp_sp_attention_simulated(C.byref(m.c()), _lib.StrategyT(2, 2), C.byref(plan.c()), ptrs, ptrs, ptrs,
                                       ptrs, 8 * 64 - 1, 64, None)
    assert rc == 4  # tokens must be whole blocks
    bad = D.PartitionPlan.of([0, 0, 1, 3], plan.q_assignment, plan.kv_assignment)
    rc = L.dbsp_sp_attention_simulated(C.byref(m.c()), _lib.StrategyT(2, 2), C.byref(bad.c()), ptrs, ptrs, ptrs,
                                       ptrs, 8 * 64, 64, None)
    assert rc == 4  # head assigned past x
    # fused O return: incomplete scatter tables
    sc2 = _lib.OutScatterT(None, 1, 1, 4)
    sched = C.c_void_p()
    assert L.dbsp_schedule_create(C.byref(sched)) == 0
    args = _lib.AttnArgsT(1, 1, 1, None, None, None, None, 64, 64, 4, 64, 0.0, 0, 0)
    assert L.dbsp_attention_launch_scatter(sched, C.byref(args), C.byref(sc2), None) == 4
    L.dbsp_schedule_destroy(sched)


def test_auto_d128_schedule_choice():
    # DBSP_SCHED_AUTO_D128 (schedule.hpp): the measured-fastest d=128 layout,
    # which since round 2 is the pair schedule (2 Q blocks per item) on every
    # mask family; the CTA-pair quad schedule stays available explicitly.
    from paper_2511_23113_b200.attention import AttentionSchedule
    H, nb = 2, 512
    for pattern in ("clustered", "banded", "random"):
        m = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, pattern, 0.15, 0.45, 1.0, 1))
        auto = AttentionSchedule().build(m, head_dim=128)
        assert auto.stats() == AttentionSchedule().build(m, flags=1).stats(), pattern
        assert auto.stats()["items"] == H * (nb // 2), pattern
        assert auto.layout()["q_blocks_per_item"] == 2
        quad = AttentionSchedule().build(m, flags=1 | 8 | 16 | 128)
        assert quad.layout()["q_blocks_per_item"] == 4 and quad.stats()["items"] == H * (nb // 4)
        assert AttentionSchedule().build(m, head_dim=64).stats()["items"] == H * (nb // 2)


@pytest.mark.parametrize("H,nb,group", [(16, 278, 7), (6, 278, 0), (9, 512, 4), (5, 512, 0), (3, 1857, 1), (4, 64, 0)])
def test_launch_order_lpt_within_l2_sized_head_groups(H, nb, group):
    # schedule.hpp lpt_head_group: heads in groups of max(1, 2048 / KV blocks)
    # (0 = a single group: global LPT, also for views of <= 4096 head x KV
    # blocks), heaviest item first within a group,
    # groups in head order.  Explicit GLOBAL_LPT / HEAD_ORDER override it.
    from paper_2511_23113_b200.attention import AttentionSchedule
    m = D.generate_mask_set(D.GeneratorSpec(H, nb, nb, 64, "clustered", 0.15, 0.45, 1.0, 3))

    def order(flags):
        items, _ = AttentionSchedule().build(m, flags=flags).download()
        return items[:, 0].astype(np.int64), items[:, 4].astype(np.int64)  # head, count

    def check_groups(heads, counts, g):
        key = heads // g if g else np.zeros_like(heads)
        assert np.all(np.diff(key) >= 0), "groups out of head order"
        for k in np.unique(key):
            c = counts[key == k]
            assert np.all(np.diff(c) <= 0), "not heaviest-first within a group"

    heads, counts = order(1)
    g = 2048 // nb
    assert (0 if (H * nb <= 4096 or g >= H) else max(g, 1)) == group
    check_groups(heads, counts, group)
    check_groups(*order(1 | 2), 0)  # GLOBAL_LPT
    check_groups(*order(1 | 4), 1)  # HEAD_ORDER
