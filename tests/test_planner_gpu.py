"""GPU selector (dbsp_select_device): K1 marginals and the batched
workload-table kernel feed the same planning code as the host select(), so
every plan, rho and latency double must match it exactly (selector.hpp:55-75,
metrics.hpp:133-168)."""
import json
import time
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2511_23113_b200 as D

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _same(a, b):
    assert (a.strategy.ulysses, a.strategy.ring) == (b.strategy.ulysses, b.strategy.ring)
    assert np.array_equal(a.outcome.plan.head_assignment, b.outcome.plan.head_assignment)
    assert np.array_equal(a.outcome.plan.q_assignment, b.outcome.plan.q_assignment)
    assert np.array_equal(a.outcome.plan.kv_assignment, b.outcome.plan.kv_assignment)
    assert a.outcome.head_replanned == b.outcome.head_replanned
    assert a.outcome.rho_pre == b.outcome.rho_pre and a.outcome.rho_post == b.outcome.rho_post
    assert a.latency == b.latency


def _words(m):
    return torch.from_numpy(np.ascontiguousarray(m.words).view(np.int64)).cuda()


@pytest.mark.parametrize("shape", [(8, 64, 64, "random", 0.5, 0.5), (40, 512, 512, "clustered", 0.15, 0.45),
                                   (48, 278, 278, "clustered", 0.15, 0.484), (24, 1857, 1857, "clustered", 0.15, 0.45),
                                   (12, 100, 37, "banded", 0.2, 0.7)])
def test_select_device_equals_host(shape):
    H, nq, nk, pat, lo, hi = shape
    prof = D.MachineProfile.from_json(json.loads(
        (ROOT / "paper_2511_23113_b200" / "profiles" / "b200_wan_measured.json").read_text()))
    m = D.generate_mask_set(D.GeneratorSpec(H, nq, nk, 64, pat, lo, hi, 1.0, 5))
    for gpus in (2, 8):
        s_host, s_dev = D.SelectorState(gpus), D.SelectorState(gpus)
        cur = m
        for step in range(3):
            if step:
                cur = D.perturb_mask_set(cur, 0.02, D.mix_seed(5, gpus, step))
            w = _words(cur)
            for layer in (0, 1):
                _same(D.select(layer, cur, prof, D.PlannerConfig(), s_host),
                      D.select_device(layer, w, nk, prof, D.PlannerConfig(), s_dev))


def test_select_device_timing_wan():
    # Report only (the bench carries the number): per-call time of the GPU
    # selector on the Wan masks, G=8, against the host selector.
    prof = D.MachineProfile.from_json(json.loads(
        (ROOT / "paper_2511_23113_b200" / "profiles" / "b200_wan_measured.json").read_text()))
    m = D.generate_mask_set(D.GeneratorSpec(40, 512, 512, 64, "clustered", 0.15, 0.45, 1.0, 1))
    w = _words(m)
    st = D.SelectorState(8)
    for _ in range(3):
        D.select_device(0, w, 512, prof, D.PlannerConfig(), st)
    t0 = time.perf_counter()
    for _ in range(20):
        D.select_device(0, w, 512, prof, D.PlannerConfig(), st)
    dev_ms = (time.perf_counter() - t0) / 20 * 1e3
    t0 = time.perf_counter()
    for _ in range(5):
        D.select(0, m, prof, D.PlannerConfig(), D.SelectorState(8))
    host_ms = (time.perf_counter() - t0) / 5 * 1e3
    print(f"select_device {dev_ms:.3f} ms/call, host select {host_ms:.3f} ms/call")
    assert dev_ms < host_ms
