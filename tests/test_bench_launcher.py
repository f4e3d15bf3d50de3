"""bench.py's driver contract on a machine without GPUs: the N>1 launcher
(`bench.py --gpus N` re-runs itself under torch.distributed.run), the
world-size checks, the per-split loop and the one-line JSON of the N>1 leg
(--dry-run: gloo on CPU, the Python executor with no attention compute), and
the reference arm's independence from the product library."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def _run(args, env=None, timeout=600):
    e = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                            "MASTER_PORT")}
    e.update(env or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py")] + args, capture_output=True, text=True,
                          timeout=timeout, env=e, cwd=str(ROOT))


def _line(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out[-3000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("gpus", [2, 4])
def test_gpus_n_self_launches_ranks(gpus):
    r = _run(["--gpus", str(gpus), "--dry-run", "--workload", "toy", "--steps", "1", "--warmup", "3"])
    assert r.returncode == 0, r.stderr[-3000:]
    j = _line(r.stdout)
    from bench import bench_config
    from paper_2511_23113_b200.workloads import WORKLOADS
    import paper_2511_23113_b200 as D
    assert j["n_gpus"] == gpus and j["dry_run"] is True
    assert j["config"] == bench_config(WORKLOADS["toy"], gpus)
    want = {f"{s}/{b}" for s in D.enumerate_strategies(gpus) for b in ("uniform", "dbsp")}
    assert set(j["splits"]) == want
    assert j["planning"]["ranks_agree"] is True
    for v in j["splits"].values():
        assert len(v["kernel_ms_per_period_per_rank"][0]) == gpus  # one column per rank
    assert j["best_uniform"]["split"].endswith("/uniform") and j["best_dbsp"]["split"].endswith("/dbsp")


def test_world_size_mismatch_fails_loudly():
    r = _run(["--gpus", "2", "--dry-run", "--workload", "toy"], env={"WORLD_SIZE": "3", "RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE=3" in r.stderr


def test_more_gpus_than_present_fails_loudly():
    import torch
    n = torch.cuda.device_count()
    r = _run(["--gpus", str(n + 2), "--workload", "toy", "--no-cpu-baseline"])
    assert r.returncode == 2 and f"needs {n + 2} GPUs" in r.stderr


def test_reference_arm_shares_config_and_never_loads_the_product():
    r = _run(["--impl", "reference", "--workload", "toy", "--steps", "1", "--warmup", "3", "--ref-budget", "0.2"])
    assert r.returncode == 0, r.stderr[-3000:]
    j = _line(r.stdout)
    from bench import bench_config
    from paper_2511_23113_b200.workloads import WORKLOADS
    assert j["impl"] == "reference" and j["config"] == bench_config(WORKLOADS["toy"], 1)
    assert not any("libdbsp_b200" in p for p in j["native_so_loaded"]), j["native_so_loaded"]
    assert j["value"] == j["ms_per_step"] == j["cpu_baseline"]["value"] == j["e2e"]["value"]
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["extrapolated_full_layer_ms"] >= j["value"] * 0.9


def test_reference_arm_under_torchrun_prints_on_rank0_only():
    r = _run(["--impl", "reference", "--gpus", "2", "--workload", "toy", "--steps", "1", "--warmup", "3",
              "--ref-budget", "0.2"])
    assert r.returncode == 0, r.stderr[-3000:]
    j = _line(r.stdout)  # exactly one line
    assert j["n_gpus"] == 2 and "reference_planner" in j
    assert j["value"] >= j["reference_planner"]["select_ms"]  # not divided by N


def test_measure_comm_dry_run(tmp_path):
    # tests/measure_comm.py (the NCCL all-to-all / ring-step sweep of the B200
    # MachineProfile) end to end on gloo: self-launch, groups per degree,
    # fit_profile, a profile JSON the selector loads.
    out = tmp_path / "prof.json"
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "measure_comm.py"), "--gpus", "4", "--dry-run",
                        "--out", str(out)], capture_output=True, text=True, timeout=600, cwd=str(ROOT),
                       env={k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE")})
    assert r.returncode == 0, r.stderr[-3000:]
    j = json.loads(out.read_text())
    assert j["comm_source"] == "dry-run" and {e["degree"] for e in j["all2all"]} == {2, 4}
    import paper_2511_23113_b200 as D
    prof = D.MachineProfile.from_json(j)
    assert prof.all2all_at(4, 1 << 20) > 0 and prof.p2p_at(2, 1 << 20) > 0
