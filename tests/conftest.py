import json
import struct
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200, sm_100a) device")
    config.addinivalue_line("markers", "slow: longer-running CPU test")


@pytest.fixture(scope="session", autouse=True)
def _built_library():
    """Build libdbsp_b200.so (and the C oracle) once per session if missing."""
    from paper_2511_23113_b200 import build as b
    if not b.LIB.exists():
        b.build()
    import oracle
    if not oracle.ATTN_LIB.exists():
        oracle.build(reference=False)


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN / "planner_golden.json") as f:
        return json.load(f)


def f64(bits: str) -> float:
    return struct.unpack("<d", struct.pack("<Q", int(bits)))[0]


def bits_of(x: float) -> str:
    return str(struct.unpack("<Q", struct.pack("<d", x))[0])


def profile_from_bits(j):
    from paper_2511_23113_b200 import MachineProfile, PiecewiseLinear
    cur = lambda t: {int(d): PiecewiseLinear([f64(v) for v in c["xs"]], [f64(v) for v in c["ys"]])
                     for d, c in t.items()}
    return MachineProfile(cur(j["all2all"]), cur(j["p2p"]), f64(j["dense_attn_seconds"]),
                          f64(j["launch_seconds"]), f64(j["exchange_overlap"]),
                          f64(j["replan_seconds"]), f64(j["bytes_per_token_per_head"]))


def spec_of(j):
    from paper_2511_23113_b200 import GeneratorSpec
    return GeneratorSpec(j["heads"], j["q_blocks"], j["kv_blocks"], j["block_size"], j["pattern"],
                         j["min_density"], j["max_density"], j["skew"], int(j["seed"]))


def fnv_words(words: np.ndarray) -> str:
    import oracle
    return oracle.fnv1a(np.ascontiguousarray(words, np.uint64))


def cuda_ok() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
