"""The reference's own acceptance suite (proj/tests/acceptance.cpp), compiled
UNCHANGED against this repo's C++ faces (include/dbsp/*.hpp over
libdbsp_b200.so).

Only the two headers that are out of scope here -- the analytic simulator
(simulator.hpp) and its thread pool (parallel.hpp), SURVEY.md §2 -- resolve
from the reference tree, which comes AFTER include/ on the search path, so
every dbsp header the suite and the simulator include (mask, mask_io,
metrics, planner, latency, selector, error, rng) is ours.  Criteria 1-11 must
PASS with detail strings equal to the reference's recorded run
(proj/test_output.txt:11-21).  Criterion 12 drives the reference CLI
(tools/dbsp.cpp, unbuildable: CLI11 is absent) and is not asserted.

Runs where the reference tree is present (this build container); the GPU box
has no /root/reference and skips it.
"""
import re
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/proj")
JSON_INC = Path("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann")

pytestmark = pytest.mark.skipif(
    not (REF / "tests" / "acceptance.cpp").exists() or not JSON_INC.exists() or shutil.which("g++") is None,
    reason="needs the reference tree, nlohmann/json and g++ (build container only)")

LINE = re.compile(r"^\[(PASS|FAIL)\] criterion\s+(\d+): (.*?) \| (.*) \(\d+ ms\)$")


def parse(text):
    out = {}
    for line in text.splitlines():
        m = LINE.match(line.strip())
        if m:
            out[int(m.group(2))] = (m.group(1), m.group(3), m.group(4))
    return out


def test_reference_acceptance_criteria_1_to_11(tmp_path):
    lib_dir = ROOT / "paper_2511_23113_b200"
    exe = tmp_path / "acceptance"
    cmd = ["g++", "-std=c++20", "-O1", "-pthread",
           f"-I{ROOT / 'include'}",        # ours first: every dbsp header the suite includes
           f"-I{REF / 'include'}",         # then only simulator.hpp / parallel.hpp resolve here
           f"-I{JSON_INC}", '-DDBSP_CLI_PATH="/nonexistent"',
           str(REF / "tests" / "acceptance.cpp"),
           f"-L{lib_dir}", "-ldbsp_b200", f"-Wl,-rpath,{lib_dir}", "-o", str(exe),
           "-H"]  # header trace on stderr: which file each include resolved to
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    used = [ln.lstrip(". ").strip() for ln in r.stderr.splitlines() if ln.startswith(".")]
    ours = {Path(p).name for p in used if Path(p).resolve().is_relative_to(ROOT / "include")}
    theirs = {Path(p).name for p in used if Path(p).resolve().is_relative_to(REF / "include")}
    for h in ("mask.hpp", "mask_io.hpp", "metrics.hpp", "planner.hpp", "latency.hpp", "selector.hpp",
              "error.hpp", "rng.hpp"):
        assert h in ours and h not in theirs, f"{h} did not resolve to include/dbsp"
    assert theirs <= {"simulator.hpp", "parallel.hpp"}, theirs

    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600, cwd=tmp_path)
    got = parse(run.stdout)
    want = parse((REF / "test_output.txt").read_text())
    for c in range(1, 12):
        assert c in got, run.stdout
        assert got[c][0] == "PASS", f"criterion {c}: {got[c]}"
        assert got[c][1:] == want[c][1:], f"criterion {c}: {got[c][2]!r} != reference {want[c][2]!r}"
