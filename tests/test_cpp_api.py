"""The C++ drop-in API (include/dbsp/*.hpp over libdbsp_b200.so) compiles with
plain g++ and passes the reference-acceptance-style checks in
tests/cpp/api_test.cpp."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
JSON_INC = Path("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann")


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_cpp_api_compiles_links_and_passes(tmp_path):
    lib_dir = ROOT / "paper_2511_23113_b200"
    exe = tmp_path / "api_test"
    cmd = ["g++", "-std=c++20", "-O1", f"-I{ROOT / 'include'}", str(ROOT / "tests" / "cpp" / "api_test.cpp"),
           f"-L{lib_dir}", "-ldbsp_b200", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)]
    if JSON_INC.exists():
        cmd.insert(3, f"-I{JSON_INC}")
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failure(s)" in out.stdout
    assert out.stdout.count("[PASS]") >= 9


@pytest.mark.gpu
@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_cpp_gpu_faces(tmp_path):
    # tests/cpp/gpu_api_test.cpp: dbsp::select_device vs dbsp::select, and
    # dbsp::sparse_attention and the CTA-pair kernel (C ABI, DBSP_SCHED_CTA_PAIR) vs a
    # CPU reference, from plain C++.
    lib_dir = ROOT / "paper_2511_23113_b200"
    exe = tmp_path / "gpu_api_test"
    prof = ROOT / "paper_2511_23113_b200" / "profiles" / "b200_wan_measured.json"
    cmd = ["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", "-I/usr/local/cuda/include",
           f'-DDBSP_PROFILE_JSON="{prof}"', str(ROOT / "tests" / "cpp" / "gpu_api_test.cpp"),
           f"-L{lib_dir}", "-ldbsp_b200", f"-Wl,-rpath,{lib_dir}", "-L/usr/local/cuda/lib64", "-lcudart",
           "-o", str(exe)]
    if JSON_INC.exists():
        cmd.insert(3, f"-I{JSON_INC}")
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failure(s)" in out.stdout
