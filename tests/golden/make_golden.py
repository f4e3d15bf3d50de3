"""Regenerate tests/golden/planner_golden.json from the compiled reference.

Run in the build container (needs /root/reference):
    make -C oracle ref && python tests/golden/make_golden.py
The generator is oracle/ref_tools/golden_dump.cpp compiled against the
unmodified reference headers; this script only runs it and writes the file.
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
OUT = Path(__file__).resolve().parent / "planner_golden.json"


def main() -> int:
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "ref"], check=True)
    tool = ROOT / "oracle" / "_ref" / "golden_dump"
    subprocess.run([str(tool), str(OUT), "/root/reference/proj/profiles/a800x8.json"], check=True)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")
    return 0


if __name__ == "__main__":
    sys.exit(main())
