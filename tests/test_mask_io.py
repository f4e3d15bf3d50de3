"""DBSPMSK1 mask files: byte-identical with files written by the compiled
reference (tests/golden/ref_*.mask from oracle/ref_tools/golden_dump.cpp),
round trips, the JSON hex sidecar and the reference's error messages
(proj/tests/test_mask.cpp:170-233)."""
import json
import struct

import numpy as np
import pytest

import paper_2511_23113_b200 as D
from conftest import GOLDEN


@pytest.mark.parametrize("name,spec", [
    ("ref_toyA.mask", D.GeneratorSpec(8, 64, 64, 64, "random", 0.5, 0.5, 1.0, 1)),
    ("ref_5x9x70.mask", D.GeneratorSpec(5, 9, 70, 64, "random", 0.2, 0.7, 1.0, 5)),
])
def test_reference_files_load_and_save_byte_identical(tmp_path, name, spec):
    m = D.generate_mask_set(spec)
    ref = GOLDEN / name
    assert D.load_mask_set(ref) == m
    out = tmp_path / "ours.mask"
    D.save_mask_set(m, out)
    assert out.read_bytes() == ref.read_bytes()


def test_round_trip_many(tmp_path):
    for seed in range(20):
        m = D.generate_mask_set(D.GeneratorSpec(1 + seed % 5, 1 + seed, 1 + 7 * seed, 64,
                                                ["random", "banded", "clustered"][seed % 3], 0.1, 0.9,
                                                1.0, seed))
        p = tmp_path / f"m{seed}.mask"
        D.save_mask_set(m, p)
        assert D.load_mask_set(p) == m
        assert not (tmp_path / f"m{seed}.mask.tmp").exists()  # atomic write leaves no temp


def test_errors(tmp_path):
    bad = tmp_path / "bad.mask"
    bad.write_bytes(b"NOTAMASK" + b"\0" * 40)
    with pytest.raises(D.ParseError, match="bad magic at byte 0"):
        D.load_mask_set(bad)
    m = D.generate_mask_set(D.GeneratorSpec(2, 3, 5, 64, "random", 0.5, 0.5, 1.0, 1))
    good = tmp_path / "good.mask"
    D.save_mask_set(m, good)
    data = good.read_bytes()
    trunc = tmp_path / "trunc.mask"
    trunc.write_bytes(data[:-1])
    with pytest.raises(D.ParseError, match="size mismatch"):
        D.load_mask_set(trunc)
    ver = tmp_path / "ver.mask"
    ver.write_bytes(data[:8] + struct.pack("<I", 2) + data[12:])
    with pytest.raises(D.ParseError, match="unsupported version 2"):
        D.load_mask_set(ver)
    pad = tmp_path / "pad.mask"
    pad.write_bytes(data[:28] + bytes([data[28] | 0x80]) + data[29:])
    with pytest.raises(D.ParseError, match="padding bit set at byte 28"):
        D.load_mask_set(pad)
    with pytest.raises(D.IoError):
        D.load_mask_set(tmp_path / "does_not_exist.mask")
    assert issubclass(D.ParseError, D.IoError)


def test_sidecar_fixture(tmp_path):
    # proj/tests/fixtures/counts_3122.json: 4 heads, 2x2, popcounts {4,3,1,0}
    j = {"heads": 4, "q_blocks": 2, "kv_blocks": 2, "block_size": 64,
         "rows": ["03", "03", "03", "01", "01", "00", "00", "00"]}
    p = tmp_path / "counts.json"
    p.write_text(json.dumps(j))
    m = D.load_mask_set(p)
    assert D.blocks_per_head(m) == [4, 3, 1, 0]
    j["rows"] = j["rows"][:-1]
    p.write_text(json.dumps(j))
    with pytest.raises(D.ParseError, match="row strings"):
        D.load_mask_set(p)
