"""Native library builder (csrc/fps_ingest.cpp) vs the reference's own outputs.

Fixtures: tests/golden/ingest.json + ingest_lines.txt, produced by running the
real ``fpscan.libstore`` (tests/golden/make_ingest_golden.py). CPU only: the
builder is host code in libfpsgpu.so and needs no GPU.

Covers libstore.build_shards (libstore.py:243-272) from a list of lines, from
lines carrying their own CR / CRLF ends and from a text file opened like the
reference CLI (cli.py:69-70, universal newlines): byte-identical shard files
(sha256), identical manifest documents (counts, labels, FNV-1a checksums);
the reference's exception class and message for malformed lines, with no
output directory created; fnv1a_64 vectors including resumption; and
validate_manifest violations on damaged libraries.
"""

import hashlib
import json
from pathlib import Path

import pytest

from paper_1906_06170_b200 import libstore

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def ing():
    from paper_1906_06170_b200 import build

    build.build()
    return json.loads((GOLDEN / "ingest.json").read_text())


def shas(manifest):
    return [hashlib.sha256(Path(s.path).read_bytes()).hexdigest() for s in manifest.shards]


def doc(d):
    return json.loads((Path(d) / "manifest.json").read_text())


@pytest.mark.parametrize("sc", ["1", "3", "7", "400"])
def test_build_from_lines_matches_reference(ing, tmp_path, sc):
    with open(GOLDEN / "ingest_lines.txt", encoding="utf-8") as f:
        lines = list(f)
    m = libstore.build_shards(lines, int(sc), tmp_path)
    want = ing["good"]["list"][sc]
    assert shas(m) == want["shas"]
    assert doc(tmp_path) == want["manifest"]
    assert (tmp_path / "manifest.json").read_text() == json.dumps(want["manifest"], indent=2) + "\n"


def test_build_from_lines_with_own_line_ends(ing, tmp_path):
    want = ing["good"]["raw"]
    m = libstore.build_shards(want["lines"], 3, tmp_path)
    assert shas(m) == want["shas"] and doc(tmp_path) == want["manifest"]


@pytest.mark.parametrize("sc", ["1", "4"])
def test_build_from_text_file_matches_reference(ing, tmp_path, sc):
    want = ing["good"]["file"][sc]
    with open(GOLDEN / "ingest_lines.txt", encoding="utf-8") as f:
        m = libstore.build_shards(f, int(sc), tmp_path / "a")  # the CLI's call shape
    assert shas(m) == want["shas"] and doc(tmp_path / "a") == want["manifest"]
    m = libstore.build_shards_from_file(GOLDEN / "ingest_lines.txt", int(sc), tmp_path / "b", threads=3)
    assert shas(m) == want["shas"] and doc(tmp_path / "b") == want["manifest"]


def test_thread_count_does_not_change_output(ing, tmp_path):
    want = ing["good"]["file"]["4"]
    for t in (1, 2, 5, 16, 64):
        m = libstore.build_shards_from_file(GOLDEN / "ingest_lines.txt", 4, tmp_path / str(t), threads=t)
        assert shas(m) == want["shas"], t


def test_malformed_lines_raise_reference_errors(ing, tmp_path):
    from paper_1906_06170_b200 import errors

    for name, case in ing["errors"].items():
        out = tmp_path / name
        with pytest.raises(Exception) as ei:
            libstore.build_shards(case["lines"], 2, out)
        cls, msg = case["error"]
        assert type(ei.value).__name__ == cls, name
        assert str(ei.value) == msg, name
        assert isinstance(ei.value, errors.LibstoreError), name
        assert out.exists() == case["wrote"], name


def test_malformed_line_in_a_file_is_located(tmp_path):
    from paper_1906_06170_b200.errors import BadCid

    text = "".join(f"{i}\t{'01' * 83}\n" for i in range(1, 5000)) + "\r\n" + "12x\t" + "0" * 166 + "\n"
    p = tmp_path / "lib.txt"
    p.write_bytes(text.encode())
    with pytest.raises(BadCid) as ei:
        libstore.build_shards_from_file(p, 3, tmp_path / "out", threads=7)
    assert str(ei.value) == "line 5001: bad CID '12x': must be a decimal integer in 1..2^64-1"
    assert not (tmp_path / "out").exists()


def test_empty_input(tmp_path):
    m = libstore.build_shards([], 1, tmp_path)
    assert m.total_records == 0 and [s.record_count for s in m.shards] == [0]
    assert (tmp_path / "shard-000.fps").read_bytes() == b"FPS1\x01\x00\x00\x00" + bytes(8)
    assert m.shards[0].checksum == libstore.FNV64_OFFSET


def test_fnv1a_vectors(ing):
    for row in ing["fnv"]:
        if row[0] == "resume":
            data = bytes.fromhex(row[2])
            assert libstore.fnv1a_64(data[300:], libstore.fnv1a_64(data[:300])) == row[1]
        else:
            assert libstore.fnv1a_64(bytes.fromhex(row[0])) == row[1]


def test_validate_manifest_matches_reference(ing, tmp_path):
    with open(GOLDEN / "ingest_lines.txt", encoding="utf-8") as f:
        m = libstore.build_shards(f, 3, tmp_path / "val")
    base = tmp_path / "val"

    def run(name, mutate):
        d = tmp_path / ("v_" + name)
        d.mkdir()
        for s in m.shards:
            (d / Path(s.path).name).write_bytes(Path(s.path).read_bytes())
        (d / "manifest.json").write_text((base / "manifest.json").read_text())
        mutate(d)
        mm = libstore.load_manifest(d)
        got = [[v.kind, Path(v.path).name if v.path != "manifest" else "manifest",
                v.message.replace(str(d) + "/", "")] for v in libstore.validate_manifest(mm)]
        assert got == ing["validate"][name], name

    def flip_byte(d):
        p = d / "shard-001.fps"
        b = bytearray(p.read_bytes())
        b[100] ^= 1
        p.write_bytes(bytes(b))

    def truncate(d):
        p = d / "shard-002.fps"
        p.write_bytes(p.read_bytes()[:-32])

    def bad_magic(d):
        p = d / "shard-000.fps"
        b = bytearray(p.read_bytes())
        b[0:4] = b"NOPE"
        p.write_bytes(bytes(b))

    def missing(d):
        (d / "shard-001.fps").unlink()

    def count(d):
        dd = json.loads((d / "manifest.json").read_text())
        dd["shards"][0]["record_count"] += 1
        dd["total_records"] += 1
        (d / "manifest.json").write_text(json.dumps(dd))

    run("clean", lambda d: None)
    run("flip_byte", flip_byte)
    run("truncate", truncate)
    run("bad_magic", bad_magic)
    run("missing", missing)
    run("count", count)


def test_built_shards_feed_the_scan_loader(tmp_path):
    """The builder's output is what the FPS1 loader reads: records come back
    with the CIDs and words the text lines spelled (host-side check)."""
    import numpy as np

    lines = [f"{i + 10}\t{format(i * 0x9E3779B97F4A7C15 % (1 << 166), '0166b')[::-1]}\n" for i in range(50)]
    m = libstore.build_shards(lines, 3, tmp_path)
    rec = libstore.read_manifest_records(m)
    assert rec[:, 0].tolist() == list(range(10, 60))
    for i in range(50):
        v = i * 0x9E3779B97F4A7C15 % (1 << 166)
        assert [int(x) for x in rec[i, 1:]] == [v & (2**64 - 1), (v >> 64) & (2**64 - 1), v >> 128]
    assert np.all(rec[:, 3] >> np.uint64(38) == 0)
