"""Host-side logic of the package (no GPU): query normalisation and the
reference-mirroring types, merge, manifests, workload plans. CPU only."""

import json
import random

import numpy as np
import pytest

import fps_oracle as orc
from paper_1906_06170_b200 import (
    Fingerprint,
    FingerprintError,
    InvalidCharacter,
    WrongLength,
    libstore,
    parse_bitstring,
    scan,
    synth,
    to_bitstring,
)
from paper_1906_06170_b200.distributed import shard_range
from paper_1906_06170_b200.fingerprint import as_query_words
from paper_1906_06170_b200.library import RangeResult, keys_to_hits


# ---------------------------------------------------------------- fingerprints
def test_parse_round_trip_and_errors():
    rng = random.Random(1234)
    for _ in range(2000):
        s = "".join(rng.choice("01") for _ in range(166))
        assert to_bitstring(parse_bitstring(s)) == s
    assert parse_bitstring("1" + "1" + "0" * 165).keys() == {1}  # 167-char form drops the leading char
    with pytest.raises(WrongLength):
        parse_bitstring("01" * 40)
    with pytest.raises(InvalidCharacter) as exc:
        parse_bitstring("0" * 80 + "x" + "0" * 85)
    assert exc.value.position == 80
    with pytest.raises(FingerprintError):
        Fingerprint((0, 0, 1 << 38))
    assert Fingerprint.from_packed(Fingerprint.from_keys({1, 64, 65, 166}).to_packed()).keys() == {1, 64, 65, 166}


def test_query_normalisation():
    fp = Fingerprint.from_keys({1, 2, 3})
    assert as_query_words(fp).tolist() == [list(fp.words)]
    assert as_query_words([fp, fp]).shape == (2, 3)
    assert as_query_words((1, 2, 3)).tolist() == [[1, 2, 3]]
    assert as_query_words(np.zeros(3, dtype=np.uint64)).shape == (1, 3)

    class RefLike:  # the reference's Fingerprint exposes .words
        words = (5, 6, 7)

    assert as_query_words(RefLike()).tolist() == [[5, 6, 7]]
    with pytest.raises(FingerprintError):
        as_query_words(np.array([[0, 0, 1 << 38]], dtype=np.uint64))
    with pytest.raises(FingerprintError):
        as_query_words(np.zeros((2, 4), dtype=np.uint64))


# ---------------------------------------------------------------- scan types
def test_search_params_validation():
    assert scan.SearchParams().kernel == "cuda"
    for kernel in ("cuda", "packed", "reference"):
        scan.SearchParams(kernel=kernel)
    with pytest.raises(ValueError):
        scan.SearchParams(n=0)
    with pytest.raises(ValueError):
        scan.SearchParams(parallelism=0)
    with pytest.raises(ValueError):
        scan.SearchParams(kernel="numpy")


def test_topk_invariants():
    H = scan.SearchHit
    with pytest.raises(ValueError):
        scan.TopK(capacity=1, hits=(H(1, 0), H(2, 1)))
    with pytest.raises(ValueError):
        scan.TopK(capacity=5, hits=(H(2, 1), H(1, 0)))
    with pytest.raises(ValueError):
        scan.TopK(capacity=5, hits=(H(1, 0), H(1, 0)))
    with pytest.raises(ValueError):
        scan.TopK(capacity=0, hits=())


def test_merge_topk_matches_reference_golden(golden):
    for case in golden["merge"]:
        parts = [scan.TopK(capacity=len(p), hits=tuple(scan.SearchHit(c, d) for c, d in p)) for p in case["parts"]]
        got = scan.merge_topk(parts, case["n"])
        assert [[h.cid, h.distance] for h in got.hits] == case["hits"]
        rng = random.Random(case["n"])
        for _ in range(3):
            rng.shuffle(parts)
            assert scan.merge_topk(parts, case["n"]) == got  # commutativity
    a = scan.TopK(capacity=5, hits=(scan.SearchHit(42, 1),))
    b = scan.TopK(capacity=5, hits=(scan.SearchHit(42, 3),))
    with pytest.raises(scan.DuplicateCid):
        scan.merge_topk([a, b], 5)


def test_merge_associativity():
    rng = random.Random(8)
    cids = iter(rng.sample(range(1, 10**6), 300))

    def part():
        pairs = sorted((rng.randint(0, 166), next(cids)) for _ in range(80))
        return scan.TopK(capacity=80, hits=tuple(scan.SearchHit(c, d) for d, c in pairs))

    a, b, c = part(), part(), part()
    assert scan.merge_topk([scan.merge_topk([a, b], 20), c], 20) == scan.merge_topk([a, scan.merge_topk([b, c], 20)], 20)


def test_empty_manifest_needs_no_gpu():
    m = libstore.ShardManifest(shards=(), total_records=0)
    top = scan.search(m, Fingerprint.zero(), scan.SearchParams(n=10))
    assert top.hits == () and top.capacity == 10
    with pytest.raises(ValueError):
        scan.batch_search(m, [], scan.SearchParams())


def test_shard_error_names_path(tmp_path):
    bad = libstore.ShardManifest(shards=(libstore.Shard(tmp_path / "gone.fps", 5, "A", 0),), total_records=5)
    with pytest.raises((scan.ScanError, OSError)) as exc:
        scan.search(bad, Fingerprint.zero(), scan.SearchParams())
    assert "gone.fps" in str(exc.value)


def test_cancel_before_launch(tmp_path):
    w = orc.generate_words(1, np.full(166, 2**30, np.uint64), 0, 100)
    mpath = orc.write_fps1_library(tmp_path, w, 2)
    m = libstore.load_manifest(mpath.parent)
    with pytest.raises(scan.ScanCancelled):
        scan.search(m, Fingerprint.zero(), scan.SearchParams(), cancel=lambda: True)


# ---------------------------------------------------------------- libstore
def test_manifest_and_records_round_trip(tmp_path):
    w = orc.generate_words(7, synth.beta_thresholds(7), 0, 1001)
    mpath = orc.write_fps1_library(tmp_path, w, 3)
    m = libstore.load_manifest(tmp_path)
    assert m.total_records == 1001
    assert [s.record_count for s in m.shards] == libstore.split_sizes(1001, 3)
    assert [s.dataset_label for s in m.shards] == ["A", "B", "C"]
    rec = libstore.read_manifest_records(m)
    assert np.array_equal(rec[:, 1:], w)
    assert np.array_equal(rec[:, 0], np.arange(1, 1002))
    doc = json.loads(mpath.read_text())
    assert doc["format_version"] == 1


def test_shard_header_errors(tmp_path):
    p = tmp_path / "x.fps"
    p.write_bytes(b"NOPE" + b"\0" * 12)
    with pytest.raises(libstore.BadMagic if hasattr(libstore, "BadMagic") else Exception):
        with open(p, "rb") as f:
            libstore.read_shard_header(f, p)
    p.write_bytes(b"FPS1" + (2).to_bytes(2, "little") + b"\0\0" + (0).to_bytes(8, "little"))
    from paper_1906_06170_b200.errors import TruncatedFile, VersionMismatch

    with pytest.raises(VersionMismatch):
        with open(p, "rb") as f:
            libstore.read_shard_header(f, p)
    p.write_bytes(b"FPS1" + (1).to_bytes(2, "little") + b"\0\0" + (5).to_bytes(8, "little") + b"\0" * 40)
    with pytest.raises(TruncatedFile):
        libstore.read_shard_records(libstore.Shard(p, 5, "A", 0))


def test_split_and_shard_ranges(golden):
    for total, count, expect in golden["split_sizes"]:
        assert libstore.split_sizes(total, count) == expect
        starts = [shard_range(total, count, r) for r in range(count)]
        assert [c for _, c in starts] == expect
        assert all(s2 == s1 + c1 for (s1, c1), (s2, _) in zip(starts, starts[1:]))


# ---------------------------------------------------------------- plans, decoding
def test_plans_are_deterministic_and_in_distribution():
    p1 = synth.make_plan("c2", n=100_000)
    p2 = synth.make_plan("c2", n=100_000)
    assert np.array_equal(p1.planted_idx, p2.planted_idx)
    assert all(np.array_equal(a, b) for a, b in zip(p1.planted_flips, p2.planted_flips))
    assert len(p1.planted_idx) == 1000 and not set(p1.planted_idx) & set(p1.source_idx)
    assert all(len(f) == 3 and f.min() >= 2 for f in p1.query_flips)  # flips drawn from keys 2..166
    assert all(0 <= len(f) <= 4 for f in p1.planted_flips)
    assert synth.beta_thresholds(5)[0] == 0  # key 1 never set
    p5 = synth.make_plan("c5", n=200_000, planted_per_query=100)
    assert len(np.unique(p5.planted_idx)) == 64 * 100
    assert synth.CONFIGS["c3"]["n"] == 95_417_114


def test_planted_distances_equal_flip_counts():
    plan = synth.make_plan("c2", seed=3, n=50_000, planted_per_query=300)
    w = orc.generate_words(plan.seed_key, plan.thresholds, 0, plan.n)
    q = synth.planted_after_sources(plan, w)
    d = orc.distances_one(w[plan.planted_idx], q[0])
    assert np.array_equal(d, [len(f) for f in plan.planted_flips])
    assert int(orc.distances_one(w[plan.source_idx], q[0])[0]) == 3


def test_key_decoding():
    keys = np.array([[(3 << 40) | 17, (5 << 40) | 2, 2**64 - 1]], dtype=np.uint64)
    res = keys_to_hits(keys, np.array([2], dtype=np.uint32))
    assert res.hits(0) == [(17, 3), (2, 5)]
    rr = RangeResult.from_keys(np.array([(7 << 48) | (4 << 40) | 123], dtype=np.uint64))
    assert rr.rows().tolist() == [[7, 123, 4]]


def test_c_generator_matches_numpy_twin():
    """orc_generate (C, threads) == generate_words (numpy) == the device gen_kernel's definition."""
    import fps_oracle as orc

    from paper_1906_06170_b200 import synth

    plan = synth.make_plan("c2", seed=99, n=5000)
    a = orc.generate_words(plan.seed_key, plan.thresholds, 123_456, 3001)
    b = orc.generate_words_parallel(plan.seed_key, plan.thresholds, 123_456, 3001, threads=3)
    assert np.array_equal(a, b)


def test_bench_rejects_more_gpus_than_visible():
    """bench.py --gpus N fails loudly (non-zero) when N GPUs are not there,
    instead of silently measuring fewer."""
    import subprocess
    import sys
    from pathlib import Path

    import torch

    if torch.cuda.device_count() >= 2:
        pytest.skip("two GPUs visible")
    root = Path(__file__).resolve().parent.parent
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "visible GPU" in r.stdout + r.stderr
