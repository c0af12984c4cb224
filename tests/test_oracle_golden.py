"""Pin the CPU oracle (numpy + C restatements) to the real reference's outputs.

Every expectation here was produced by running /root/reference's fpscan in the
build container (tests/golden/make_golden.py). CPU only.
"""

import hashlib

import numpy as np
import pytest

import fps_oracle as orc
from paper_1906_06170_b200 import synth


def words_sha(w):
    return hashlib.sha256(np.ascontiguousarray(w, dtype="<u8").tobytes()).hexdigest()


def library(seed, n):
    return orc.generate_words(synth.seed_key(seed), synth.beta_thresholds(seed), 0, n)


def test_kat_distances(golden):
    for a, b, d in golden["kat"]:
        assert orc.distance_packed(a, b) == d
        assert orc.manhattan_reference(a, b) == d
        assert int(orc.distances_one(np.array([a], dtype=np.uint64), np.array(b, dtype=np.uint64))[0]) == d


def test_single_bit_pairs_are_two_apart():
    # test_acceptance.py:98-100: every pair of distinct single-key fingerprints is at distance 2
    from paper_1906_06170_b200.fingerprint import Fingerprint

    singles = np.array([Fingerprint.from_keys({j}).words for j in range(1, 167)], dtype=np.uint64)
    for j in range(166):
        d = orc.distances_one(singles, singles[j])
        assert int(d[j]) == 0
        assert np.all(np.delete(d, j) == 2)


def test_split_sizes(golden):
    for total, count, expect in golden["split_sizes"]:
        assert orc.split_sizes(total, count) == expect


def test_generator_pinned(golden):
    for g in golden["generator"]:
        w = library(g["seed"], g["n"])
        assert words_sha(w) == g["sha256"]
        assert [[int(x) for x in r] for r in w[:4]] == g["first"]
        # key 1 is never set (p_1 = 0) and padding bits stay clear
        assert not np.any(w[:, 0] & np.uint64(1))
        assert not np.any(w[:, 2] >> np.uint64(38))


def test_generator_host_rows_match_twin():
    seed = 99
    thr = synth.beta_thresholds(seed)
    idx = np.array([0, 5, 77, 4095])
    w = orc.generate_words(synth.seed_key(seed), thr, 0, 4096)
    assert np.array_equal(synth.generate_rows(synth.seed_key(seed), thr, idx), w[idx])
    # chunk determinism: any window of the stream is reproducible on its own
    assert np.array_equal(orc.generate_words(synth.seed_key(seed), thr, 1000, 50), w[1000:1050])


def test_fps1_writer_byte_identical_to_reference(golden, tmp_path):
    for f in golden["fps1"]:
        w = library(f["seed"], f["n"])
        path = orc.write_fps1_library(tmp_path / str(f["seed"]), w, f["shards"])
        shards = sorted(path.parent.glob("shard-*.fps"))
        assert [hashlib.sha256(s.read_bytes()).hexdigest() for s in shards] == f["sha256"]
        import json

        doc = json.loads(path.read_text())
        assert [s["checksum"] for s in doc["shards"]] == f["checksums"]


def _case_library(case):
    plan = synth.make_plan(case["case"], seed=case["seed"], n=case["n"],
                           planted_per_query=200 if case["case"] == "c2" else None)
    w = orc.generate_words(plan.seed_key, plan.thresholds, 0, case["n"])
    q = synth.planted_after_sources(plan, w)
    assert words_sha(w) == case["sha256"]
    return w, q


def test_search_cases(golden):
    for case in golden["search"]:
        w, q = _case_library(case)
        assert [int(x) for x in q[0]] == case["query"]
        expect = [(c - 1, d) for c, d in case["hits"]]  # cid = index + 1
        k = case["k"]
        assert orc.search(w, q[0], k, shard_count=case["shards"], parallelism=case["parallelism"]) == expect
        assert orc.topk_full_sort(w, q[0], k) == expect
        idx, dist, cnt = orc.c_topk(w, q[:1], k, threads=3)
        assert list(zip(idx[0, :cnt[0]].tolist(), dist[0, :cnt[0]].tolist())) == expect


def test_per_query_cases(golden):
    for case in golden["per_query"]:
        plan = synth.make_plan("c4", seed=case["seed"], n=case["n"], Q=case["Q"])
        w = orc.generate_words(plan.seed_key, plan.thresholds, 0, plan.n)
        q = synth.planted_after_sources(plan, w)
        assert words_sha(w) == case["sha256"]
        assert q.tolist() == case["queries"]
        idx, dist, cnt = orc.c_topk(w, q, case["k"])
        for qi, hits in enumerate(case["hits"]):
            expect = [(c - 1, d) for c, d in hits]
            assert orc.batch_topk(w, q[qi:qi + 1], case["k"])[0] == expect
            assert list(zip(idx[qi, :cnt[qi]].tolist(), dist[qi, :cnt[qi]].tolist())) == expect


def test_batch_min_case(golden):
    case = golden["batch_min"][0]
    plan = synth.make_plan("c4", seed=case["seed"], n=case["n"], Q=12)
    w = orc.generate_words(plan.seed_key, plan.thresholds, 0, plan.n)
    synth.planted_after_sources(plan, w)
    q = np.array(case["queries"], dtype=np.uint64)
    expect = [(c - 1, d) for c, d in case["hits"]]
    assert orc.batch_min_topk(w, q, case["k"]) == expect
    assert orc.search(w, q, case["k"], shard_count=2) == expect


def test_range_case(golden):
    case = golden["range"][0]
    plan = synth.make_plan("c5", seed=case["seed"], n=case["n"], Q=case["Q"], planted_per_query=50)
    w = orc.generate_words(plan.seed_key, plan.thresholds, 0, plan.n)
    q = synth.planted_after_sources(plan, w)
    assert words_sha(w) == case["sha256"]
    rows = np.array(case["rows"], dtype=np.int64).reshape(-1, 3)
    assert np.array_equal(orc.range_search(w, q, case["radius"]), rows)
    assert np.array_equal(orc.c_range(w, q, case["radius"]), rows)
    # every planted near-duplicate (0..6 flips) is found at its flip count
    for i, qi, f in zip(plan.planted_idx, plan.planted_query, plan.planted_flips):
        hit = rows[(rows[:, 0] == qi) & (rows[:, 1] == i)]
        assert len(hit) == 1 and hit[0, 2] == len(f)


def test_tensor_core_shaped_cases(golden):
    """The >= 192-query goldens (the GPU's tensor-core path) pin the oracles too."""
    case = golden["per_query_tc"]
    plan = synth.make_plan("c4", seed=case["seed"], n=case["n"], Q=case["Q"])
    w = orc.generate_words(plan.seed_key, plan.thresholds, 0, plan.n)
    q = synth.planted_after_sources(plan, w)
    assert words_sha(w) == case["sha256"] and q.tolist() == case["queries"]
    idx, dist, cnt = orc.c_topk(w, q, case["k"])
    for qi, hits in enumerate(case["hits"]):
        assert list(zip(idx[qi, :cnt[qi]].tolist(), dist[qi, :cnt[qi]].tolist())) == [(c - 1, d) for c, d in hits]
    for bm in golden["batch_min_large"]:
        assert orc.batch_min_topk(w, np.array(bm["queries"], dtype=np.uint64), bm["k"]) == \
            [(c - 1, d) for c, d in bm["hits"]]
    rc = golden["range_tc"]
    plan = synth.make_plan("c5", seed=rc["seed"], n=rc["n"], Q=rc["Q"], planted_per_query=rc["planted_per_query"])
    w = orc.generate_words(plan.seed_key, plan.thresholds, 0, plan.n)
    q = synth.planted_after_sources(plan, w)
    assert words_sha(w) == rc["sha256"]
    assert np.array_equal(orc.c_range(w, q, rc["radius"]), np.array(rc["rows"], dtype=np.int64).reshape(-1, 3))


def test_cid_library_search(golden):
    from pathlib import Path

    rec = np.load(Path(__file__).parent / "golden" / "cid_library.npy")
    words, cids = rec[:, 1:], rec[:, 0]
    for case in golden["cid_search"]:
        got = orc.scan_shard(words, np.array(case["query"], dtype=np.uint64), case["k"], ids=cids)
        assert [[c, d] for c, d in got] == case["hits"]
    cb = golden["cid_batch_min"]
    got = orc.scan_shard(words, np.array(cb["queries"], dtype=np.uint64), cb["k"], ids=cids)
    assert [[c, d] for c, d in got] == cb["hits"]


def test_merge_cases(golden):
    for case in golden["merge"]:
        parts = [[(c, d) for c, d in p] for p in case["parts"]]
        assert [[c, d] for c, d in orc.merge_topk(parts, case["n"])] == case["hits"]
    with pytest.raises(ValueError):
        orc.merge_topk([[(42, 1)], [(42, 3)]], 5)


def test_top_k_is_prefix_of_range():
    """Pins the range restatement through the top-k oracle: the k nearest are
    exactly the first k range hits when the radius covers them."""
    w = library(5, 20000)
    q = w[17].copy()
    q[1] ^= np.uint64(0b1011)
    top = orc.topk_full_sort(w, q, 25)
    r = orc.range_search(w, q, top[-1][1])
    assert [(int(i), int(d)) for _, i, d in r[:25]] == top
