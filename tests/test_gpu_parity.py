"""CUDA path vs the oracle and the reference's golden outputs (needs a B200).

Every call goes through libfpsgpu.so's C ABI (via the ctypes shim). Integer
work: the bar is bit-exact equality of (index or cid, distance) lists in the
reference's (distance, id) order.
"""

import hashlib
from pathlib import Path

import numpy as np
import pytest

import fps_oracle as orc
from paper_1906_06170_b200 import FingerprintError, scan, synth
from paper_1906_06170_b200.fingerprint import Fingerprint
from paper_1906_06170_b200.library import Library, keys_to_hits, merge_async

pytestmark = pytest.mark.gpu

GOLDEN_DIR = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module", autouse=True)
def _device():
    import torch

    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    from paper_1906_06170_b200 import build

    build.build()
    yield
    scan.clear_cache()


def words_sha(w):
    return hashlib.sha256(np.ascontiguousarray(w, dtype="<u8").tobytes()).hexdigest()


def as_pairs(res, q=0):
    return res.hits(q)


def oracle_topk(w, q, k):
    idx, dist, cnt = orc.c_topk(w, q, k)
    return [list(zip(idx[i, :cnt[i]].tolist(), dist[i, :cnt[i]].tolist())) for i in range(len(q))]


# ---------------------------------------------------------------- generator
def test_device_generator_matches_numpy_twin():
    seed = 31337
    thr = synth.beta_thresholds(seed)
    lib = Library.generate(100_003, synth.seed_key(seed), thr, start=0)
    w = lib.words_host()
    assert np.array_equal(w, orc.generate_words(synth.seed_key(seed), thr, 0, 100_003))
    part = Library.generate(777, synth.seed_key(seed), thr, start=5000)
    assert np.array_equal(part.words_host(), w[5000:5777])
    assert part.index_base == 5000


# ---------------------------------------------------------------- golden pins
def _case(case):
    plan = synth.make_plan(case["case"], seed=case["seed"], n=case["n"],
                           planted_per_query=200 if case["case"] == "c2" else None)
    lib, q = synth.build_library(plan)
    w = lib.words_host()
    assert words_sha(w) == case["sha256"]
    return lib, q, w


def test_search_matches_reference_golden(golden):
    for case in golden["search"]:
        lib, q, _ = _case(case)
        assert [int(x) for x in q[0]] == case["query"]
        got = lib.search(q[0], case["k"])
        assert got == [(c - 1, d) for c, d in case["hits"]], (case["case"], case["k"])


def test_search_through_fps1_manifest(golden, tmp_path):
    """The drop-in path: FPS1 shards + manifest -> scan.search -> TopK of (cid, distance)."""
    for case in golden["search"][:4]:
        plan = synth.make_plan(case["case"], seed=case["seed"], n=case["n"],
                               planted_per_query=200 if case["case"] == "c2" else None)
        w = orc.generate_words(plan.seed_key, plan.thresholds, 0, plan.n)
        q = synth.planted_after_sources(plan, w)
        mpath = orc.write_fps1_library(tmp_path / f"{case['case']}_{case['k']}", w, case["shards"])
        from paper_1906_06170_b200 import libstore

        manifest = libstore.load_manifest(mpath.parent)
        seen = []
        top = scan.search(manifest, Fingerprint(tuple(int(x) for x in q[0])),
                          scan.SearchParams(n=case["k"], parallelism=case["parallelism"]),
                          progress=lambda label, done, total: seen.append((label, done, total)))
        assert [[h.cid, h.distance] for h in top.hits] == case["hits"]
        assert {s[0] for s in seen} == {s.dataset_label for s in manifest.shards}
        assert all(d == t for _, d, t in seen)


def test_per_query_matches_reference_golden(golden):
    case = golden["per_query"][0]
    plan = synth.make_plan("c4", seed=case["seed"], n=case["n"], Q=case["Q"])
    lib, q = synth.build_library(plan)
    assert q.tolist() == case["queries"]
    res = lib.search_batch(q, case["k"])
    for qi, hits in enumerate(case["hits"]):
        assert res.hits(qi) == [(c - 1, d) for c, d in hits]


def test_batch_min_matches_reference_golden(golden):
    case = golden["batch_min"][0]
    plan = synth.make_plan("c4", seed=case["seed"], n=case["n"], Q=12)
    lib, _ = synth.build_library(plan)
    got = lib.search_min(np.array(case["queries"], dtype=np.uint64), case["k"])
    assert got == [(c - 1, d) for c, d in case["hits"]]


def test_range_matches_reference_golden(golden):
    case = golden["range"][0]
    plan = synth.make_plan("c5", seed=case["seed"], n=case["n"], Q=case["Q"], planted_per_query=50)
    lib, q = synth.build_library(plan)
    r = lib.range_search(q, case["radius"])
    assert np.array_equal(r.rows(), np.array(case["rows"], dtype=np.int64).reshape(-1, 3))


@pytest.mark.parametrize("kind", [None, "fp4x", "fp4"])
def test_tensor_core_per_query_matches_reference_golden(golden, kind, monkeypatch):
    """256 queries take the tcgen05 kernel by default (int8; also the fp4
    kinds: from the operand copy and expanded in the kernel); pinned directly
    to the reference's own search() outputs (make_golden.py per_query_tc)."""
    if kind:
        monkeypatch.setenv("FPS_MMA_KIND", kind)
    case = golden["per_query_tc"]
    plan = synth.make_plan("c4", seed=case["seed"], n=case["n"], Q=case["Q"])
    lib, q = synth.build_library(plan)
    assert words_sha(lib.words_host()) == case["sha256"]
    assert q.tolist() == case["queries"]
    res = lib.search_batch(q, case["k"])
    assert lib.last_kernel == "tensor-core multi-query scan"
    assert lib.last_mma_kind == (kind or "i8")
    for qi, hits in enumerate(case["hits"]):
        assert res.hits(qi) == [(c - 1, d) for c, d in hits], qi
    if kind is None:
        # 100 of the queries: one fp4 chunk, the default fp4 operand-copy kernel
        res = lib.search_batch(q[:100], case["k"])
        assert lib.last_kernel == "tensor-core multi-query scan" and lib.last_mma_kind == "fp4x"
        for qi, hits in enumerate(case["hits"][:100]):
            assert res.hits(qi) == [(c - 1, d) for c, d in hits], qi


@pytest.mark.parametrize("kind", [None, "fp4x"])
def test_tensor_core_range_matches_reference_golden(golden, kind, monkeypatch):
    if kind:
        monkeypatch.setenv("FPS_MMA_KIND", kind)
    case = golden["range_tc"]
    plan = synth.make_plan("c5", seed=case["seed"], n=case["n"], Q=case["Q"],
                           planted_per_query=case["planted_per_query"])
    lib, q = synth.build_library(plan)
    assert words_sha(lib.words_host()) == case["sha256"]
    r = lib.range_search(q, case["radius"])
    assert lib.last_kernel == "tensor-core multi-query scan"
    assert np.array_equal(r.rows(), np.array(case["rows"], dtype=np.int64).reshape(-1, 3))


def test_batch_min_large_n_matches_reference_golden(golden):
    """batch_search with n > 1024 (the reference accepts any n >= 1)."""
    plan = synth.make_plan("c4", seed=20240813, n=40_000, Q=256)
    lib, _ = synth.build_library(plan)
    for case in golden["batch_min_large"]:
        got = lib.search_min(np.array(case["queries"], dtype=np.uint64), case["k"])
        assert got == [(c - 1, d) for c, d in case["hits"]], case["k"]


def test_random_cid_library_matches_reference_golden(golden, tmp_path):
    rec = np.load(GOLDEN_DIR / "cid_library.npy")
    mpath = orc.write_fps1_library(tmp_path / "cids", rec[:, 1:], 3, cids=rec[:, 0])
    from paper_1906_06170_b200 import libstore

    manifest = libstore.load_manifest(mpath.parent)
    for case in golden["cid_search"]:
        top = scan.search(manifest, tuple(case["query"]), scan.SearchParams(n=case["k"]))
        assert [[h.cid, h.distance] for h in top.hits] == case["hits"]
    cb = golden["cid_batch_min"]
    top = scan.batch_search(manifest, [tuple(x) for x in cb["queries"]], scan.SearchParams(n=cb["k"]))
    assert [[h.cid, h.distance] for h in top.hits] == cb["hits"]


def test_random_cids_heavy_ties_match_oracle(tmp_path):
    """Arbitrary (non-monotone) CIDs with heavy distance ties: 40 % of the
    records are copies of 40 hub fingerprints, so hundreds of records tie at
    every distance near a hub. The resident library is uploaded in CID order,
    so the plain top-k is exact in (distance, cid) order — checked against the
    reference's search restated over the same FPS1 shards (scan.py:173-287),
    for search and for batch_search (min over queries, scan.py:306-318)."""
    from paper_1906_06170_b200 import libstore

    rng = np.random.default_rng(77)
    n = 120_000
    w = orc.generate_words(synth.seed_key(77), synth.beta_thresholds(77), 0, n)
    hubs = w[rng.integers(0, n, 40)].copy()
    pick = rng.random(n) < 0.4
    w[pick] = hubs[rng.integers(0, 40, int(pick.sum()))]
    cids = rng.choice(1 << 62, size=n, replace=False).astype(np.uint64)
    mpath = orc.write_fps1_library(tmp_path / "ties", w, 5, cids=cids)
    manifest = libstore.load_manifest(mpath.parent)
    queries = [hubs[0], hubs[7] ^ np.array([1 << 3, 0, 0], dtype=np.uint64), w[5]]
    for q in queries:
        for k in (1, 10, 100, 1000):
            top = scan.search(manifest, tuple(int(x) for x in q), scan.SearchParams(n=k))
            exp = orc.search_fps1(mpath, np.asarray(q, dtype=np.uint64), k)
            assert [(h.cid, h.distance) for h in top.hits] == [(int(c), int(d)) for c, d in exp], k
    qs = np.stack(queries[:2])
    dmin = np.minimum(orc.distances_one(w, qs[0]), orc.distances_one(w, qs[1])).astype(np.int64)
    order = np.lexsort((cids, dmin))[:50]
    top = scan.batch_search(manifest, [tuple(int(x) for x in q) for q in qs], scan.SearchParams(n=50))
    assert [(h.cid, h.distance) for h in top.hits] == [(int(cids[i]), int(dmin[i])) for i in order]


# ---------------------------------------------------------------- oracle sweeps
@pytest.mark.parametrize("n", [1, 5, 31, 127, 128, 129, 1000, 4097, 65_537, 300_001])
def test_topk_tail_sizes(n):
    w = orc.generate_words(12345, np.full(166, 2**30, np.uint64), 0, n)
    lib = Library.from_words(w)
    q = w[n // 2:n // 2 + 1].copy()
    q[0, 1] ^= np.uint64(0xF0F0)
    for k in (1, 10, 100):
        assert lib.search(q[0], k) == oracle_topk(w, q, k)[0]


@pytest.mark.parametrize("popc", [False, True])
@pytest.mark.parametrize("Q", [1, 2, 3, 4, 5, 7, 8, 9, 16, 17, 33])
def test_topk_query_counts(Q, popc, monkeypatch):
    """Q >= 2 takes the bit-sliced kernel (1, 2 or 4 queries per warp by Q);
    FPS_BITSLICE=0 keeps the POPC kernels (QW = 2/4/8 query words in
    registers) covered too."""
    if popc:
        monkeypatch.setenv("FPS_BITSLICE", "0")
    seed = 4242 + Q
    thr = synth.beta_thresholds(seed)
    w = orc.generate_words(synth.seed_key(seed), thr, 0, 200_000)
    rng = np.random.default_rng(Q)
    q = w[rng.integers(0, len(w), Q)].copy()
    q[:, 0] ^= rng.integers(0, 2**20, Q).astype(np.uint64) << np.uint64(1)
    lib = Library.from_words(w)
    for k in (1, 10, 64):
        res = lib.search_batch(q, k)
        exp = oracle_topk(w, q, k)
        for i in range(Q):
            assert res.hits(i) == exp[i], (Q, k, i)


@pytest.mark.parametrize("k", [1000, 1024, 1025, 4000])
def test_large_k(k):
    w = orc.generate_words(777, np.full(166, 2**31, np.uint64), 0, 150_000)
    q = w[:3].copy()
    lib = Library.from_words(w)
    res = lib.search_batch(q, k)
    exp = oracle_topk(w, q, k)
    for i in range(3):
        assert res.hits(i) == exp[i]


def test_k_larger_than_library():
    w = orc.generate_words(5, np.full(166, 2**31, np.uint64), 0, 50)
    lib = Library.from_words(w)
    assert lib.search(w[3], 100) == oracle_topk(w, w[3:4], 100)[0]
    assert len(lib.search(w[3], 100)) == 50
    assert lib.search(w[3], 2000) == oracle_topk(w, w[3:4], 2000)[0]


def test_all_ties_library():
    """Every entry identical: the answer is the first k indices (index tie-break),
    and the threshold ties overflow the shared-memory tie buffer."""
    w = np.tile(np.array([[0x1234, 0x5678, 0x9]], dtype=np.uint64), (200_000, 1))
    lib = Library.from_words(w)
    for k in (1, 10, 100, 1024):
        got = lib.search(np.array([0x1234, 0x5678, 0x8], dtype=np.uint64), k)
        assert got == [(i, 1) for i in range(k)]


def test_adversarial_decreasing_distances():
    """Distances fall with the index, so every block improves the running top-k."""
    n = 120_000
    w = np.zeros((n, 3), dtype=np.uint64)
    bits = 166 - (np.arange(n) * 166 // n)  # popcount decreasing from 166
    for i, b in enumerate(bits):
        v = (1 << int(b)) - 1
        w[i] = (v & (2**64 - 1), (v >> 64) & (2**64 - 1), v >> 128)
    lib = Library.from_words(w)
    q = np.zeros(3, dtype=np.uint64)
    for k in (10, 100, 500):
        assert lib.search(q, k) == oracle_topk(w, q[None], k)[0]


def test_empty_library():
    lib = Library.from_words(np.zeros((0, 3), dtype=np.uint64))
    assert lib.search(np.zeros(3, dtype=np.uint64), 5) == []
    assert len(lib.range_search(np.zeros((2, 3), dtype=np.uint64), 10)) == 0


def test_padding_bits_rejected():
    lib = Library.from_words(np.zeros((10, 3), dtype=np.uint64))
    with pytest.raises(FingerprintError):
        lib.search(np.array([0, 0, 1 << 38], dtype=np.uint64), 3)
    with pytest.raises(FingerprintError):
        Library.from_words(np.array([[0, 0, 1 << 40]], dtype=np.uint64))


def test_fps1_padding_scanned_as_stored():
    """The reference scan XORs the full third word of the record view
    (scan.py:142), so stray pad bits count; FPS1 ingestion keeps them."""
    rec = np.zeros((100, 4), dtype=np.uint64)
    rec[:, 0] = np.arange(1, 101)
    rec[7, 3] = np.uint64(0xFF) << np.uint64(40)  # 8 bits set in the record pad area
    lib = Library.from_records(rec)
    got = lib.search(np.zeros(3, dtype=np.uint64), 100)
    assert got[-1] == (7, 8)


@pytest.mark.parametrize("popc", [False, True])
@pytest.mark.parametrize("radius", [0, 3, 6, 40])
def test_range_vs_oracle(radius, popc, monkeypatch):
    if popc:  # the POPC kernels instead of the bit-sliced one
        monkeypatch.setenv("FPS_BITSLICE", "0")
    seed = 99
    thr = synth.beta_thresholds(seed)
    w = orc.generate_words(synth.seed_key(seed), thr, 0, 250_000)
    q = w[[3, 77, 1000, 200_000, 5, 6, 7, 8, 9]].copy()
    q[:, 1] ^= np.uint64(0b111)
    lib = Library.from_words(w)
    r = lib.range_search(q, radius)
    assert np.array_equal(r.rows(), orc.c_range(w, q, radius))


def test_range_per_query_radius_and_overflow_retry():
    w = orc.generate_words(3, np.full(166, 2**31, np.uint64), 0, 400_000)
    q = w[:5].copy()
    radii = np.array([0, 95, 90, 80, 166], dtype=np.uint8)  # > 1M hits: first pass overflows
    lib = Library.from_words(w)
    r = lib.range_search(q, radii)
    exp = np.concatenate([orc.c_range(w, q[i:i + 1], int(radii[i])) + np.array([i, 0, 0]) for i in range(5)])
    assert len(r) > 1 << 20
    assert np.array_equal(r.rows(), exp)


def test_multi_shard_merge_on_one_gpu():
    """G logical shards with global index_base, per-shard device top-k, then the
    device merge kernel: equals a single-library search (merge_topk semantics)."""
    import torch

    seed = 2024
    thr = synth.beta_thresholds(seed)
    n = 300_000
    w = orc.generate_words(synth.seed_key(seed), thr, 0, n)
    rng = np.random.default_rng(0)
    q = w[rng.integers(0, n, 6)].copy()
    q[:, 2] ^= np.uint64(1)
    for G in (2, 3, 8):
        offs = [0]
        for s in orc.split_sizes(n, G):
            offs.append(offs[-1] + s)
        k = 25
        dq = torch.from_numpy(q.view(np.int64)).cuda()
        keys = torch.empty((G, len(q), k), dtype=torch.int64, device="cuda")
        cnt = torch.empty((G, len(q)), dtype=torch.int32, device="cuda")
        libs = [Library.from_words(w[a:b], index_base=a) for a, b in zip(offs, offs[1:])]
        stream = torch.cuda.current_stream().cuda_stream
        for g, lib in enumerate(libs):
            lib.topk_prepare(len(q), k)
            lib.topk_async(dq, len(q), k, keys[g], cnt[g], stream)
        out_k = torch.empty((len(q), k), dtype=torch.int64, device="cuda")
        out_c = torch.empty((len(q),), dtype=torch.int32, device="cuda")
        merge_async(keys, cnt, G, len(q), k, out_k, out_c, stream)
        torch.cuda.synchronize()
        res = keys_to_hits(out_k.cpu().numpy().view(np.uint64), out_c.cpu().numpy().astype(np.uint32))
        exp = oracle_topk(w, q, k)
        for i in range(len(q)):
            assert res.hits(i) == exp[i], (G, i)


def test_repeated_calls_are_deterministic():
    seed = 11
    thr = synth.beta_thresholds(seed)
    w = orc.generate_words(synth.seed_key(seed), thr, 0, 500_000)
    lib = Library.from_words(w)
    q = w[[1, 2, 3]].copy()
    first = lib.search_batch(q, 30)
    for _ in range(5):
        again = lib.search_batch(q, 30)
        assert np.array_equal(first.index, again.index) and np.array_equal(first.distance, again.distance)
    assert first.hits(0)[0] == (1, 0)


def test_compact_and_full_layouts_agree(monkeypatch):
    """With FPS_LAYOUT=compact valid fingerprints use the 21-byte tiles; an FPS1
    record with pad bits beyond bit 39 of word 2 forces the 24-byte layout.
    Both answer identically to the oracle."""
    monkeypatch.setenv("FPS_LAYOUT", "compact")
    seed = 77
    thr = synth.beta_thresholds(seed)
    w = orc.generate_words(synth.seed_key(seed), thr, 0, 70_001)
    q = w[[5, 6, 7]].copy()
    q[:, 0] ^= np.uint64(0b110)
    lib = Library.from_words(w)
    assert lib.layout() == (True, 21)
    rec = orc.records_from_words(w)
    rec[100, 3] |= np.uint64(1) << np.uint64(45)  # a pad byte set in the FPS1 record
    wide = Library.from_records(rec)
    assert wide.layout() == (False, 24)
    w_wide = rec[:, 1:].copy()
    for k in (1, 10, 100):
        assert lib.search_batch(q, k).hits(0) == oracle_topk(w, q, k)[0]
        res = wide.search_batch(q, k)
        exp = oracle_topk(w_wide, q, k)
        assert [res.hits(i) for i in range(3)] == exp
    assert np.array_equal(wide.words_host(), w_wide)
    with pytest.raises(ValueError):
        lib.write_entries(np.array([3]), np.array([[0, 0, 1 << 41]], dtype=np.uint64))


def test_fps1_loader_retiles_to_compact(tmp_path, monkeypatch):
    """FPS1 records stream into 24 B tiles and are re-tiled to the 21 B layout
    when no record uses bits 40.. of word 2; a record with such a pad bit keeps
    the 24 B tiles (and is counted, as the reference counts it); FPS_LAYOUT=full
    forces them. Every layout answers like the oracle."""
    seed = 4321
    thr = synth.beta_thresholds(seed)
    w = orc.generate_words(synth.seed_key(seed), thr, 0, 200_003)
    q = w[[11, 12]].copy()
    q[:, 1] ^= np.uint64(0b1011)
    orc.write_fps1_library(tmp_path / "ok", w, 2)
    paths = sorted(str(p) for p in (tmp_path / "ok").glob("shard-*.fps"))
    lib = Library.from_fps1(paths)
    assert lib.layout() == (True, 21)
    assert np.array_equal(lib.words_host(), w)
    for k in (1, 10, 100):
        assert [lib.search_batch(q, k).hits(i) for i in range(2)] == oracle_topk(w, q, k)
    monkeypatch.setenv("FPS_LAYOUT", "full")
    full = Library.from_fps1(paths)
    assert full.layout() == (False, 24)
    assert full.search_batch(q, 10).hits(0) == lib.search_batch(q, 10).hits(0)
    monkeypatch.delenv("FPS_LAYOUT")
    ww = w.copy()
    ww[777, 2] |= np.uint64(1) << np.uint64(50)  # a pad bit past key 166, beyond the compact word
    orc.write_fps1_library(tmp_path / "wide", ww, 2)
    paths = sorted(str(p) for p in (tmp_path / "wide").glob("shard-*.fps"))
    wide = Library.from_fps1(paths)
    assert wide.layout() == (False, 24)
    qq = w[777:778].copy()  # the record's pad bit counts as one differing key
    assert wide.search(qq, 3) == oracle_topk(ww, qq, 3)[0]
    assert wide.search(qq, 1)[0] == (777, 1)
    assert [wide.search_batch(q, 10).hits(i) for i in range(2)] == oracle_topk(ww, q, 10)


def test_fps1_streaming_loader(tmp_path):
    """FPS1 shards stream straight into HBM; any record slice of the
    concatenation (a rank's shard) loads with its global index base."""
    seed = 1234
    thr = synth.beta_thresholds(seed)
    n = 2_500_011  # > 2 loader chunks
    w = orc.generate_words(synth.seed_key(seed), thr, 0, 300_000)
    w = np.concatenate([w] * 8 + [w[:n - 8 * len(w)]])
    cids = np.arange(7, 7 + 3 * n, 3, dtype=np.uint64)
    mpath = orc.write_fps1_library(tmp_path, w, 3, cids=cids)
    paths = sorted(str(p) for p in tmp_path.glob("shard-*.fps"))
    lib = Library.from_fps1(paths)
    assert lib.n == n and lib.index_base == 0
    assert np.array_equal(lib.words_host(), w)
    assert np.array_equal(lib.cids, cids)
    start, count = 833_000, 900_001  # crosses a shard boundary
    part = Library.from_fps1(paths, start=start, count=count)
    assert part.index_base == start and part.n == count
    assert np.array_equal(part.words_host(), w[start:start + count])
    assert np.array_equal(part.cids, cids[start:start + count])
    q = w[start + 5].copy()
    assert part.search(q, 5)[0] == (start + 5, 0)
    from paper_1906_06170_b200 import libstore

    via_manifest = scan.search(libstore.load_manifest(mpath.parent), tuple(int(x) for x in q), scan.SearchParams(n=3))
    assert via_manifest.hits[0].distance == 0


@pytest.mark.parametrize("n", [2048, 2049, 2080, 2081, 4095, 70_001, 132_127])
def test_bitslice_tails_and_query_groups(n, monkeypatch):
    """Q >= 32 runs the bit-sliced kernel: 2,048-entry tiles, two 32-entry
    blocks per lane. Library sizes around the tile / block / lane-pair
    boundaries, two query groups (Q = 70 > 64 per CTA), sparse and dense
    queries (|q| > 83 counts the zero keys), top-k and range: all equal the
    oracle (FPS_MMA=0: batches of >= 64 queries default to the tensor cores)."""
    monkeypatch.setenv("FPS_MMA", "0")
    seed = 9000 + n
    thr = synth.beta_thresholds(seed)
    w = orc.generate_words(synth.seed_key(seed), thr, 0, n)
    rng = np.random.default_rng(n)
    Q = 70
    q = w[rng.integers(0, n, Q)].copy()
    q[:, 0] ^= rng.integers(0, 2**16, Q).astype(np.uint64) << np.uint64(1)
    dense = np.array([~np.uint64(0), ~np.uint64(0), np.uint64((1 << 38) - 1)], dtype=np.uint64)
    q[:8] = dense ^ q[:8] & np.uint64(0x0F0F0F0F)  # mostly-ones queries
    q[:8, 2] &= np.uint64((1 << 38) - 1)
    lib = Library.from_words(w)
    for k in (1, 10, 100):
        res = lib.search_batch(q, k)
        exp = oracle_topk(w, q, k)
        for i in range(Q):
            assert res.hits(i) == exp[i], (n, k, i)
    assert lib.last_kernel == "bit-sliced multi-query scan"
    r = lib.range_search(q[:40], 12)
    assert np.array_equal(r.rows(), orc.c_range(w, q[:40], 12))


@pytest.mark.parametrize("popc", [False, True])
@pytest.mark.parametrize("Q", [2, 5, 40])
def test_batch_min_on_the_batched_kernel(Q, popc, monkeypatch):
    """batch_search (min over queries, one top-k; scan.py:306-318): per-query
    top-k on the bit-sliced kernel + the on-device min merge, or the
    single-pass POPC min kernel (FPS_BITSLICE=0). Both equal the oracle,
    including entries that several queries list and distance ties."""
    if popc:
        monkeypatch.setenv("FPS_BITSLICE", "0")
    seed = 515 + Q
    thr = synth.beta_thresholds(seed)
    w = orc.generate_words(synth.seed_key(seed), thr, 0, 150_000)
    rng = np.random.default_rng(Q)
    src = rng.integers(0, len(w), Q)
    src[1] = src[0]  # two queries near the same entry: shared hits
    q = w[src].copy()
    q[:, 0] ^= rng.integers(0, 2**12, Q).astype(np.uint64) << np.uint64(1)
    lib = Library.from_words(w)
    for k in (1, 10, 100, 1000):
        assert lib.search_min(q, k) == orc.batch_min_topk(w, q, k), (Q, k)


# ---------------------------------------------------------------- single-query plane scan
def _dev_topk(lib, q, k):
    """fps_topk_async with the query on the device (the plane count is not known to the host)."""
    import torch

    dq = torch.from_numpy(np.ascontiguousarray(q[:1]).view(np.int64).copy()).cuda()
    keys = torch.empty((1, k), dtype=torch.int64, device="cuda")
    cnt = torch.empty((1,), dtype=torch.int32, device="cuda")
    lib.topk_prepare(1, k)
    lib.topk_async(dq, 1, k, keys, cnt, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return keys_to_hits(keys.cpu().numpy().view(np.uint64), cnt.cpu().numpy()).hits(0)


def _query_with_pop(rng, pop):
    bits = rng.choice(np.arange(1, 166), size=pop, replace=False)  # key 1 (bit 0) stays clear
    q = np.zeros(3, dtype=np.uint64)
    for b in bits:
        q[b // 64] |= np.uint64(1) << np.uint64(b % 64)
    return q


@pytest.mark.parametrize("n", [1, 31, 2047, 2048, 2049, 4097, 100_003])
def test_plane_scan_sizes_and_query_densities(n, monkeypatch):
    """Q = 1 reads only the query's planes (|q| <= 83: set keys, else zero
    keys): both host (query inline) and device query paths, list lengths on
    both sides of the 8-plane padding and of the dense switch, against the
    oracle and the POPC scan (FPS_PLANEQ=0)."""
    seed = 9000 + n
    w = orc.generate_words(synth.seed_key(seed), synth.beta_thresholds(seed), 0, n)
    lib = Library.from_words(w)
    rng = np.random.default_rng(n)
    for pop in (0, 1, 8, 9, 38, 83, 84, 120, 165):
        q = _query_with_pop(rng, pop)
        for k in (1, 10, 100):
            exp = oracle_topk(w, q[None], k)[0]
            assert lib.search(q, k) == exp, (n, pop, k)
            assert lib.last_kernel == "single-query plane scan"
            assert _dev_topk(lib, q[None], k) == exp, (n, pop, k)
    monkeypatch.setenv("FPS_PLANEQ", "0")
    q = _query_with_pop(rng, 40)
    assert lib.search(q, 10) == oracle_topk(w, q[None], 10)[0]
    assert lib.last_kernel == "single-query HBM scan"


@pytest.mark.parametrize("copy", [0, 1])
@pytest.mark.parametrize("bpl,warps,stages", [(2, 1, 1), (2, 4, 2), (2, 8, 1), (2, 8, 4), (2, 16, 2), (1, 16, 2),
                                              (1, 12, 2), (1, 3, 4)])
def test_plane_scan_ring_shapes(bpl, warps, stages, copy, monkeypatch):
    """Blocks per lane x warps per CTA x ring stages x copy engine (bulk copies
    or cp.async); wide lists fold warps to keep >= 2 stages."""
    monkeypatch.setenv("FPS_PQ_BPL", str(bpl))
    monkeypatch.setenv("FPS_PQ_COPY", str(copy))
    monkeypatch.setenv("FPS_PQ_WARPS", str(warps))
    monkeypatch.setenv("FPS_PQ_STAGES", str(stages))
    seed = 77
    w = orc.generate_words(synth.seed_key(seed), synth.beta_thresholds(seed), 0, 300_001)
    lib = Library.from_words(w)
    rng = np.random.default_rng(warps * 10 + stages)
    for pop in (20, 60, 83, 100):
        q = _query_with_pop(rng, pop)
        for k in (10, 1024):
            exp = oracle_topk(w, q[None], k)[0]
            assert lib.search(q, k) == exp, (warps, stages, pop, k)
            assert _dev_topk(lib, q[None], k) == exp, (warps, stages, pop, k)


def test_plane_copy_follows_entry_writes():
    """The plane copies are derived from the entries: a write invalidates them."""
    seed = 31
    w = orc.generate_words(synth.seed_key(seed), synth.beta_thresholds(seed), 0, 50_000)
    lib = Library.from_words(w)
    q = w[123].copy()
    assert lib.search(q, 3) == oracle_topk(w, q[None], 3)[0]
    qq = np.stack([q, w[7]])
    lib.search_batch(qq, 3)  # builds the bit-slice tiles too
    lib.write_entries(np.array([40_000], dtype=np.uint64), q[None])
    w[40_000] = q
    assert lib.search(q, 3) == oracle_topk(w, q[None], 3)[0]
    res = lib.search_batch(qq, 3)
    exp = oracle_topk(w, qq, 3)
    assert [res.hits(0), res.hits(1)] == exp
    assert (40_000, 0) in res.hits(0)


def test_plane_scan_not_used_with_pad_bits():
    rec = np.zeros((3000, 4), dtype=np.uint64)
    rec[:, 0] = np.arange(1, 3001)
    rec[5, 3] = np.uint64(1) << np.uint64(45)
    lib = Library.from_records(rec)
    assert lib.search(np.zeros(3, dtype=np.uint64), 3000)[-1] == (5, 1)
    assert lib.last_kernel == "single-query HBM scan"


@pytest.mark.parametrize("refresh", [1, 3, 8])
def test_plane_scan_bound_refresh_periods(refresh, monkeypatch):
    """The global bound read every `refresh` steps (long scans: 8)."""
    monkeypatch.setenv("FPS_PQ_REFRESH", str(refresh))
    seed = 1234
    w = orc.generate_words(synth.seed_key(seed), synth.beta_thresholds(seed), 0, 400_003)
    lib = Library.from_words(w)
    rng = np.random.default_rng(refresh)
    for pop in (30, 45):
        q = _query_with_pop(rng, pop)
        for k in (10, 100):
            assert lib.search(q, k) == oracle_topk(w, q[None], k)[0], (refresh, pop, k)


# ---------------------------------------------------------------- popcount-sorted plane copy
@pytest.mark.parametrize("n", [1, 2047, 2049, 100_003, 300_001])
def test_sorted_plane_scan_sizes_and_densities(n, monkeypatch):
    """FPS_PQ_SORTED=1: planes ordered by popcount (uniform-|a| steps skip the
    popcount planes, out-of-range steps are skipped, ties at the own k-th
    distance resolved by index)."""
    monkeypatch.setenv("FPS_PQ_SORTED", "1")
    seed = 4000 + n
    w = orc.generate_words(synth.seed_key(seed), synth.beta_thresholds(seed), 0, n)
    lib = Library.from_words(w)
    rng = np.random.default_rng(n + 1)
    for pop in (0, 9, 38, 84, 140):
        q = _query_with_pop(rng, pop)
        for k in (1, 10, 100, 1024):
            exp = oracle_topk(w, q[None], k)[0]
            assert lib.search(q, k) == exp, (n, pop, k)
            assert _dev_topk(lib, q[None], k) == exp, (n, pop, k)
    # library entries as queries (planted-like: distance 0 exists)
    for i in (0, n // 3, n - 1):
        q = w[i].copy()
        assert lib.search(q, 10) == oracle_topk(w, q[None], 10)[0]


@pytest.mark.parametrize("bpl,warps", [(2, 8), (1, 16), (2, 3)])
def test_sorted_plane_scan_ties_and_adversarial(bpl, warps, monkeypatch):
    monkeypatch.setenv("FPS_PQ_SORTED", "1")
    monkeypatch.setenv("FPS_PQ_BPL", str(bpl))
    monkeypatch.setenv("FPS_PQ_WARPS", str(warps))
    # every entry identical: the first k indices, ties overflow the scratch
    w = np.tile(np.array([[0x1234, 0x5678, 0x9]], dtype=np.uint64), (200_000, 1))
    lib = Library.from_words(w)
    for k in (1, 10, 33, 100, 1024):
        assert lib.search(np.array([0x1234, 0x5678, 0x8], dtype=np.uint64), k) == [(i, 1) for i in range(k)]
    # two popcount classes interleaved by index, equal distances across classes
    rng = np.random.default_rng(5)
    base = np.array([0x0F0F, 0x3, 0x0], dtype=np.uint64)
    w2 = np.tile(base, (150_000, 1))
    flip = rng.integers(0, 2, 150_000).astype(bool)
    w2[flip, 1] ^= np.uint64(0x4)          # one extra key: popcount +1, distance 1
    w2[~flip, 0] ^= np.uint64(0x1)         # one key fewer: popcount -1, distance 1
    lib2 = Library.from_words(w2)
    for k in (5, 64, 500):
        assert lib2.search(base, k) == oracle_topk(w2, base[None], k)[0]
    # distances falling with the index
    n = 120_000
    w3 = np.zeros((n, 3), dtype=np.uint64)
    bits = 166 - (np.arange(n) * 166 // n)
    for i, b in enumerate(bits):
        v = (1 << int(b)) - 1
        w3[i] = (v & (2**64 - 1), (v >> 64) & (2**64 - 1), v >> 128)
    lib3 = Library.from_words(w3)
    for k in (10, 100, 500):
        assert lib3.search(np.zeros(3, dtype=np.uint64), k) == oracle_topk(w3, np.zeros((1, 3), np.uint64), k)[0]


def test_sorted_plane_scan_config_shapes(monkeypatch):
    """C1/C2-shaped runs (planted near-duplicates: small bounds prune popcount classes)."""
    monkeypatch.setenv("FPS_PQ_SORTED", "1")
    for wl, n in (("c1", 1_000_000), ("c2", 2_000_000)):
        plan = synth.make_plan(wl, n=n, planted_per_query=200 if wl == "c2" else None)
        lib, q = synth.build_library(plan)
        w = lib.words_host()
        assert lib.search(q[0], plan.k) == oracle_topk(w, q[:1], plan.k)[0]
        assert _dev_topk(lib, q[:1], plan.k) == oracle_topk(w, q[:1], plan.k)[0]


# ---------------------------------------------------------------- tensor-core multi-query path
MMA_KINDS = ["fp4x", "i8", "fp4"]


@pytest.mark.parametrize("kind", MMA_KINDS)
@pytest.mark.parametrize("n", [1, 127, 128, 129, 70_001, 300_007])
def test_mma_multi_query_vs_oracle(n, kind, monkeypatch):
    """tcgen05 MMA path (FPS_MMA=1), every operand kind (fp4 from the operand
    copy, int8 and fp4 expanded in the kernel): every pair within the seeded
    bound collected, select keeps the k smallest (distance, index); several
    query chunks, columns ordered by bound, tails of 128-entry tiles."""
    monkeypatch.setenv("FPS_MMA", "1")
    monkeypatch.setenv("FPS_MMA_KIND", kind)
    seed = 600 + n
    w = orc.generate_words(synth.seed_key(seed), synth.beta_thresholds(seed), 0, n)
    lib = Library.from_words(w)
    rng = np.random.default_rng(n)
    # accumulators of 64 / 128 / 208-256 columns, 1-3 chunks (fp4: 230 and 470
    # queries run 240-column chunks, 257 and 600 208-column ones)
    for Q in (2, 100, 230, 257, 470, 600):
        q = w[rng.integers(0, n, Q)].copy()
        q[:, 0] ^= rng.integers(0, 2**24, Q).astype(np.uint64) << np.uint64(1)
        q[Q // 2] = _query_with_pop(rng, 120)  # a dense query
        for k in (1, 10, 100):
            res = lib.search_batch(q, k)
            exp = oracle_topk(w, q, k)
            for i in range(Q):
                assert res.hits(i) == exp[i], (n, Q, k, i)
            if n >= 128:
                assert lib.last_kernel == "tensor-core multi-query scan" and lib.last_mma_kind == kind
                # no candidate list overflowed (the exact fallback pass would hide
                # a kernel that reports spurious hits)
                assert not lib.mma_overflowed, (n, Q, k)


def test_mma_candidate_overflow_falls_back(monkeypatch):
    """Every entry ties (all within the seed bound): the candidate lists
    overflow and the call is recomputed by the bit-sliced kernel."""
    monkeypatch.setenv("FPS_MMA", "1")
    w = np.tile(np.array([[0x1234, 0x5678, 0x9]], dtype=np.uint64), (300_000, 1))
    lib = Library.from_words(w)
    q = np.tile(np.array([[0x1234, 0x5678, 0x8]], dtype=np.uint64), (300, 1))
    res = lib.search_batch(q, 10)
    for i in range(300):
        assert res.hits(i) == [(j, 1) for j in range(10)]
    assert lib.mma_overflowed


def test_mma_pad_bits_counted():
    """The MMA path covers all 192 bits: FPS1 pad bits count like the reference."""
    rec = np.zeros((5000, 4), dtype=np.uint64)
    rec[:, 0] = np.arange(1, 5001)
    rng = np.random.default_rng(3)
    rec[:, 1] = rng.integers(0, 2**63, 5000, dtype=np.uint64)
    rec[17, 3] = np.uint64(0xF) << np.uint64(44)
    lib = Library.from_records(rec)
    w = rec[:, 1:].copy()
    q = w[rng.integers(0, 5000, 256)].copy()
    q[0] = w[17] & ~(np.uint64(0xF) << np.uint64(44))
    q[:, 2] &= np.uint64((1 << 38) - 1)
    import os
    os.environ["FPS_MMA"] = "1"
    try:
        res = lib.search_batch(q, 5)
    finally:
        del os.environ["FPS_MMA"]
    exp = oracle_topk(w, q, 5)
    for i in range(256):
        assert res.hits(i) == exp[i]


@pytest.mark.parametrize("kind", MMA_KINDS)
@pytest.mark.parametrize("n", [127, 129, 70_001, 300_007])
def test_mma_range_vs_oracle(n, kind, monkeypatch):
    """Range search on the tensor cores (FPS_MMA=1): the radius is the bound,
    every pair with d <= r is emitted; 64 / 128 / 256-column accumulators,
    several chunks, tails of library tiles, a dense query; every operand kind."""
    monkeypatch.setenv("FPS_MMA", "1")
    monkeypatch.setenv("FPS_MMA_KIND", kind)
    seed = 700 + n
    w = orc.generate_words(synth.seed_key(seed), synth.beta_thresholds(seed), 0, n)
    lib = Library.from_words(w)
    rng = np.random.default_rng(n)
    for Q in (2, 64, 65, 130, 300):
        q = w[rng.integers(0, n, Q)].copy()
        q[:, 1] ^= rng.integers(0, 8, Q).astype(np.uint64)
        q[Q // 2] = _query_with_pop(rng, 120)
        for radius in (0, 6, 40):
            r = lib.range_search(q, radius)
            assert np.array_equal(r.rows(), orc.c_range(w, q, radius)), (n, Q, radius)


def test_mma_range_per_query_radius_and_overflow_retry(monkeypatch):
    """Per-query radii on the tensor-core range path; > 1 M hits: the first
    pass overflows the output and the call is re-run with a larger buffer."""
    monkeypatch.setenv("FPS_MMA", "1")
    w = orc.generate_words(3, np.full(166, 2**31, np.uint64), 0, 400_000)
    q = w[:40].copy()
    radii = np.zeros(40, dtype=np.uint8)
    radii[:5] = [0, 95, 90, 80, 166]
    radii[5:] = 50
    lib = Library.from_words(w)
    r = lib.range_search(q, radii)
    exp = np.concatenate([orc.c_range(w, q[i:i + 1], int(radii[i])) + np.array([i, 0, 0]) for i in range(40)])
    assert len(r) > 1 << 20
    assert np.array_equal(r.rows(), exp)


def test_mma_range_default_dispatch_config_shape():
    """C5-shaped calls (radius 6, planted near-duplicates): 40 queries take
    the bit-sliced kernel, 64 the fp4 operand-copy tensor-core kernel (two
    epilogue groups), 256 the int8 tensor-core kernel; all match the oracle."""
    plan = synth.make_plan("c5", n=1_000_000, planted_per_query=300)
    lib, q = synth.build_library(plan)
    w = lib.words_host()
    r = lib.range_search(q[:40], plan.radius)
    assert lib.last_kernel == "bit-sliced multi-query scan"
    assert np.array_equal(r.rows(), orc.c_range(w, q[:40], plan.radius))
    r = lib.range_search(q, plan.radius)
    assert lib.last_kernel == "tensor-core multi-query scan" and lib.last_mma_kind == "fp4x"
    assert np.array_equal(r.rows(), orc.c_range(w, q, plan.radius))
    q4 = np.concatenate([q, q ^ np.uint64(1), q ^ np.uint64(2), q ^ np.uint64(4)])
    r = lib.range_search(q4, plan.radius)
    assert lib.last_kernel == "tensor-core multi-query scan" and lib.last_mma_kind == "i8"
    assert np.array_equal(r.rows(), orc.c_range(w, q4, plan.radius))


@pytest.mark.parametrize("Q", [20, 40, 300])
def test_bitslice_all_ties_buffer_capacity(Q, monkeypatch):
    """Every entry at the same distance from every query: each warp step of
    the bit-sliced kernel passes a whole 2,048-entry tile after its buffer was
    compacted to k, so the per-(warp, query) buffer needs k + one tile (1, 2
    and 4 queries per warp)."""
    monkeypatch.setenv("FPS_MMA", "0")
    w = np.tile(np.array([[0x1234, 0x5678, 0x9]], dtype=np.uint64), (300_000, 1))
    lib = Library.from_words(w)
    q = np.tile(np.array([[0x1234, 0x5678, 0x8]], dtype=np.uint64), (Q, 1))
    for k in (10, 100):
        res = lib.search_batch(q, k)
        assert lib.last_kernel == "bit-sliced multi-query scan"
        for i in range(Q):
            assert res.hits(i) == [(j, 1) for j in range(k)], (Q, k, i)


@pytest.mark.parametrize("prefix_log2", [12, 14, "11,13,15", "0", "12,12,9,16"])
def test_mma_two_pass_prefix_bound(prefix_log2, monkeypatch):
    """Tensor-core top-k in range passes (each pass scans the entries after
    the previous one, starting from the exact top-k so far, carried into its
    candidate lists), forced on a small library: every pair within each
    pass's bound is collected and no entry is read twice, so the result is the
    exact top-k -- with one prefix range, several, none, or a malformed list."""
    monkeypatch.setenv("FPS_MMA", "1")
    monkeypatch.setenv("FPS_MMA_PREFIX", str(prefix_log2))
    monkeypatch.setenv("FPS_MMA_SEED", "10")
    n = 300_007
    w = orc.generate_words(synth.seed_key(77), synth.beta_thresholds(77), 0, n)
    lib = Library.from_words(w)
    rng = np.random.default_rng(5)
    q = w[rng.integers(0, n, 300)].copy()
    q[:, 0] ^= rng.integers(0, 2**20, 300).astype(np.uint64) << np.uint64(1)
    q[7] = _query_with_pop(rng, 150)
    for k in (1, 10, 64):
        res = lib.search_batch(q, k)
        exp = oracle_topk(w, q, k)
        for i in range(300):
            assert res.hits(i) == exp[i], (prefix_log2, k, i)


def test_fp4_operand_copy_rebuilt_after_writes_and_released():
    """The fp4 operand copy (96 B/entry, built by the first fp4x call) follows
    entry writes (invalidated, rebuilt on the next call) and fps_release_derived;
    the 64-query range and top-k results always equal the oracle's."""
    seed = 4711
    n = 200_003
    w = orc.generate_words(synth.seed_key(seed), synth.beta_thresholds(seed), 0, n)
    lib = Library.from_words(w)
    rng = np.random.default_rng(seed)
    q = w[rng.integers(0, n, 64)].copy()
    q[:, 1] ^= np.uint64(0b101)
    r = lib.range_search(q, 10)
    assert lib.last_mma_kind == "fp4x"
    assert np.array_equal(r.rows(), orc.c_range(w, q, 10))
    before = lib.memory()["derived_bytes"]
    assert before >= (n + 127) // 128 * 12288
    # rewrite 1,000 entries as exact copies of queries: new distance-0 hits
    idx = rng.choice(n, 1000, replace=False).astype(np.uint64)
    w2 = w.copy()
    w2[idx.astype(np.int64)] = q[rng.integers(0, 64, 1000)]
    lib.write_entries(idx, w2[idx.astype(np.int64)])
    r = lib.range_search(q, 10)
    assert lib.last_mma_kind == "fp4x"
    assert np.array_equal(r.rows(), orc.c_range(w2, q, 10))
    res = lib.search_batch(q, 10)
    exp = oracle_topk(w2, q, 10)
    for i in range(64):
        assert res.hits(i) == exp[i], i
    lib.release_derived()
    assert lib.memory()["derived_bytes"] == 0
    r = lib.range_search(q, 10)
    assert np.array_equal(r.rows(), orc.c_range(w2, q, 10))
    lib.close()
