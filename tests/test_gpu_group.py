"""Multi-device library (fps_group_*, LibraryGroup) and the round-2 C-ABI
changes, vs the single-library path and the C oracle (needs a B200).

One GPU is available, so groups are built with repeated devices
(``devices=[0, 0, 0, 0]``: four shards, four streams, one root): every shard
is a separate fps_lib and the root's merge kernel reads the other shards'
result blocks exactly as it reads peer HBM on an 8-GPU box (no kernel waits
on another: the root stream waits on per-shard events). The NCCL gather
needs distinct devices; it is exercised with a one-shard group (a self
send/recv through libnccl) and rejected for shared devices.

Reference semantics: merge_topk over contiguous split_sizes shards
(scan.py:225-236, :256-287; libstore.py:174-179).
"""

import numpy as np
import pytest

import fps_oracle as orc
from paper_1906_06170_b200 import scan, synth
from paper_1906_06170_b200.library import Library, LibraryGroup, load_library

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _device():
    import torch

    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    yield
    scan.clear_cache()


def oracle_lists(w, q, k):
    idx, dist, cnt = orc.c_topk(w, q, k)
    return [list(zip(idx[i, :cnt[i]].tolist(), dist[i, :cnt[i]].tolist())) for i in range(len(q))]


@pytest.fixture(scope="module")
def mid():
    """A 1.5 M-entry C1-distribution library (host words) with 300 queries."""
    plan = synth.make_plan("c1", seed=424242, n=1_500_000)
    w = orc.generate_words_parallel(plan.seed_key, plan.thresholds, 0, plan.n)
    rng = np.random.default_rng(5)
    q = w[rng.integers(0, len(w), 300)].copy()
    q[:, 0] ^= np.uint64(0b10110)
    q[:, 2] ^= np.uint64(1 << 7)
    return w, q


@pytest.mark.parametrize("gather", ["p2p", "copy"])
def test_group_topk_equals_single(mid, gather):
    w, q = mid
    single = Library.from_words(w)
    grp = load_library(w, devices=[0, 0, 0], gather=gather)
    assert isinstance(grp, LibraryGroup) and grp.gather == gather
    assert [s.n for s in grp.shards] == [500_000] * 3
    assert [s.index_base for s in grp.shards] == [0, 500_000, 1_000_000]
    for Q, k in ((1, 10), (1, 100), (7, 10), (300, 10), (5, 1025)):
        a = single.search_batch(q[:Q], k)
        b = grp.search_batch(q[:Q], k)
        for i in range(Q):
            assert b.hits(i) == a.hits(i), (gather, Q, k, i)
    exp = oracle_lists(w, q[:7], 10)
    got = grp.search_batch(q[:7], 10)
    assert [got.hits(i) for i in range(7)] == exp
    grp.close()
    single.close()


def test_group_uneven_and_empty_shards():
    """split_sizes with more shards than a small library fills: sizes differ
    by at most one, trailing shards may be empty."""
    rng = np.random.default_rng(9)
    w = rng.integers(0, 1 << 63, size=(5, 3), dtype=np.uint64)
    w[:, 2] &= np.uint64((1 << 38) - 1)
    grp = LibraryGroup.from_words(w, [0] * 8)
    assert [s.n for s in grp.shards] == [1, 1, 1, 1, 1, 0, 0, 0]
    got = grp.search_batch(w[:3], 10)
    exp = oracle_lists(w, w[:3], 10)
    assert [got.hits(i) for i in range(3)] == exp
    assert np.array_equal(grp.read_entries(), w)
    grp.close()


def test_group_range_and_min(mid):
    w, q = mid
    single = Library.from_words(w)
    grp = LibraryGroup.from_words(w, [0, 0, 0, 0])
    r1 = single.range_search(q[:64], 30)
    r2 = grp.range_search(q[:64], 30)
    assert len(r1) > 64
    assert np.array_equal(r1.rows(), r2.rows())
    assert np.array_equal(r2.rows(), orc.c_range(w, q[:64], 30))
    for Q, k in ((3, 30), (40, 100), (300, 10), (4, 4000)):
        assert grp.search_min(q[:Q], k) == single.search_min(q[:Q], k), (Q, k)
    grp.close()
    single.close()


def test_group_async_device_api(mid):
    import torch

    w, q = mid
    grp = LibraryGroup.from_words(w, [0, 0])
    Q, k = 256, 10
    grp.topk_prepare(Q, k)
    dq = torch.from_numpy(q[:Q].view(np.int64).copy()).cuda()
    keys = torch.empty((Q, k), dtype=torch.int64, device="cuda")
    cnt = torch.empty((Q,), dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        grp.topk_async(dq, Q, k, keys, cnt, s)
    torch.cuda.synchronize()
    from paper_1906_06170_b200.library import keys_to_hits

    got = keys_to_hits(keys.cpu().numpy().view(np.uint64), cnt.cpu().numpy().view(np.uint32))
    exp = oracle_lists(w, q[:Q], k)
    for i in range(Q):
        assert got.hits(i) == exp[i], i
    grp.close()


def test_group_nccl_single_shard_and_rejects_shared_device(mid):
    w, q = mid
    try:
        grp = LibraryGroup.from_words(w[:200_000], [0], gather="nccl")
    except Exception as exc:  # libnccl missing on this box would be an environment problem
        pytest.fail(f"NCCL group: {exc}")
    assert grp.gather == "nccl"
    exp = oracle_lists(w[:200_000], q[:5], 10)
    got = grp.search_batch(q[:5], 10)
    assert [got.hits(i) for i in range(5)] == exp
    r = grp.range_search(q[:5], 10)
    assert np.array_equal(r.rows(), orc.c_range(w[:200_000], q[:5], 10))
    grp.close()
    with pytest.raises(ValueError, match="NCCL"):
        LibraryGroup.from_words(w[:1000], [0, 0], gather="nccl")


def test_group_from_fps1_and_scan_devices(tmp_path, monkeypatch):
    rng = np.random.default_rng(11)
    n = 300_001
    plan = synth.make_plan("c1", seed=7, n=n)
    w = orc.generate_words_parallel(plan.seed_key, plan.thresholds, 0, n)
    cids = rng.permutation(np.arange(10, 10 + n, dtype=np.uint64))
    mpath = orc.write_fps1_library(tmp_path / "lib", w, shard_count=3, cids=cids)
    from paper_1906_06170_b200 import libstore

    manifest = libstore.load_manifest(mpath.parent)
    grp = LibraryGroup.from_fps1([s.path for s in manifest.shards], [0, 0, 0, 0])
    single = Library.from_fps1([s.path for s in manifest.shards])
    assert np.array_equal(grp.cids, single.cids)
    assert np.array_equal(grp.cids, cids)
    q = w[[5, 77, 123456]].copy()
    q[:, 1] ^= np.uint64(3)
    a, b = single.search_batch(q, 25), grp.search_batch(q, 25)
    for i in range(3):
        assert a.hits(i) == b.hits(i)
    grp.close()
    single.close()
    # the drop-in search over a manifest on a 3-shard group == on one device
    from paper_1906_06170_b200.fingerprint import Fingerprint

    fq = Fingerprint(tuple(int(x) for x in q[0]))
    scan.clear_cache()
    one = scan.search(manifest, fq, scan.SearchParams(n=40))
    scan.clear_cache()
    monkeypatch.setenv("FPS_DEVICES", "0,0,0")
    many = scan.search(manifest, fq, scan.SearchParams(n=40))
    multi = scan.batch_search(manifest, [fq, Fingerprint(tuple(int(x) for x in q[1]))], scan.SearchParams(n=40))
    monkeypatch.delenv("FPS_DEVICES")
    scan.clear_cache()
    assert one == many
    assert multi == scan.batch_search(manifest, [fq, Fingerprint(tuple(int(x) for x in q[1]))],
                                      scan.SearchParams(n=40))
    scan.clear_cache()


def test_group_c3_full_size_equals_single():
    """The verdict's bar: C3 (95,417,114 entries) as four shards on one B200
    equals the single-library answer, for the single query and a batch."""
    plan = synth.make_plan("c3")
    single, q = synth.build_library(plan)
    exp = single.search(q[0], plan.k)
    words_rows = single.read_entries(0, 1000)
    single.close()
    grp, q2 = synth.build_library(plan, devices=[0, 0, 0, 0])
    assert np.array_equal(q, q2)
    assert np.array_equal(grp.read_entries(0, 1000), words_rows)
    assert grp.search(q[0], plan.k) == exp
    assert grp.last_kernel == "single-query plane scan"
    grp.close()


# ------------------------------------------------------- round-2 C-ABI changes
def test_tensor_core_overflow_falls_back_on_device():
    """All-identical entries: every (query, entry) pair is within the bound, so
    the tensor-core candidate lists overflow; the device flag gates the exact
    POPC pass, with no host synchronisation in the call."""
    n = 300_000
    row = np.array([0x00FF00FF00FF00FF, 0x1234, 0x5], dtype=np.uint64)
    w = np.tile(row, (n, 1))
    lib = Library.from_words(w)
    rng = np.random.default_rng(2)
    q = np.tile(row, (200, 1))
    q[:, 1] ^= rng.integers(0, 1 << 20, size=200, dtype=np.uint64)
    res = lib.search_batch(q, 10)
    assert lib.last_kernel == "tensor-core multi-query scan"
    exp = oracle_lists(w, q, 10)
    for i in range(200):
        assert res.hits(i) == exp[i], i
        assert [h[0] for h in res.hits(i)] == list(range(10))
    lib.close()


def test_tensor_core_path_is_graph_capturable(mid):
    import torch

    w, q = mid
    lib = Library.from_words(w)
    Q, k = 256, 10
    lib.topk_prepare(Q, k)
    dq = torch.from_numpy(q[:Q].view(np.int64).copy()).cuda()
    keys = torch.empty((Q, k), dtype=torch.int64, device="cuda")
    cnt = torch.empty((Q,), dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        lib.topk_async(dq, Q, k, keys, cnt, s.cuda_stream)  # warm (derived copies, scratch)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        lib.topk_async(dq, Q, k, keys, cnt, s.cuda_stream)
    keys.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert lib.last_kernel == "tensor-core multi-query scan"
    from paper_1906_06170_b200.library import keys_to_hits

    got = keys_to_hits(keys.cpu().numpy().view(np.uint64), cnt.cpu().numpy().view(np.uint32))
    exp = oracle_lists(w, q[:Q], k)
    for i in range(Q):
        assert got.hits(i) == exp[i], i
    lib.close()


def test_topk_async_large_k(mid):
    import torch

    w, q = mid
    lib = Library.from_words(w[:400_000])
    Q, k = 3, 2500
    dq = torch.from_numpy(q[:Q].view(np.int64).copy()).cuda()
    keys = torch.empty((Q, k), dtype=torch.int64, device="cuda")
    cnt = torch.empty((Q,), dtype=torch.int32, device="cuda")
    lib.topk_async(dq, Q, k, keys, cnt, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    from paper_1906_06170_b200.library import keys_to_hits

    got = keys_to_hits(keys.cpu().numpy().view(np.uint64), cnt.cpu().numpy().view(np.uint32))
    exp = oracle_lists(w[:400_000], q[:Q], k)
    for i in range(Q):
        assert got.hits(i) == exp[i]
    lib.close()


@pytest.mark.parametrize("k", [1025, 4000])
def test_batch_search_large_n(mid, k):
    """batch_search accepts any n >= 1 (scan.py:82-84, :306-318)."""
    w, q = mid
    lib = Library.from_words(w[:300_000])
    for Q in (1, 2, 9):
        got = lib.search_min(q[:Q], k)
        exp = orc.batch_min_topk(w[:300_000], q[:Q], k)
        assert got == exp, (Q, k)
    lib.close()


def test_open_close_does_not_leak_hbm(mid):
    """Every buffer a handle allocates (library, derived plane copies, scratch)
    is returned by fps_close."""
    import torch

    w, q = mid
    torch.cuda.synchronize()

    def cycle():
        lib = Library.from_words(w)
        lib.search(q[0], 10)            # plane-major copy + single-query scratch
        lib.search_batch(q[:40], 10)    # bit-plane copy + multi-query scratch
        lib.search_batch(q[:256], 10)   # tensor-core scratch
        lib.range_search(q[:4], 8)
        lib.read_entries(0, 1000)
        lib.write_entries(np.array([3], np.uint64), w[4:5])
        m = lib.memory()
        assert m["derived_bytes"] == 0 or m["derived_bytes"] > 0
        lib.close()

    cycle()
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(4):
        cycle()
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 < (64 << 20), (free0, free1)


def test_memory_report_and_release(mid):
    w, q = mid
    lib = Library.from_words(w)
    m0 = lib.memory()
    assert m0["library_bytes"] >= 21 * len(w) and m0["derived_bytes"] == 0
    lib.search(q[0], 10)
    m1 = lib.memory()
    assert m1["derived_bytes"] > 20 * len(w) and m1["derived_build_ms"] > 0
    lib.release_derived()
    assert lib.memory()["derived_bytes"] == 0
    assert lib.search(q[0], 10) == oracle_lists(w, q[:1], 10)[0]  # rebuilt on demand
    lib.close()


def test_merge_runs_async_equals_sorted_union():
    """fps_merge_runs_async (the torchrun range gather's rank-0 merge):
    G sorted runs of unique keys, some empty, merged by rank on the device."""
    import torch

    from paper_1906_06170_b200 import distributed as D

    rng = np.random.default_rng(11)
    for G in (1, 2, 3, 8, 32):
        pool = rng.choice(1 << 50, size=G * 700, replace=False).astype(np.int64)
        cuts = np.sort(rng.integers(0, len(pool), G - 1))
        runs_h = [np.sort(p) for p in np.split(pool, cuts)]
        if G > 2:
            runs_h[1] = runs_h[1][:0]  # an empty run
        runs = [torch.from_numpy(r.copy()).cuda() for r in runs_h]
        got = D.device_merge_runs(runs)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), np.sort(np.concatenate(runs_h)))


def test_merge_packed_async_equals_merge_topk():
    """fps_merge_packed_async (the torchrun top-k gather's rank-0 merge): G
    per-rank blocks of Q x k sorted keys + Q u32 counts in one buffer, merged
    with one kernel; equals merge_topk over the rank lists (scan.py:225-236)."""
    import torch

    from paper_1906_06170_b200 import _native as N
    from paper_1906_06170_b200 import distributed as D

    rng = np.random.default_rng(5)
    for G, Q, k in ((2, 1, 10), (3, 7, 100), (8, 33, 17), (32, 2, 5)):
        pool = rng.choice(1 << 48, size=G * Q * k, replace=False).astype(np.int64).reshape(G, Q, k)
        cnts = rng.integers(0, k + 1, size=(G, Q))
        L = Q * k + Q
        buf = np.zeros((G, L), dtype=np.int64)
        for g in range(G):
            keys = np.full((Q, k), -1, dtype=np.int64)
            for q in range(Q):
                keys[q, :cnts[g, q]] = np.sort(pool[g, q, :cnts[g, q]])
            buf[g, :Q * k] = keys.reshape(-1)
            buf[g, Q * k:].view(np.int32)[:Q] = cnts[g]
        dbuf = torch.from_numpy(buf).cuda()
        out_k = torch.empty((Q, k), dtype=torch.int64, device="cuda")
        out_c = torch.empty((Q,), dtype=torch.int32, device="cuda")
        N.check(N.load().fps_merge_packed_async(dbuf.data_ptr(), L * 8, G, Q, k, out_k.data_ptr(), out_c.data_ptr(),
                                                torch.cuda.current_stream().cuda_stream), "fps_merge_packed_async")
        torch.cuda.synchronize()
        gk, gc = out_k.cpu().numpy(), out_c.cpu().numpy()
        for q in range(Q):
            allk = np.sort(np.concatenate([pool[g, q, :cnts[g, q]] for g in range(G)]))[:k]
            assert gc[q] == len(allk)
            assert np.array_equal(gk[q, :len(allk)], allk)
    # the packed block helper writes the same layout
    blk, kv, cv = D.packed_block(3, 4, "cuda")
    assert kv.data_ptr() == blk.data_ptr() and cv.data_ptr() == blk.data_ptr() + 3 * 4 * 8
