"""Full-size parity: every BASELINE.json config at its real size, CUDA path vs
the C oracle (oracle/fps_oracle.c, multi-threaded) on the same seeded library.

The library is generated on the GPU and copied back once; the oracle scans the
host copy. Bit-exact equality of (index, distance) lists / range triples, plus
size-independent properties (sortedness, recomputed distances, planted
near-duplicates found at their flip counts, shard-merge associativity).
"""

import numpy as np
import pytest

import fps_oracle as orc
from paper_1906_06170_b200 import synth
from paper_1906_06170_b200.library import Library, keys_to_hits, merge_async

pytestmark = pytest.mark.gpu

_cache = {}


def full(name):
    if name not in _cache:
        _cache.clear()
        plan = synth.make_plan(name)
        lib, q = synth.build_library(plan)
        _cache[name] = (plan, lib, q, lib.words_host())
    return _cache[name]


def oracle_lists(w, q, k):
    idx, dist, cnt = orc.c_topk(w, q, k)
    return [list(zip(idx[i, :cnt[i]].tolist(), dist[i, :cnt[i]].tolist())) for i in range(len(q))]


def recomputed(w, q, hits):
    ids = np.array([i for i, _ in hits], dtype=np.int64)
    return orc.distances_one(w[ids], q).tolist() == [d for _, d in hits]


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_single_query_full_size(name):
    plan, lib, q, w = full(name)
    got = lib.search(q[0], plan.k)
    assert got == oracle_lists(w, q[:1], plan.k)[0]
    assert got == sorted(got, key=lambda t: (t[1], t[0]))
    assert recomputed(w, q[0], got)
    if name == "c2":
        # k = 100 of the 1,000 planted near-duplicates (0-4 flips): all at distance 0
        planted0 = sorted(int(i) for i, f in zip(plan.planted_idx, plan.planted_flips) if len(f) == 0)
        assert [i for i, _ in got] == planted0[:100]


def test_config4_full_size(monkeypatch):
    plan, lib, q, w = full("c4")
    res = lib.search_batch(q, plan.k)
    assert lib.last_kernel == "tensor-core multi-query scan" and lib.last_mma_kind == "fp4x"
    assert not lib.mma_overflowed
    exp = oracle_lists(w, q, plan.k)
    for i in range(plan.Q):
        assert res.hits(i) == exp[i], i
        # the query's source entry is within its flip count
        assert res.hits(i)[0][1] <= len(plan.query_flips[i])
    # 240 queries: one 240-column fp4 chunk
    res240 = lib.search_batch(q[:240], plan.k)
    assert not lib.mma_overflowed
    for i in range(240):
        assert res240.hits(i) == exp[i], i
    # the bit-sliced kernel (FPS_MMA=0) gives the same lists
    monkeypatch.setenv("FPS_MMA", "0")
    res2 = lib.search_batch(q, plan.k)
    assert lib.last_kernel == "bit-sliced multi-query scan"
    for i in range(plan.Q):
        assert res2.hits(i) == exp[i], i


def test_config5_full_size():
    plan, lib, q, w = full("c5")
    r = lib.range_search(q, plan.radius)
    assert lib.last_kernel == "tensor-core multi-query scan" and lib.last_mma_kind == "fp4x"
    rows = r.rows()
    assert np.array_equal(rows, orc.c_range(w, q, plan.radius))
    # every planted near-duplicate (0-6 flips) is present at its flip count
    got = set(map(tuple, rows.tolist()))
    for i, qi, f in zip(plan.planted_idx, plan.planted_query, plan.planted_flips):
        assert (int(qi), int(i), len(f)) in got
    assert len(rows) >= 640_064
    # the bit-sliced kernel (FPS_MMA=0) and the int8 tensor-core kernel give
    # the same triples
    import os
    for env, kernel in ((("FPS_MMA", "0"),), "bit-sliced multi-query scan"), \
                       ((("FPS_MMA", "1"), ("FPS_MMA_KIND", "i8")), "tensor-core multi-query scan"):
        for key, v in env:
            os.environ[key] = v
        try:
            r2 = lib.range_search(q, plan.radius)
            assert lib.last_kernel == kernel
        finally:
            for key, _ in env:
                del os.environ[key]
        assert np.array_equal(r2.rows(), rows)


def test_config3_sharded_merge_full_size():
    """C3 split into 8 contiguous shards (the 8-GPU layout) on one GPU, merged
    by the device merge kernel: identical to the single-library answer."""
    import torch

    plan, lib, q, w = full("c3")
    G, k = 8, plan.k
    offs = [0]
    for s in orc.split_sizes(plan.n, G):
        offs.append(offs[-1] + s)
    dq = torch.from_numpy(q.view(np.int64)).cuda()
    keys = torch.empty((G, 1, k), dtype=torch.int64, device="cuda")
    cnt = torch.empty((G, 1), dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    for g in range(G):
        part = Library.from_words(w[offs[g]:offs[g + 1]], index_base=offs[g])
        part.topk_prepare(1, k)
        part.topk_async(dq, 1, k, keys[g], cnt[g], stream)
        torch.cuda.synchronize()
        part.close()
    out_k = torch.empty((1, k), dtype=torch.int64, device="cuda")
    out_c = torch.empty((1,), dtype=torch.int32, device="cuda")
    merge_async(keys, cnt, G, 1, k, out_k, out_c, stream)
    torch.cuda.synchronize()
    res = keys_to_hits(out_k.cpu().numpy().view(np.uint64), out_c.cpu().numpy().astype(np.uint32))
    assert res.hits(0) == lib.search(q[0], k)


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_scan_schedules_agree(name, monkeypatch):
    """The single-query bulk-copy scan has three tile schedules -- static
    per-warp parts, CTA-dynamic (shared counter) and the global dynamic tail
    (long scans only) -- selected per call; FPS_SCAN_FLAGS 64 / 256 switch the
    dynamic ones off. Every schedule returns the oracle's exact list, for
    several queries and k values (ties at the k-th distance included)."""
    plan, lib, q, w = full(name)
    rng = np.random.default_rng(7)
    queries = [q[0], w[int(rng.integers(len(w)))], w[int(rng.integers(len(w)))]]
    for k in (1, 10, 100, 1000):
        want = [oracle_lists(w, np.asarray(qq).reshape(1, 3), k)[0] for qq in queries]
        for flags in ("0", "64", "256", "320"):
            monkeypatch.setenv("FPS_SCAN_FLAGS", flags)
            for qq, exp in zip(queries, want):
                assert lib.search(qq, k) == exp, (flags, k)
    monkeypatch.delenv("FPS_SCAN_FLAGS")
