"""First-wave bound exchange of the single-query plane scan (fps_planeq.cuh).

Libraries with at least two steps per warp (>= 4.85 M entries on 148 SMs)
take the wave: every warp posts its first step's witnesses, one warp
per CTA polls the global histogram and hands the bound to the others before
the second step. Results must stay the reference's (scan.py:194-203: distance,
then ascending index) whatever the wave sees -- half of the witnesses, none
(timeout), or no wave at all -- on ordinary, dense, all-ties and adversarially
ordered libraries. Checked bit-exactly against the C oracle.
"""

import numpy as np
import pytest

import fps_oracle as orc
from paper_1906_06170_b200 import synth
from paper_1906_06170_b200.library import Library

pytestmark = pytest.mark.gpu

N = 6_000_000  # > 2 steps per warp: the wave is on


def oracle(w, q, k):
    idx, dist, cnt = orc.c_topk(w, np.atleast_2d(q), k)
    return list(zip(idx[0, :cnt[0]].tolist(), dist[0, :cnt[0]].tolist()))


@pytest.fixture(scope="module")
def words():
    plan = synth.make_plan("c2", n=N)
    lib, q = synth.build_library(plan)
    w = lib.words_host()
    lib.close()
    return plan, w, q


def queries(plan, w, q):
    rng = np.random.default_rng(7)
    dense = rng.integers(0, 1 << 63, size=3, dtype=np.uint64) | rng.integers(0, 1 << 63, size=3, dtype=np.uint64)
    dense[2] &= np.uint64((1 << 38) - 1)
    dense[0] &= ~np.uint64(1)
    return [q[0], w[N // 2].copy(), dense, np.zeros(3, dtype=np.uint64)]


@pytest.mark.parametrize("env", [{}, {"FPS_PQ_WAVE_PCT": "0"}, {"FPS_PQ_WAVE_NS": "0"}, {"FPS_PQ_WAVE_PCT": "100"},
                                 {"FPS_PQ_SHAPE": "0"}, {"FPS_PQ_SHAPE": "2"}])
def test_wave_variants_match_oracle(words, monkeypatch, env):
    plan, w, q = words
    for k_, v in env.items():
        monkeypatch.setenv(k_, v)
    lib = Library.from_words(w)  # (the knobs are read once per handle)
    try:
        for qi, qq in enumerate(queries(plan, w, q)):
            for k in (1, 10, 100, 1000):
                got = lib.search(qq, k)
                assert lib.last_kernel == "single-query plane scan"
                assert got == oracle(w, qq, k), (env, qi, k)
    finally:
        lib.close()


def test_wave_all_ties():
    """Every entry at the same distance: the k smallest indices, in order."""
    row = np.array([0x0123456789ABCDEE, 0x0F0F0F0F0F0F0F0F, 0x2A2A2A2A2A], dtype=np.uint64)
    w = np.tile(row, (N, 1))
    lib = Library.from_words(w)
    try:
        q = row.copy()
        q[1] ^= np.uint64(0b111)
        for k in (1, 10, 100, 1024):
            assert lib.search(q, k) == [(i, 3) for i in range(k)]
    finally:
        lib.close()


@pytest.mark.parametrize("order", ["falling", "rising"])
def test_wave_adversarial_order(words, order):
    """Entries ordered by distance to the query: with falling distances every
    step beats the bound so far (the best entries come last), with rising
    distances the first step already holds the answer."""
    plan, w, q = words
    d = orc.distances_one(w, q[0]).astype(np.int64)
    perm = np.argsort(-d if order == "falling" else d, kind="stable")
    ws = np.ascontiguousarray(w[perm])
    lib = Library.from_words(ws)
    try:
        for k in (10, 100):
            assert lib.search(q[0], k) == oracle(ws, q[0], k), (order, k)
    finally:
        lib.close()


@pytest.mark.parametrize("hint", [True, False])
def test_plane_list_widths_device_query(hint):
    """Device-resident single queries across the widths at which the ring and
    warp count change (48 / 56 / 96 stage positions), with the host hint
    (fps_query_hint: ring sized to the list) and without (ring sized for 48
    positions, wider lists fold warps): same answers as the oracle."""
    import torch

    from paper_1906_06170_b200.library import keys_to_hits

    n = 400_000
    w = orc.generate_words(synth.seed_key(31), synth.beta_thresholds(31), 0, n)
    lib = Library.from_words(w)
    rng = np.random.default_rng(11)
    k = 10
    keys = torch.empty((1, k), dtype=torch.int64, device="cuda")
    cnt = torch.empty((1,), dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    try:
        lib.topk_prepare(1, k)
        for pop in (1, 38, 40, 41, 48, 49, 70, 83, 84, 100, 126, 165):
            bits = rng.choice(np.arange(1, 166), size=pop, replace=False)
            qq = np.zeros((1, 3), dtype=np.uint64)
            for b in bits:
                qq[0, b // 64] |= np.uint64(1) << np.uint64(b % 64)
            lib.query_hint(qq[0] if hint else None)
            dq = torch.from_numpy(qq.view(np.int64).copy()).cuda()
            lib.topk_async(dq, 1, k, keys, cnt, s)
            torch.cuda.synchronize()
            got = keys_to_hits(keys.cpu().numpy().view(np.uint64), cnt.cpu().numpy().view(np.uint32)).hits(0)
            assert lib.last_kernel == "single-query plane scan"
            assert got == oracle(w, qq[0], k), (hint, pop)
            # a stale hint (the previous, different query's width) must not matter
        lib.query_hint(None)
    finally:
        lib.close()
