import sys, os
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import numpy as np
import fps_oracle as orc
from paper_1906_06170_b200 import synth
from paper_1906_06170_b200.library import Library
for Q in (2, 3, 4, 5, 8):
    seed = 4242 + Q
    thr = synth.beta_thresholds(seed)
    w = orc.generate_words(synth.seed_key(seed), thr, 0, 200_000)
    rng = np.random.default_rng(Q)
    q = w[rng.integers(0, len(w), Q)].copy()
    q[:, 0] ^= rng.integers(0, 2**20, Q).astype(np.uint64) << np.uint64(1)
    lib = Library.from_words(w)
    for k in (1, 10, 64):
        res = lib.search_batch(q, k)
        idx, dist, cnt = orc.c_topk(w, q, k)
        bad = [i for i in range(Q) if res.hits(i) != list(zip(idx[i, :cnt[i]].tolist(), dist[i, :cnt[i]].tolist()))]
        print("flags", os.environ.get("FPS_SCAN_FLAGS", "0"), "Q", Q, "k", k, "bad", bad,
              [(res.hits(i)[:2], list(zip(idx[i, :2].tolist(), dist[i, :2].tolist()))) for i in bad][:2])
