import sys, os
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import numpy as np
import fps_oracle as orc
from paper_1906_06170_b200 import synth
from paper_1906_06170_b200.library import Library
Q = int(sys.argv[1]) if len(sys.argv) > 1 else 33
seed = 4242 + Q
thr = synth.beta_thresholds(seed)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200_000
w = orc.generate_words(synth.seed_key(seed), thr, 0, n)
rng = np.random.default_rng(Q)
q = w[rng.integers(0, len(w), Q)].copy()
q[:, 0] ^= rng.integers(0, 2**20, Q).astype(np.uint64) << np.uint64(1)
lib = Library.from_words(w)
mode = sys.argv[3] if len(sys.argv) > 3 else "topk"
try:
    if mode == "range":
        r = lib.range_search(q, 30)
        exp = orc.c_range(w, q, 30)
        print("range ok", np.array_equal(r.rows(), exp), len(exp))
    else:
        for k in (1, 10, 64):
            res = lib.search_batch(q, k)
            idx, dist, cnt = orc.c_topk(w, q, k)
            bad = [i for i in range(Q) if res.hits(i) != list(zip(idx[i, :cnt[i]].tolist(), dist[i, :cnt[i]].tolist()))]
            print("k", k, "bad", bad[:10], [(res.hits(i)[:3], list(zip(idx[i, :3].tolist(), dist[i, :3].tolist()))) for i in bad[:2]])
except Exception as e:
    print("ERR", e)
