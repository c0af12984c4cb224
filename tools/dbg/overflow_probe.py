"""Probe: tensor-core candidate overflow (all-identical library), one process per variant."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "oracle"))
import fps_oracle as orc  # noqa: E402
from paper_1906_06170_b200.library import Library  # noqa: E402

n = int(os.environ.get("N", 300_000))
Q = int(os.environ.get("Q", 200))
row = np.array([0x00FF00FF00FF00FF, 0x1234, 0x5], dtype=np.uint64)
w = np.tile(row, (n, 1))
lib = Library.from_words(w)
rng = np.random.default_rng(2)
q = np.tile(row, (Q, 1))
q[:, 1] ^= rng.integers(0, 1 << 20, size=Q, dtype=np.uint64)
try:
    res = lib.search_batch(q, 10)
    print("kernel", lib.last_kernel)
    idx, dist, cnt = orc.c_topk(w, q, 10)
    ok = all(res.hits(i) == list(zip(idx[i, :cnt[i]].tolist(), dist[i, :cnt[i]].tolist())) for i in range(Q))
    print("ok", ok)
except Exception as exc:
    print("ERR", exc)
