"""Per-tile timeline of the fp4 operand-copy tensor-core scan (CTA 0, tiles
2000..2063): run with FPS_SCAN_FLAGS=1048576 (+ other flags), WL=c4|c5."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from paper_1906_06170_b200 import _native as N, synth  # noqa: E402

wl = os.environ.get("WL", "c4")
plan = synth.make_plan(wl, n=int(os.environ.get("N", 20_000_000)))
lib, q = synth.build_library(plan)
for _ in range(2):
    if plan.radius is None:
        lib.search_batch(q, plan.k)
    else:
        lib.range_search(q, plan.radius)
print("kernel", lib.last_kernel)
f = N.load().fps_dbg_mm4_trace
f.argtypes = [C.c_void_p]
buf = np.zeros(64 * 8, dtype=np.uint64)
print("rc", f(buf.ctypes.data))
t = buf.reshape(64, 8).astype(np.int64)
t0 = t[0, 0]
names = ["mma_pre", "mma_full_ok", "mma_commit", "ld_empty_ok", "epi7_arrive", "epi7_tfull", "epi0_tfull", "epi0_arrive"]
print("tile " + " ".join(f"{n:>11s}" for n in names))
for i in range(64):
    print(f"{2000 + i:4d} " + " ".join(f"{(v - t0):11d}" for v in t[i]))
med = lambda x: float(np.median(x))
print("issue period", med(np.diff(t[:, 2])))
print("mma_pre -> full ok (tempty + full wait)", med(t[:, 1] - t[:, 0]))
print("commit -> epi0 tfull", med(t[:, 6] - t[:, 2]), " commit -> epi7 tfull", med(t[:, 5] - t[:, 2]))
print("epi0 tfull -> arrive", med(t[:, 7] - t[:, 6]), " epi7 tfull -> arrive", med(t[:, 4] - t[:, 5]))
print("last arrive(it-2) -> mma full ok(it)", med(t[2:, 1] - np.maximum(t[:-2, 7], t[:-2, 4])))
print("mma full ok -> commit", med(t[:, 2] - t[:, 1]))
print("loader: empty ok period", med(np.diff(t[:, 3])), " loader lead over mma (tiles*period)", med(t[:, 1] - t[:, 3]))
