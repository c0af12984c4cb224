"""Per-tile timeline of the fp4 tensor-core scan (CTA 0, tiles 2000..2063).
Run with FPS_SCAN_FLAGS=1048576 (+ other flags)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from paper_1906_06170_b200 import _native as N, synth  # noqa: E402

plan = synth.make_plan("c4", n=int(os.environ.get("N", 20_000_000)))
lib, q = synth.build_library(plan)
res = lib.search_batch(q, 10)
res = lib.search_batch(q, 10)
print("kernel", lib.last_kernel)
so = N.load()
f = so.fps_dbg_mm4_trace
f.argtypes = [C.c_void_p]
buf = np.zeros(64 * 8, dtype=np.uint64)
print("rc", f(buf.ctypes.data))
t = buf.reshape(64, 8).astype(np.int64)
t0 = t[0, 0]
names = ["iss_tempty", "iss_full", "iss_commit", "prod_raw", "prod_empty", "prod_arrive", "epi_tfull", "epi_done"]
print("tile " + " ".join(f"{n:>11s}" for n in names))
for i in range(0, 64):
    print(f"{2000 + i:4d} " + " ".join(f"{(v - t0):11d}" for v in t[i]))
d = np.diff(t[:, 2])
print("issue period (clk): median", np.median(d), "mean", d.mean())
print("producer arrive -> issuer full wait done (median):", np.median(t[:, 1] - t[:, 5]))
print("issuer commit -> epilogue tfull (median):", np.median(t[:, 6] - t[:, 2]))
print("epilogue tfull -> done (median):", np.median(t[:, 7] - t[:, 6]))
print("epilogue done(it-2) -> issuer tempty(it) (median):", np.median(t[2:, 0] - t[:-2, 7]))
print("producer: raw ready -> empty ok (median):", np.median(t[:, 4] - t[:, 3]), " empty ok -> arrive:", np.median(t[:, 5] - t[:, 4]))
print("producer period:", np.median(np.diff(t[:, 5])))
