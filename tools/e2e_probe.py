import sys, time, ctypes as C
sys.path.insert(0, ".")
import numpy as np
from paper_1906_06170_b200 import synth, _native as N
plan = synth.make_plan("c2")
lib, q = synth.build_library(plan)
k = plan.k
qa = np.ascontiguousarray(q)
idx = np.empty((1, k), np.uint64); dist = np.empty((1, k), np.uint16); cnt = np.empty(1, np.uint32)
L = N.load()
for _ in range(20): lib.search_batch(qa, k)
def t(f, n=200):
    t0 = time.perf_counter()
    for _ in range(n): f()
    return (time.perf_counter() - t0) / n * 1e6
print("search_batch us", t(lambda: lib.search_batch(qa, k)))
h = lib._h
print("raw ctypes us", t(lambda: L.fps_topk(h, qa.ctypes.data, 1, k, idx.ctypes.data, dist.ctypes.data, cnt.ctypes.data)))
import os
