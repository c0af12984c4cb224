"""Host-overhead floor for one single-query call (C2 shape)."""
import sys, time, ctypes as C
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1906_06170_b200 import synth, _native as N
plan = synth.make_plan(sys.argv[1] if len(sys.argv) > 1 else "c2")
lib, q = synth.build_library(plan)
L = N.load()
k = plan.k
qa = np.ascontiguousarray(q[:1])
idx = np.empty((1, k), np.uint64); dist = np.empty((1, k), np.uint16); cnt = np.empty(1, np.uint32)
def t(f, n=300):
    for _ in range(20): f()
    t0 = time.perf_counter()
    for _ in range(n): f()
    return (time.perf_counter() - t0) / n * 1e6
h = lib._h
qp, ip, dp, cp = qa.ctypes.data, idx.ctypes.data, dist.ctypes.data, cnt.ctypes.data
print("fps_version ctypes us %.2f" % t(lambda: L.fps_version()))
print("raw fps_topk us %.2f" % t(lambda: L.fps_topk(h, qp, 1, k, ip, dp, cp)))
print("search_batch us %.2f" % t(lambda: lib.search_batch(qa, k)))
x = torch.zeros(1, device="cuda")
def empty():
    x.add_(1); torch.cuda.synchronize()
print("torch tiny kernel + sync us %.2f" % t(empty))
# device time of one isolated call (events around it)
s = torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
keys = torch.empty((1, k), dtype=torch.int64, device="cuda"); cntd = torch.empty((1,), dtype=torch.int32, device="cuda")
dq = torch.from_numpy(qa.view(np.int64).copy()).cuda()
lib.topk_prepare(1, k)
ts = []
with torch.cuda.stream(s):
    for _ in range(50):
        torch.cuda.synchronize()
        e0.record(s); lib.topk_async(dq, 1, k, keys, cntd, s.cuda_stream); e1.record(s); e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
print("isolated device call (events) us median %.2f" % np.median(ts))
