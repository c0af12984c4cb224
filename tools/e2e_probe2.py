"""Host-path cost of a single-query call: public API vs raw C ABI vs device time."""
import sys, time, ctypes as C
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1906_06170_b200 import synth, _native as N

for wl in sys.argv[1:] or ["c2"]:
    plan = synth.make_plan(wl)
    lib, q = synth.build_library(plan)
    k = plan.k
    qa = np.ascontiguousarray(q[:1])
    idx = np.empty((1, k), np.uint64); dist = np.empty((1, k), np.uint16); cnt = np.empty(1, np.uint32)
    L = N.load()
    h = lib._h
    for _ in range(20):
        lib.search_batch(qa, k)

    def t(f, n=300):
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            for _ in range(n):
                f()
            best = min(best, (time.perf_counter() - t0) / n * 1e6)
        return best

    a = t(lambda: lib.search_batch(qa, k))
    qp, ip, dp, cp = qa.ctypes.data, idx.ctypes.data, dist.ctypes.data, cnt.ctypes.data
    b = t(lambda: L.fps_topk(h, qp, 1, k, ip, dp, cp))
    dq = torch.from_numpy(qa.view(np.int64).copy()).cuda()
    keys = torch.empty((1, k), dtype=torch.int64, device="cuda")
    cc = torch.empty((1,), dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    lib.topk_prepare(1, k)
    for _ in range(10):
        lib.topk_async(dq, 1, k, keys, cc, s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(300):
        lib.topk_async(dq, 1, k, keys, cc, s)
    e1.record()
    torch.cuda.synchronize()
    d = e0.elapsed_time(e1) / 300 * 1e3
    print(f"{wl}: search_batch {a:.1f} us | raw fps_topk {b:.1f} us | device back-to-back {d:.1f} us", flush=True)
    lib.close()
