"""Plane scan vs the query's popcount (plane list width, warp folding): back-to-back
topk_async calls on the C2 / C3 libraries, CUDA events (relative numbers)."""
import os
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1906_06170_b200 import synth

for wl in sys.argv[1:] or ["c2"]:
    plan = synth.make_plan(wl)
    lib, q = synth.build_library(plan)
    rng = np.random.default_rng(3)
    keys = torch.empty((1, plan.k), dtype=torch.int64, device="cuda")
    cnt = torch.empty((1,), dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for pop in (20, 30, 38, 40, 41, 44, 48, 56, 70, 83, 100, 126, 140):
        bits = rng.choice(np.arange(1, 166), size=pop, replace=False)
        qq = np.zeros((1, 3), dtype=np.uint64)
        for b in bits:
            qq[0, b // 64] |= np.uint64(1) << np.uint64(b % 64)
        dq = torch.from_numpy(qq.view(np.int64).copy()).cuda()
        lib.topk_prepare(1, plan.k)
        if not os.environ.get('NOHINT'):
            lib.query_hint(qq[0])
        for _ in range(5):
            lib.topk_async(dq, 1, plan.k, keys, cnt, s)
        torch.cuda.synchronize()
        best = 1e9
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            K = 40
            e0.record()
            for _ in range(K):
                lib.topk_async(dq, 1, plan.k, keys, cnt, s)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / K * 1e3)
        print(f"{wl} |q| = {pop:3d} (planes {8 + min(pop, 166 - pop):3d})  step {best:7.1f} us", flush=True)
    lib.close()
