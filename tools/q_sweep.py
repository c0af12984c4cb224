"""Multi-query top-k throughput vs Q on the 95.4 M library: POPC kernels
(FPS_BITSLICE=0) vs the bit-sliced kernel. Device time per call (events)."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1906_06170_b200 import synth
plan = synth.make_plan("c4")
lib, q = synth.build_library(plan)
s = torch.cuda.Stream()
for Q in [int(x) for x in (sys.argv[1:] or ["8", "16", "24", "32", "48", "64", "128"])]:
    dq = torch.from_numpy(np.ascontiguousarray(q[:Q]).view(np.int64).copy()).cuda()
    keys = torch.empty((Q, 10), dtype=torch.int64, device="cuda"); cnt = torch.empty((Q,), dtype=torch.int32, device="cuda")
    row = []
    for bs in ("0", "1"):
        os.environ["FPS_BITSLICE"] = bs
        lib.topk_prepare(Q, 10)
        with torch.cuda.stream(s):
            for _ in range(2):
                lib.topk_async(dq, Q, 10, keys, cnt, s.cuda_stream)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(5):
                lib.topk_async(dq, Q, 10, keys, cnt, s.cuda_stream)
            e1.record(s)
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        row.append(f"{'bitslice' if bs == '1' else 'popc'} {ms:.3f} ms ({Q * plan.n / ms / 1e9:.1f} Gcmp/s, {lib.last_kernel})")
    print(f"Q={Q}: " + " | ".join(row), flush=True)
