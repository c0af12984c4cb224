"""Short libraries: host-path single-query call time against the plane scan's warp
count (8 warps x 2,048-entry steps is the default below 4.85 M entries)."""
import os
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1906_06170_b200 import synth

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for n in (250_000, 1_000_000, 2_000_000, 4_000_000):
    for warps in os.environ.get("WARPS", "2,4,6,8").split(","):
        os.environ["FPS_PQ_SHAPE"] = "0"
        os.environ["FPS_PQ_WARPS"] = warps
        plan = synth.make_plan("c1", n=n)
        lib, q = synth.build_library(plan)
        q1 = np.ascontiguousarray(q[:1])
        for _ in range(20):
            lib.search_batch(q1, plan.k)
        t0 = time.perf_counter()
        for _ in range(300):
            lib.search_batch(q1, plan.k)
        warm = (time.perf_counter() - t0) / 300 * 1e6
        cold = 0.0
        for i in range(30):
            flush.fill_(i & 1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            lib.search_batch(q1, plan.k)
            cold += time.perf_counter() - t0
        print(f"n = {n:9d} warps {warps:>2s}: call {warm:6.1f} us back to back, {cold / 30 * 1e6:6.1f} us after an L2 flush", flush=True)
        lib.close()
