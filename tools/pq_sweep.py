"""Plane-scan shape sweep (warps per CTA x ring stages) on C2/C3/C1, back-to-back
topk_async calls timed with CUDA events (relative comparisons only)."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1906_06170_b200 import build, synth  # noqa: E402

build.build()
def parse(sh):  # "[bpl:]warps x stages"
    b, _, ws = sh.rpartition(":")
    w, s = ws.split("x")
    return (b or "2", int(w), int(s))


shapes = [parse(s) for s in os.environ.get("SHAPES", "8x2,4x2,4x4,8x3,16x2,16x1,12x2").split(",")]
shapes = [(c, b, w, s) for c in os.environ.get("COPIES", "1").split(",") for (b, w, s) in shapes]
for wl in os.environ.get("WLS", "c3,c2,c1").split(","):
    plan = synth.make_plan(wl)
    lib, q = synth.build_library(plan)
    dq = torch.from_numpy(np.ascontiguousarray(q[:1]).view(np.int64).copy()).cuda()
    keys = torch.empty((1, plan.k), dtype=torch.int64, device="cuda")
    cnt = torch.empty((1,), dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    ref = None
    for cp, bpl, wv, st in shapes:
        os.environ["FPS_PQ_COPY"] = cp
        os.environ["FPS_PQ_BPL"] = bpl
        os.environ["FPS_PQ_WARPS"] = str(wv)
        os.environ["FPS_PQ_STAGES"] = str(st)
        lib.topk_prepare(1, plan.k)
        for _ in range(5):
            lib.topk_async(dq, 1, plan.k, keys, cnt, s)
        torch.cuda.synchronize()
        res = keys.cpu().numpy().tolist()
        if ref is None:
            ref = res
        ok = res == ref
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
        lib.timing(True)
        for _ in range(20):
            lib.topk_async(dq, 1, plan.k, keys, cnt, s)
        torch.cuda.synchronize()
        t, c = lib.timing_read()
        lib.timing(False)
        print(f"{wl} copy={cp} bpl={bpl} warps={wv:2d} stages={st} step {best:7.1f} us  scan(events) {t / c * 1e3:7.1f} us  same={ok}",
              flush=True)
    lib.close()
