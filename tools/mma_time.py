import os, sys, time
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1906_06170_b200 import build, synth
build.build()
plan = synth.make_plan(os.environ.get("WL", "c4"))
lib, q = synth.build_library(plan)
dq = torch.from_numpy(np.ascontiguousarray(q).view(np.int64).copy()).cuda()
keys = torch.empty((plan.Q, plan.k or 1), dtype=torch.int64, device="cuda")
cnt = torch.empty((plan.Q,), dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for mode in os.environ.get("MODES", "1 0").split():
    os.environ["FPS_MMA"] = mode
    if plan.radius is not None:
        call = lambda: lib.range_search(q, plan.radius)
    else:
        lib.topk_prepare(plan.Q, plan.k)
        call = lambda: lib.topk_async(dq, plan.Q, plan.k, keys, cnt, s)
    call()
    torch.cuda.synchronize()
    lib.timing(True)
    t0 = time.perf_counter()
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    t, c = lib.timing_read()
    lib.timing(False)
    print(f"{plan.name if hasattr(plan,'name') else ''} FPS_MMA={mode} {lib.last_kernel}: call {dt*1e3:.2f} ms, scan kernel {t/c:.2f} ms", flush=True)
