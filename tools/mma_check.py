"""Bring-up of the tcgen05 multi-query path (FPS_MMA=1): parity vs the C oracle and C4 timing."""
import os, sys, time
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle"))
import fps_oracle as orc
from paper_1906_06170_b200 import build, synth
from paper_1906_06170_b200.library import Library
build.build()
os.environ["FPS_MMA"] = "1"
fails = 0
for n in [1000, 200_003]:
    seed = 77 + n
    w = orc.generate_words(synth.seed_key(seed), synth.beta_thresholds(seed), 0, n)
    lib = Library.from_words(w)
    rng = np.random.default_rng(n)
    for Q in [2, 33, 256, 300]:
        q = w[rng.integers(0, n, Q)].copy()
        q[:, 0] ^= rng.integers(0, 2**20, Q).astype(np.uint64) << np.uint64(1)
        for k in [1, 10, 100]:
            res = lib.search_batch(q, k)
            idx, dist, cnt = orc.c_topk(w, q, k)
            for i in range(Q):
                exp = list(zip(idx[i, :cnt[i]].tolist(), dist[i, :cnt[i]].tolist()))
                if res.hits(i) != exp:
                    fails += 1
                    if fails < 5:
                        print("MISMATCH n", n, "Q", Q, "k", k, "q", i, lib.last_kernel, res.hits(i)[:4], exp[:4], flush=True)
        print("n", n, "Q", Q, "kernel", lib.last_kernel, "fails so far", fails, flush=True)
    lib.close()
print("FAILS", fails, flush=True)
plan = synth.make_plan("c4")
lib, q = synth.build_library(plan)
dq = torch.from_numpy(np.ascontiguousarray(q).view(np.int64).copy()).cuda()
keys = torch.empty((plan.Q, plan.k), dtype=torch.int64, device="cuda")
cnt = torch.empty((plan.Q,), dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for mode in ["1", "0"]:
    os.environ["FPS_MMA"] = mode
    lib.topk_prepare(plan.Q, plan.k)
    lib.topk_async(dq, plan.Q, plan.k, keys, cnt, s)
    torch.cuda.synchronize()
    r = keys.cpu().numpy().copy()
    t0 = time.perf_counter()
    for _ in range(3):
        lib.topk_async(dq, plan.Q, plan.k, keys, cnt, s)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"c4 FPS_MMA={mode} kernel={lib.last_kernel} {dt*1e3:.2f} ms/call  {plan.Q*plan.n/dt:.3e} cmp/s", flush=True)
    if mode == "1":
        r1 = r
    else:
        print("c4 mma == bit-sliced:", np.array_equal(r1, r), flush=True)
