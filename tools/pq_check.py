"""Plane-scan bring-up: parity vs the C oracle (host and device query paths) and
quick timings against the POPC single-query scan. Run on the GPU box."""
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import fps_oracle as orc  # noqa: E402
from paper_1906_06170_b200 import build, synth  # noqa: E402
from paper_1906_06170_b200.library import Library  # noqa: E402

build.build()


def oracle(w, q, k):
    idx, dist, cnt = orc.c_topk(w, q, k)
    return [list(zip(idx[i, :cnt[i]].tolist(), dist[i, :cnt[i]].tolist())) for i in range(len(q))]


def dev_topk(lib, q, k):
    dq = torch.from_numpy(np.ascontiguousarray(q[:1]).view(np.int64).copy()).cuda()
    keys = torch.empty((1, k), dtype=torch.int64, device="cuda")
    cnt = torch.empty((1,), dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    lib.topk_prepare(1, k)
    lib.topk_async(dq, 1, k, keys, cnt, s)
    torch.cuda.synchronize()
    kk = keys.cpu().numpy().view(np.uint64)[0][: int(cnt[0])]
    return [(int(x & ((1 << 40) - 1)), int(x >> 40)) for x in kk]


fails = 0
rng = np.random.default_rng(7)
for n in [1, 31, 2047, 2048, 2049, 100_000, 1_000_003]:
    for dens in [2**30, 2**62, 2**63 + 2**62]:  # sparse, ~25 %, dense queries
        w = orc.generate_words(1234 + n, np.full(166, dens, np.uint64), 0, n)
        lib = Library.from_words(w)
        q = w[n // 2:n // 2 + 1].copy()
        q[0, 1] ^= np.uint64(0xF0F0)
        for k in (1, 10, 100, 1000):
            exp = oracle(w, q, k)[0]
            got = lib.search(q[0], k)
            gd = dev_topk(lib, q, k)
            ok = got == exp and gd == exp
            if not ok:
                fails += 1
                print("MISMATCH", n, dens, k, lib.last_kernel, got[:5], gd[:5], exp[:5], flush=True)
        print("n", n, "dens", dens, "kernel", lib.last_kernel, "ok", flush=True)
        lib.close()
# all-identical library: every entry ties
w = np.tile(orc.generate_words(5, np.full(166, 2**62, np.uint64), 0, 1), (50_000, 1))
lib = Library.from_words(w)
for k in (1, 10, 100, 1024):
    exp = oracle(w, w[:1], k)[0]
    if lib.search(w[0], k) != exp or dev_topk(lib, w[:1], k) != exp:
        fails += 1
        print("MISMATCH identical", k)
print("identical ok", flush=True)
lib.close()

for wl in ["c2", "c3"]:
    plan = synth.make_plan(wl)
    lib, q = synth.build_library(plan)
    w = lib.words_host()
    exp = oracle(w, q[:1], plan.k)[0]
    for mode in ["1", "0"]:
        os.environ["FPS_PLANEQ"] = mode
        got = lib.search(q[0], plan.k)
        gd = dev_topk(lib, q, plan.k)
        if got != exp or gd != exp:
            fails += 1
            print("MISMATCH", wl, mode, got[:5], exp[:5])
        dq = torch.from_numpy(np.ascontiguousarray(q[:1]).view(np.int64).copy()).cuda()
        keys = torch.empty((1, plan.k), dtype=torch.int64, device="cuda")
        cnt = torch.empty((1,), dtype=torch.int32, device="cuda")
        s = torch.cuda.current_stream().cuda_stream
        for _ in range(5):
            lib.topk_async(dq, 1, plan.k, keys, cnt, s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 50
        e0.record()
        for _ in range(K):
            lib.topk_async(dq, 1, plan.k, keys, cnt, s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        t0 = time.perf_counter()
        for _ in range(20):
            lib.search(q[0], plan.k)
        e2e = (time.perf_counter() - t0) / 20 * 1e3
        print(f"{wl} PLANEQ={mode} kernel={lib.last_kernel} step {ms * 1e3:.1f} us  e2e {e2e * 1e3:.1f} us "
              f"cmp/s {plan.n / ms * 1e3:.3e}", flush=True)
    os.environ["FPS_PLANEQ"] = "1"
    lib.close()
print("FAILS", fails)
