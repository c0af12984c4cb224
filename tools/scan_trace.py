"""Timeline of one single-query top-k call (build with -DFPS_SCAN_TRACE).

Marker kernel on the library stream -> scan warps (start / first tile / end)
-> select start (after griddepcontrol.wait) -> select end, all in globaltimer
ns relative to the marker. Shows launch gap, warp-end spread (tail), PDL gap."""
import ctypes as C, os, sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1906_06170_b200 import synth, _native as N

L = N.load()
for wl in sys.argv[1:] or ["c2"]:
    plan = synth.make_plan(wl)
    lib, q = synth.build_library(plan)
    q1 = np.ascontiguousarray(q[:1])
    for _ in range(3):
        lib.search_batch(q1, plan.k)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    marks = np.zeros(8, np.uint64)
    warps = np.zeros(16384 * 4, np.uint64)
    for r in range(3):
        if not os.environ.get("NOFLUSH"):
            flush.fill_(r + 1)
            flush.sum()
        torch.cuda.synchronize()
        L.fps_trace_clear()
        L.fps_trace_mark(lib._h, 0)
        lib.search_batch(q1, plan.k)
        L.fps_trace_read(marks.ctypes.data, warps.ctypes.data)
        t = warps.reshape(-1, 4).astype(np.int64)
        t = t[t[:, 0] > 0]
        m0 = int(marks[0])
        st, en, en2 = t[:, 0] - m0, t[:, 1] - m0, t[:, 2] - m0
        fi = t[:, 3][t[:, 3] > 0] - m0
        pct = lambda v: " ".join("%6.1f" % (np.percentile(v, p) / 1e3) for p in (0, 10, 50, 90, 99, 100))
        print(f"{wl} run {r}: warps {len(t)}  [us after marker: p0 p10 p50 p90 p99 max]")
        print("  warp start ", pct(st))
        if len(fi):
            print("  first tile ", pct(fi))
        print("  loop end   ", pct(en))
        print("  warp exit / plane scan: second step start ", pct(en2[t[:, 2] > 0]) if (t[:, 2] > 0).any() else "-")
        ph = np.zeros(16384 * 8, np.uint64)
        if hasattr(L, "fps_trace_phases"):
            L.fps_trace_phases(ph.ctypes.data)
            ph = ph.reshape(-1, 8).astype(np.int64)[: len(warps) // 4]
            okr = ph[:, 0] > 0
            for i, name in enumerate(["csa done", "refill issue", "after X", "mask (2nd)", "-", "inserted(2nd)", "D done", "selected"]):
                v = ph[okr, i]
                v = v[v > 0] - m0
                if len(v):
                    print(f"  1st step {name:14s}", pct(v))
        if hasattr(L, "fps_trace_phases") and len(t) % 8 == 0:
            allw = warps.reshape(-1, 4).astype(np.int64)[: len(t)]
            seed = np.arange(len(t)) % 8 == 0
            f3 = allw[:, 3] - m0
            print("  first tile, seed warps ", pct(f3[seed & (allw[:, 3] > 0)]))
            print("  first tile, other warps", pct(f3[~seed & (allw[:, 3] > 0)]))
            p4 = ph[: len(t), 4]
            opened = (p4 < 0).sum()
            p4 = (p4 & ((1 << 62) - 1))
            if (p4 > 0).any():
                print("  seed tightened          ", pct(p4[p4 > 0] - m0), " still open:", opened)
            took = ph[: len(t), 6] > 0
            print("  warps on the bound-less first step: seed %d / %d, others %d / %d" % (
                (took & seed).sum(), seed.sum(), (took & ~seed).sum(), (~seed).sum()))
        if hasattr(L, "fps_trace_prologue"):
            pro = np.zeros(16384 * 4, np.uint64)
            L.fps_trace_prologue(pro.ctypes.data)
            pro = pro.reshape(-1, 4).astype(np.int64)[: len(t)]
            for i, name in enumerate(["list built (sync 2)", "ring initialised", "requests issued", "dependency wait over"]):
                print(f"  prologue {name:22s}", pct(pro[:, i] - m0))
        if hasattr(L, "fps_trace_steps"):
            stp = np.zeros(16384 * 8, np.uint64)
            L.fps_trace_steps(stp.ctypes.data)
            stp = stp.reshape(-1, 8).astype(np.int64)[: len(t)]
            for i in range(8):
                v = stp[:, i]
                v = v[v > 0] - m0
                if len(v):
                    print(f"  step {i} tile ready ({len(v):4d} warps)", pct(v))
        if hasattr(L, "fps_trace_s1"):
            s1 = np.zeros(16384 * 4, np.uint64)
            L.fps_trace_s1(s1.ctypes.data)
            s1 = s1.reshape(-1, 4).astype(np.int64)[: len(t)]
            for i, name in enumerate(["bound taken", "held-back inserted", "csa done"]):
                v = s1[:, i]
                v = v[v > 0] - m0
                if len(v):
                    print(f"  2nd step {name:20s}", pct(v))
        print("  select start %.1f  end %.1f" % ((int(marks[2]) - m0) / 1e3, (int(marks[3]) - m0) / 1e3))
        if int(marks[4]):
            print("  last warp found %.1f  its selection done %.1f" % ((int(marks[4]) - m0) / 1e3, (int(marks[5]) - m0) / 1e3 if int(marks[5]) else -1))
    lib.close()
