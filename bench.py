#!/usr/bin/env python
"""bench.py — fingerprint comparisons/s of the B200 scan (and of the reference CPU path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--impl ours|reference]

A step is one pass of the hot path over one batch of synthetic input: the
workload's queries against the whole library (sharded contiguously over the
N ranks, per-rank top-k merged on rank 0 over NCCL when N > 1). The default
workload is BASELINE.json configs[1] (C2: one query vs 10,000,000 entries,
k = 100, 1,000 planted near-duplicates) — the single-GPU HBM-bound scan.
Other configs (c1, c3, c4, c5) are selectable with --workload.

`value` is device-timed (CUDA events on the launching stream, inputs resident
in HBM, L2 flushed between steps when the per-GPU library is within a few
L2 sizes); `e2e` is the same metric through the public API with host
buffers (query H2D + result D2H inside the timed region). `roofline` is for
the scan kernel, timed live with CUDA events around each of its launches.
`--impl reference` times the reference algorithm (the numpy restatement of
fpscan.scan in oracle/, reading FPS1 shard files like the reference) on the
host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fingerprint comparisons/sec (query×library pairs) and % of HBM/popcount roofline"
UNIT = "comparisons/s"
POPC_PER_SM_CLK = 16.0   # measured on B200 (tools/microbench, profiles/r01_microbench.txt)
POPC_PER_CMP_NAIVE = 6.0  # 3 x __popcll = 6 x 32-bit POPC per comparison
POPC_PER_CMP_CSA = 4.0    # multi-query kernel: carry-save fold, 4 POPC per comparison (dist3_csa)


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--seed", type=int, default=20240808)
    p.add_argument("--e2e-steps", type=int, default=None)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-flush", action="store_true")
    p.add_argument("--k", type=int, default=None, help="override the workload's k (experiments)")
    p.add_argument("--radius", type=int, default=None, help="run a range search at this radius instead")
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def measured_peaks() -> dict:
    for p in (ROOT / "MEASURED_PEAKS.json", Path("/root/repo/MEASURED_PEAKS.json")):
        if p.exists():
            try:
                d = json.loads(p.read_text())
                d["_source"] = "measured"
                return d
            except Exception:
                pass
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_source": "fallback"}


class ClockSampler(threading.Thread):
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during the timed region."""

    REASONS = {
        "hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
        "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
        "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
        "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
        "hw_power_brake_slowdown": "nvmlClocksEventReasonHwPowerBrakeSlowdown",
    }

    def __init__(self, index: int):
        super().__init__(daemon=True)
        self.index = index
        self.samples: list[int] = []
        self.reasons: set[str] = set()
        self.max_mhz = None
        self._halt = threading.Event()
        self._lock = threading.Lock()
        self.ok = False
        self._nv = self._h = None
        try:  # NVML set up before the timed region, so the first sample is not late
            import pynvml as nv

            nv.nvmlInit()
            self._nv, self._h = nv, nv.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            self._masks = {k: getattr(nv, v, 0) for k, v in self.REASONS.items()}
            self.ok = True
        except Exception as exc:  # pragma: no cover
            self.reasons.add(f"nvml_error:{type(exc).__name__}")

    def sample(self):
        """One clock + throttle-reason reading (also called inline from the
        timed region while the GPU drains the queued steps)."""
        if not self.ok:
            return
        nv, h = self._nv, self._h
        mhz = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        with self._lock:
            self.samples.append(mhz)
            for name, m in self._masks.items():
                if m and (r & m):
                    self.reasons.add(name)

    def run(self):
        try:
            while not self._halt.is_set():
                self.sample()
                self._halt.wait(0.005)
        except Exception as exc:  # pragma: no cover
            self.reasons.add(f"nvml_error:{type(exc).__name__}")

    def stop(self) -> dict:
        self._halt.set()
        self.join(timeout=2)
        return {"sm_mhz": float(statistics.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def plane_scan_planes(q) -> int:
    """Planes the single-query plane scan reads (fps_planeq.cuh): the 8
    popcount planes + the query's set keys (or zero keys when |q| > 83)."""
    w = [int(x) for x in q]
    pop = sum(bin(x).count("1") for x in w)
    pop166 = bin(w[0]).count("1") + bin(w[1]).count("1") + bin(w[2] & ((1 << 38) - 1)).count("1")
    return 8 + (166 - pop166 if pop > 83 else pop166)


def roofline_model(workload: str) -> dict:
    """Per-kernel instruction-mix constants measured once with ncu (profiles/roofline_model.json)."""
    p = ROOT / "profiles" / "roofline_model.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get(workload, {})
        except Exception:
            return {}
    return {}


def traffic_for(workload: str):
    """dram bytes per scan-kernel launch from the committed ncu --set full capture."""
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get(workload)
        except Exception:
            return None
    return None


# ---------------------------------------------------------------------------
# CPU reference (oracle port of fpscan.scan) — test/baseline infrastructure
# ---------------------------------------------------------------------------
def cpu_reference(plan, threads: int, budget_s: float, min_runs: int = 1, max_runs: int = 3,
                  words: np.ndarray | None = None, queries: np.ndarray | None = None):
    """Time the reference algorithm on a bounded sample of the workload.

    The sample library is written as FPS1 shards (shard_count = threads, the
    reference's unit of parallelism) and scanned by the numpy restatement of
    scan.search, which reads the shard files block by block like the
    reference. Returns (comparisons/s, description, runs)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import fps_oracle as orc

    from paper_1906_06170_b200 import synth

    # bounded sample: at most 16M entries, and at most 4 queries
    n_s = min(plan.n, 16_000_000)
    q_s = min(plan.Q, 4)
    if words is None:
        words = orc.generate_words_parallel(plan.seed_key, plan.thresholds, 0, n_s, threads)
        if len(plan.planted_idx):
            src = synth.generate_rows(plan.seed_key, plan.thresholds, plan.source_idx)
            queries = plan.queries_from_sources(src)
            pw = plan.planted_words(queries)
            m = plan.planted_idx < n_s
            words[plan.planted_idx[m]] = pw[m]
        else:
            src = synth.generate_rows(plan.seed_key, plan.thresholds, plan.source_idx[:q_s])
            queries = np.zeros((plan.Q, 3), dtype=np.uint64)
            queries[:q_s] = src
            for i in range(q_s):
                queries[i] ^= synth.flip_mask(plan.query_flips[i])
    words = words[:n_s]
    with tempfile.TemporaryDirectory(dir="/dev/shm" if Path("/dev/shm").exists() else None) as td:
        mpath = orc.write_fps1_library(Path(td), words, shard_count=max(1, threads))
        times = []
        t_start = time.perf_counter()
        for r in range(max_runs):
            t0 = time.perf_counter()
            for qi in range(q_s):
                if plan.radius is not None:
                    orc.range_search(words, queries[qi:qi + 1], plan.radius)
                else:
                    orc.search_fps1(mpath, queries[qi], plan.k, parallelism=threads)
            times.append(time.perf_counter() - t0)
            if r + 1 >= min_runs and time.perf_counter() - t_start > budget_s:
                break
    best = min(times)
    sample = (f"{q_s} quer{'y' if q_s == 1 else 'ies'} x {n_s:,} entries of workload {plan.name} "
              f"(FPS1 shards={threads}, {'range restatement' if plan.radius is not None else 'scan.search port'}), "
              f"best of {len(times)}")
    return q_s * n_s / best, sample, times


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return 0
    sys.path.insert(0, str(ROOT / "oracle"))
    import fps_oracle as orc

    from paper_1906_06170_b200 import synth

    plan = synth.make_plan(args.workload, seed=args.seed)
    threads = orc.cpu_threads()
    # warm-up + timed steps: each step is one bounded-sample search
    n_s = min(plan.n, 16_000_000)
    q_s = min(plan.Q, 4)
    words = orc.generate_words_parallel(plan.seed_key, plan.thresholds, 0, n_s, threads)
    if len(plan.planted_idx):
        src = synth.generate_rows(plan.seed_key, plan.thresholds, plan.source_idx)
        queries = plan.queries_from_sources(src)
        pw = plan.planted_words(queries)
        m = plan.planted_idx < n_s
        words[plan.planted_idx[m]] = pw[m]
    else:
        queries = plan.queries_from_sources(synth.generate_rows(plan.seed_key, plan.thresholds, plan.source_idx))
    with tempfile.TemporaryDirectory(dir="/dev/shm" if Path("/dev/shm").exists() else None) as td:
        mpath = orc.write_fps1_library(Path(td), words, shard_count=threads)

        def step():
            for qi in range(q_s):
                if plan.radius is not None:
                    orc.range_search(words, queries[qi:qi + 1], plan.radius)
                else:
                    orc.search_fps1(mpath, queries[qi], plan.k, parallelism=threads)

        for _ in range(args.warmup):
            step()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            step()
        wall = time.perf_counter() - t0
    ms = wall * 1e3 / args.steps
    value = q_s * n_s * args.steps / wall
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": args.workload, **plan.describe(), "sample_entries": n_s, "sample_queries": q_s},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{q_s} quer{'y' if q_s == 1 else 'ies'} x {n_s:,} entries per step, FPS1 "
                                   f"shards={threads}, numpy restatement of fpscan.scan (oracle/fps_oracle.py)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, rank: int, local_rank: int, world: int):
    import torch
    import torch.distributed as dist

    from paper_1906_06170_b200 import distributed as D
    from paper_1906_06170_b200 import synth
    from paper_1906_06170_b200.library import keys_to_hits

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_stream(torch.cuda.Stream(dev))  # a real stream: kernels, events and copies share it
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    plan = synth.make_plan(args.workload, seed=args.seed)
    if args.k is not None:
        plan.k, plan.radius = args.k, None
    if args.radius is not None:
        plan.k, plan.radius = None, args.radius
    start, count = D.shard_range(plan.n, world, rank)
    lib, queries = synth.build_library(plan, device=local_rank, start=start, count=count)
    Q = plan.Q
    dq = torch.from_numpy(queries.view(np.int64).copy()).to(dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    props = torch.cuda.get_device_properties(dev)
    l2 = getattr(props, "L2_cache_size", 126 << 20) or (126 << 20)
    flush_buf = clean_buf = None

    def flush_l2():
        # write a buffer larger than L2 (evicts the library), then read another
        # one so the dirty lines are written back before the timed region
        flush_buf.zero_()
        clean_buf.sum()

    if plan.radius is None:
        k = plan.k
        lib.topk_prepare(Q, k)
        keys = torch.empty((Q, k), dtype=torch.int64, device=dev)
        cnt = torch.empty((Q,), dtype=torch.int32, device=dev)

        def step():
            lib.topk_async(dq, Q, k, keys, cnt, stream)
            if world > 1:
                return D.gather_topk(keys, cnt, k, D.device_merge)
            return keys, cnt
    else:
        rad = torch.full((Q,), plan.radius, dtype=torch.uint8, device=dev)
        count_t = torch.zeros((1,), dtype=torch.int64, device=dev)
        cap = 1 << 22
        out = torch.empty((cap,), dtype=torch.int64, device=dev)
        lib.range_async(dq, Q, rad, out, cap, count_t, stream)
        torch.cuda.synchronize()
        hits = int(count_t.item())
        if hits > cap:
            cap = hits + 1024
            out = torch.empty((cap,), dtype=torch.int64, device=dev)
        state = {"hits": hits}

        def step():
            lib.range_async(dq, Q, rad, out, cap, count_t, stream)
            lib.sort_keys(out, state["hits"], stream)
            if world > 1:
                return D.gather_range(out[: state["hits"]], D.device_sort)
            return out[: state["hits"]]

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local_rank])

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # Library bytes one step reads: the whole tiled library, or for the
    # single-query plane scan only the planes of the query (8 popcount planes +
    # min(|q|, 166 - |q|) key planes, 1 bit per entry each).
    kernel = lib.last_kernel
    compact, bpe = lib.layout()
    if kernel == "single-query plane scan":
        bytes_per_launch = float(count) * plane_scan_planes(queries[0]) / 8.0
    else:
        bytes_per_launch = float(bpe) * count
    # Bytes read per step larger than L2 are their own flush: the scans stream
    # with an L2 evict-first policy, so K steps run back to back between one
    # event pair. Smaller ones (C1; C2 on the plane scan) get an explicit flush
    # between steps, outside per-step events.
    flush = (not args.no_flush) and bytes_per_launch <= l2
    if flush:
        flush_buf = torch.empty(max(2 * l2, 256 << 20), dtype=torch.uint8, device=dev)
        clean_buf = torch.ones(max(2 * l2, 256 << 20) // 8, dtype=torch.int64, device=dev)
    launches0 = lib.launches
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    sampler = ClockSampler(local_rank)
    sampler.start()
    barrier()
    torch.cuda.synchronize()
    if flush:
        for i in range(args.steps):
            flush_l2()
            ev0[i].record()
            step()
            ev1[i].record()
    else:
        ev0 = ev0[:1]
        ev1 = ev1[:1]
        ev0[0].record()
        for i in range(args.steps):
            step()
        ev1[0].record()
        sampler.sample()  # the queued steps are still executing
    torch.cuda.synchronize()
    barrier()
    launches_timed = lib.launches - launches0
    # the scan kernel alone, bracketed by CUDA events inside the library, in a
    # separate pass so the extra event records do not perturb the timed steps
    lib.timing(True)
    for i in range(args.steps):
        if flush:
            flush_l2()
        step()
    torch.cuda.synchronize()
    scan_ms, scan_launches = lib.timing_read()
    lib.timing(False)
    clocks = sampler.stop()
    launches = launches_timed + (args.steps if (world > 1 and rank == 0 and plan.radius is None) else 0)
    total_ms = sum(a.elapsed_time(b) for a, b in zip(ev0, ev1))
    t = torch.tensor([total_ms, scan_ms / max(scan_launches, 1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, scan_avg_ms = float(t[0]), float(t[1])
    comparisons = Q * plan.n
    value = comparisons * args.steps / (total_ms / 1e3)

    # e2e through the public API with host buffers
    e2e_steps = args.e2e_steps or max(3, min(args.steps, 20))
    qhost = np.ascontiguousarray(queries)
    if world == 1:
        if plan.radius is None:
            lib.search_batch(qhost, plan.k)
            torch.cuda.synchronize()
            if flush:
                # bytes per call below L2: flush between calls, time each call
                # alone (the call is synchronous: host query in, host results out)
                e2e_s = 0.0
                for _ in range(e2e_steps):
                    flush_l2()
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    res = lib.search_batch(qhost, plan.k)
                    e2e_s += time.perf_counter() - t0
            else:
                t0 = time.perf_counter()
                for _ in range(e2e_steps):
                    res = lib.search_batch(qhost, plan.k)
                e2e_s = time.perf_counter() - t0
            d2h = Q * plan.k * 8 + Q * 4
        else:
            lib.range_search(qhost, plan.radius)
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                rr = lib.range_search(qhost, plan.radius)
            e2e_s = time.perf_counter() - t0
            d2h = len(rr) * 8 + 8
        h2d = Q * 24 + (Q if plan.radius is not None else 0)
    else:
        pinned = torch.from_numpy(qhost.view(np.int64).copy()).pin_memory()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            dq.copy_(pinned, non_blocking=True)
            r = step()
            if rank == 0:
                if plan.radius is None:
                    kk, cc = r
                    host_k, host_c = kk.cpu(), cc.cpu()
                else:
                    host_k = r.cpu()
            torch.cuda.synchronize()
        barrier()
        e2e_s = time.perf_counter() - t0
        tt = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt[0])
        h2d = Q * 24
        d2h = Q * plan.k * 8 + Q * 4 if plan.radius is None else int(state["hits"]) * 8
    e2e_value = comparisons * e2e_steps / e2e_s

    # roofline of the scan kernel
    peaks = measured_peaks()
    if plan.radius is None and Q <= 4:
        achieved = bytes_per_launch / (scan_avg_ms / 1e3) / 1e9
        peak = float(peaks.get("hbm_gbs", 6650.0))
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic_for(args.workload), "peak_source": peaks["_source"],
                "algorithmic_bytes_per_launch": bytes_per_launch, "scan_kernel_ms": scan_avg_ms, "kernel": kernel,
                "nominal_8tbs_frac": achieved / 8000.0}
    else:
        sm = props.multi_processor_count
        mhz = clocks["sm_mhz"] or float(peaks.get("sm_max_mhz", 1965.0))
        achieved = Q * count / (scan_avg_ms / 1e3) / 1e9
        naive = sm * POPC_PER_SM_CLK / POPC_PER_CMP_NAIVE * mhz * 1e6 / 1e9
        model = roofline_model(args.workload)
        if kernel == "tensor-core multi-query scan":
            # int8 GEMM on tcgen05: K = 192 bytes (3 x 64 bits) per pair, 2 ops
            # per multiply-add. There is no measured int8 peak on this pool:
            # the denominator is the nominal dense int8/fp8 tensor rate of a
            # B200 (4.5 POP/s, /opt/skills/guides/B200_PROFILING.md); the
            # ratio to 2 x the driver-measured dense bf16 rate (int8 issues at
            # twice the bf16 rate) is reported beside it.
            ops = 2.0 * 192 * Q * count
            tops = ops / (scan_avg_ms / 1e3) / 1e12
            bf16 = float(peaks.get("bf16_tflops", 1590.0))
            peak = 4500.0
            roof = {"bound": "tensor", "achieved": tops, "peak": peak, "unit": "TOP/s (int8)", "frac": tops / peak,
                    "traffic": traffic_for(args.workload),
                    "peak_source": "nominal dense int8 tensor rate of a B200 (4.5 POP/s, no measured int8 peak); "
                                   f"vs 2 x measured dense bf16 {2 * bf16:.0f} TOP/s ({peaks['_source']}): "
                                   f"{tops / (2 * bf16):.3f}",
                    "algorithmic_ops_per_launch": ops, "comparisons_per_s": achieved * 1e9}
        elif kernel == "bit-sliced multi-query scan" and model.get("alu_warp_instr_per_cmp"):
            # ALU-pipe bound: 2 warp-instructions/clk/SM issue on the ALU pipe;
            # ALU instructions per comparison of this kernel measured by ncu
            per = float(model["alu_warp_instr_per_cmp"])
            peak = sm * 2.0 * mhz * 1e6 / per / 1e9
            roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Gcmp/s", "frac": achieved / peak,
                    "traffic": traffic_for(args.workload),
                    "peak_source": f"{sm} SMs x 2 ALU warp-instructions/clk x {mhz:.0f} MHz / {per:.4f} ALU "
                                   f"warp-instructions per comparison (ncu, {model.get('source', 'profiles')})"}
        else:
            # binding pipe of the POPC formulation: XU at 16 lanes/clk/SM;
            # Q >= 2 kernels issue 4 POPC per comparison (carry-save), Q == 1 issues 6
            per_cmp = POPC_PER_CMP_CSA if Q >= 2 else POPC_PER_CMP_NAIVE
            peak = sm * POPC_PER_SM_CLK / per_cmp * mhz * 1e6 / 1e9  # G comparisons/s
            roof = {"bound": "popc", "achieved": achieved, "peak": peak, "unit": "Gcmp/s", "frac": achieved / peak,
                    "traffic": traffic_for(args.workload),
                    "peak_source": f"{sm} SMs x 16 POPC/clk/SM (measured) / {per_cmp:.0f} POPC per comparison x "
                                   f"{mhz:.0f} MHz (median SM clock in the timed region)"}
        roof.update({"naive_6popc_peak": naive, "naive_6popc_frac": achieved / naive,
                     "scan_kernel_ms": scan_avg_ms, "hbm_bytes_per_launch": float(bpe) * count,
                     "kernel": kernel})

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {**plan.describe(), "parallelism": f"shard{world}",
                   "l2": "flushed between steps outside the timed events (2xL2 write, then 2xL2 read so no dirty "
                         "lines are left)" if flush else
                   "library larger than L2 and streamed with an L2 evict-first policy: no flush, the K steps "
                   "run back to back between one event pair",
                   "layout": (f"plane-major bit planes (1 bit/entry/plane); the query reads "
                              f"{plane_scan_planes(queries[0])} of 174 planes = "
                              f"{plane_scan_planes(queries[0]) / 8:.3f} B/entry"
                              if kernel == "single-query plane scan" else
                              f"tiles of 128 entries, SoA inside a tile, {bpe} B/entry "
                              f"({'compact: word 2 as u32 + u8' if compact else 'full: 3 x u64'})")},
        "roofline": roof,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_s * 1e3 / e2e_steps, "steps": e2e_steps,
                "l2": "flushed before every call, calls timed one by one" if (flush and world == 1)
                      else "calls back to back"},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sys.path.insert(0, str(ROOT / "oracle"))
        import fps_oracle as orc

        threads = orc.cpu_threads()
        cv, sample, _ = cpu_reference(plan, threads, budget_s=10.0)
        line["cpu_baseline"] = {"value": cv, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample}
    elif rank == 0:
        line["cpu_baseline"] = None
    # sanity: results are real (first query's best hit is at a small distance)
    if rank == 0 and plan.radius is None and world == 1:
        res = lib.search_batch(qhost[:1], plan.k)
        line["check"] = {"q0_best": list(res.hits(0)[:1][0]) if res.count[0] else None}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    lib.close()
    return 0


def main():
    args = parse_args()
    rank, local_rank, world = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, local_rank, world)


if __name__ == "__main__":
    sys.exit(main())
