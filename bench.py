#!/usr/bin/env python
"""bench.py — fingerprint comparisons/s of the B200 scan (and of the reference CPU path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3] [--impl ours|reference]

A step is one pass of the hot path over one batch of synthetic input: the
workload's queries against the whole library. The default workload is
BASELINE.json configs[2] (C3: one query vs the 95,417,114-entry paper-scale
library, k = 10) — the north-star single-query HBM-bound scan; c1, c2, c4,
c5 are selectable with --workload.

Multi-GPU (contiguous shards, libstore.split_sizes): under torchrun each of
the N ranks holds one shard and per-rank top-k lists are merged on rank 0
(NCCL gather + the device merge kernel); without torchrun, --gpus N drives N
GPUs from one process (LibraryGroup: the root's merge kernel reads the other
shards' results from peer HBM). N must match the ranks and the visible GPUs:
anything else exits non-zero.

`value` is device-timed (CUDA events on the launching stream, inputs resident
in HBM, L2 flushed between steps when the bytes a step reads fit in L2);
`e2e` is the same metric through the public API with host buffers (query
H2D + result D2H inside the timed region). `roofline` is for the scan
kernel, timed live with CUDA events around each of its launches.
`--impl reference` times the reference CPU path on the host cores, rank 0
only: the unmodified reference ``fpscan.scan.search`` (installed under
baseline/_ref by tools/install_reference.sh) over FPS1 shards of the same
library, else the numpy restatement in oracle/.
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
    p.add_argument("--workload", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--seed", type=int, default=20240808)
    p.add_argument("--e2e-steps", type=int, default=None)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-flush", action="store_true")
    p.add_argument("--k", type=int, default=None, help="override the workload's k (experiments)")
    p.add_argument("--queries", type=int, default=None, help="override the workload's batch size (experiments)")
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


L2_BYTES = 126 << 20  # B200 L2 (cudaDeviceProp.l2CacheSize); both arms' configs state the same L2 policy


def l2_policy(plan, queries, world: int) -> str:
    """The timing rule's L2 choice for this workload, per GPU: the bytes one
    scan launch reads (the query's bit planes for a single query, the 21
    B/entry tiles otherwise) against L2 -- larger is its own flush, smaller is
    flushed between steps. Stated in both arms' config dicts."""
    shard = -(-plan.n // max(world, 1))
    if plan.Q == 1 and plan.radius is None:
        nbytes = shard * plane_scan_planes(queries[0]) / 8.0
    else:
        nbytes = shard * 21.0
    return "flushed between steps" if nbytes <= L2_BYTES else "inputs larger than L2 (no flush)"


def roofline_model(workload: str) -> dict:
    """Per-kernel instruction-mix constants measured once with ncu (profiles/roofline_model.json)."""
    p = ROOT / "profiles" / "roofline_model.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get(workload, {})
        except Exception:
            return {}
    return {}


def tensor_peaks() -> dict:
    """Measured tcgen05 dense rates per operand kind and accumulator width."""
    p = ROOT / "profiles" / "tensor_peaks.json"
    try:
        return json.loads(p.read_text())
    except Exception:
        return {"nominal": {"i8": 4500.0, "mxf4": 9000.0}}


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
# CPU reference path — baseline infrastructure (never the thing measured on GPU)
# ---------------------------------------------------------------------------
def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _reference_fpscan():
    """The unmodified reference package from baseline/_ref (tools/install_reference.sh), or None."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "fpscan" / "scan.py").exists():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        import fpscan.fingerprint as ff
        import fpscan.libstore as fl
        import fpscan.scan as fs

        return fs, fl, ff
    except Exception:  # pragma: no cover - broken install
        return None


def _scratch_dir(nbytes: int) -> str | None:
    """/dev/shm when it holds the FPS1 files with room to spare (page-cache
    resident, like the reference's warmed-up runs), else the default temp dir."""
    import shutil

    for d in ("/dev/shm", None):
        try:
            if d is None or shutil.disk_usage(d).free > 1.5 * nbytes + (1 << 30):
                return d
        except OSError:
            continue
    return None


class CpuWorkload:
    """The workload's library (generated on the host by the C twin of the
    device generator), planted entries, queries, and FPS1 shards + manifest
    (shard_count = host threads, the reference's unit of parallelism)."""

    def __init__(self, plan, n: int, q_count: int, threads: int):
        sys.path.insert(0, str(ROOT / "oracle"))
        import fps_oracle as orc

        from paper_1906_06170_b200 import synth

        self.orc, self.plan, self.n, self.threads = orc, plan, n, threads
        t0 = time.perf_counter()
        words = orc.generate_words_parallel(plan.seed_key, plan.thresholds, 0, n, threads)
        src = synth.generate_rows(plan.seed_key, plan.thresholds, plan.source_idx)
        self.queries = plan.queries_from_sources(src)
        if len(plan.planted_idx):
            pw = plan.planted_words(self.queries)
            m = plan.planted_idx < n
            words[plan.planted_idx[m]] = pw[m]
        self.words = words
        self.q_count = q_count
        self._td = tempfile.TemporaryDirectory(dir=_scratch_dir(n * 32))
        self.manifest_path = orc.write_fps1_library(Path(self._td.name), words, shard_count=max(1, threads))
        self.prep_s = time.perf_counter() - t0
        self.ref = _reference_fpscan()
        self.kind = "reference" if self.ref is not None else "port"
        if self.ref is not None:
            fs, fl, ff = self.ref
            self.ref_manifest = fl.load_manifest(self.manifest_path.parent)
            self.ref_queries = [ff.Fingerprint(tuple(int(x) for x in q)) for q in self.queries[:q_count]]

    def describe(self) -> str:
        if self.plan.radius is not None:
            how = "range restatement (numpy, oracle/fps_oracle.py; the reference has no range op)"
        elif self.ref is not None:
            how = "the unmodified reference fpscan.scan.search (baseline/_ref)"
        else:
            how = "numpy restatement of fpscan.scan.search (oracle/fps_oracle.py)"
        return (f"{self.q_count} quer{'y' if self.q_count == 1 else 'ies'} x {self.n:,} entries of workload "
                f"{self.plan.name} per step, FPS1 shards={self.threads}, {how}")

    def step(self, parallelism: int):
        plan = self.plan
        for qi in range(self.q_count):
            if plan.radius is not None:
                self.orc.range_search(self.words, self.queries[qi:qi + 1], plan.radius)
            elif self.ref is not None:
                fs, _, _ = self.ref
                fs.search(self.ref_manifest, self.ref_queries[qi], fs.SearchParams(n=plan.k, parallelism=parallelism))
            else:
                self.orc.search_fps1(self.manifest_path, self.queries[qi], plan.k, parallelism=parallelism)

    def close(self):
        self._td.cleanup()


def _cpu_queries(plan) -> int:
    """Queries per CPU step: the whole batch for single-query configs, a
    labelled 4-query sample of C4 / C5 (1,024 or 64 full-library passes would
    take minutes per step on the host)."""
    return plan.Q if plan.Q == 1 else min(plan.Q, 4)


def cpu_baseline(plan, budget_s: float = 20.0) -> dict:
    """The reference CPU path timed on this host (rank 0, N = 1): a bounded
    sample of the workload, at P = all host threads and at P = 1."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import fps_oracle as orc

    threads = orc.cpu_threads()
    n_s = min(plan.n, 16_000_000)
    wl = CpuWorkload(plan, n_s, _cpu_queries(plan), threads)
    try:
        wl.step(threads)  # page cache / first-touch warm-up (as test_acceptance.py:179)
        times = []
        t_start = time.perf_counter()
        while len(times) < 3 and (not times or time.perf_counter() - t_start < budget_s / 2):
            t0 = time.perf_counter()
            wl.step(threads)
            times.append(time.perf_counter() - t0)
        value = wl.q_count * n_s / min(times)
        t0 = time.perf_counter()
        wl.step(1)
        p1 = wl.q_count * n_s / (time.perf_counter() - t0)
        return {"value": value, "unit": UNIT, "cores": threads, "kind": wl.kind,
                "sample": wl.describe() + f" (bounded sample), best of {len(times)}",
                "p1": {"value": p1, "cores": 1}, "cpu_model": cpu_model()}
    finally:
        wl.close()


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return 0
    sys.path.insert(0, str(ROOT / "oracle"))
    import fps_oracle as orc

    from paper_1906_06170_b200 import synth

    plan = synth.make_plan(args.workload, seed=args.seed)
    threads = orc.cpu_threads()
    wl = CpuWorkload(plan, plan.n, _cpu_queries(plan), threads)  # the full library
    try:
        for _ in range(args.warmup):
            wl.step(threads)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            wl.step(threads)
        wall = time.perf_counter() - t0
        t1 = time.perf_counter()
        wl.step(1)
        p1 = wl.q_count * plan.n / (time.perf_counter() - t1)
        sample = wl.describe()
        kind, prep = wl.kind, wl.prep_s
        l2_queries_policy = l2_policy(plan, wl.queries, world)
    finally:
        wl.close()
    ms = wall * 1e3 / args.steps
    value = wl.q_count * plan.n * args.steps / wall
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": dict(plan.describe(), l2=l2_queries_policy),
        "sample": sample,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample,
                         "p1": {"value": p1, "cores": 1}, "cpu_model": cpu_model(),
                         "input_prep_s": prep},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def fail(msg: str) -> int:
    print(json.dumps({"error": msg}), flush=True)
    print(f"bench.py: {msg}", file=sys.stderr, flush=True)
    return 2


def run_ours(args, rank: int, local_rank: int, world: int):
    import torch
    import torch.distributed as dist

    from paper_1906_06170_b200 import distributed as D
    from paper_1906_06170_b200 import synth

    visible = torch.cuda.device_count()
    group_devs = None  # single process driving args.gpus GPUs
    # test-only plumbing check (tests/test_gpu_torchrun.py): several ranks may
    # share the visible GPUs, with the gloo backend (no cross-rank GPU waits)
    share = os.environ.get("FPS_BENCH_SHARE_GPU") == "1"
    backend = os.environ.get("FPS_BENCH_DIST_BACKEND", "nccl")
    if world > 1:
        if args.gpus != world:
            return fail(f"--gpus {args.gpus} but torchrun started {world} ranks")
        if visible < world and not share:
            return fail(f"{world} ranks but only {visible} visible GPU(s)")
        if share and backend == "nccl":
            return fail("FPS_BENCH_SHARE_GPU needs a non-NCCL backend (NCCL rejects ranks sharing a GPU)")
        local_rank = local_rank % max(visible, 1)
    elif args.gpus > 1:
        if visible < args.gpus:
            return fail(f"--gpus {args.gpus} but only {visible} visible GPU(s)")
        group_devs = list(range(args.gpus))
    n_gpus = world if world > 1 else args.gpus

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_stream(torch.cuda.Stream(dev))  # a real stream: kernels, events and copies share it
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    plan = synth.make_plan(args.workload, seed=args.seed, Q=args.queries)
    if args.k is not None:
        plan.k, plan.radius = args.k, None
    if args.radius is not None:
        plan.k, plan.radius = None, args.radius
    start, count = D.shard_range(plan.n, world, rank)
    t_load = time.perf_counter()
    lib, queries = synth.build_library(plan, device=local_rank, start=start, count=count, devices=group_devs)
    torch.cuda.synchronize()
    load_ms = (time.perf_counter() - t_load) * 1e3
    shard0 = lib.shards[0] if group_devs else lib
    shard_n = shard0.n  # entries one scan launch covers (the largest shard)
    Q = plan.Q
    dq = torch.from_numpy(queries.view(np.int64).copy()).to(dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    props = torch.cuda.get_device_properties(dev)
    l2 = getattr(props, "L2_cache_size", 126 << 20) or (126 << 20)
    flush_buf = clean_buf = None

    def flush_l2():
        # write a buffer larger than L2 (evicts the library), then read another
        # one so the dirty lines are written back before the timed region
        for d in (group_devs or [local_rank]):
            with torch.cuda.device(d):
                flush_buf[d].zero_()
                clean_buf[d].sum()

    state = {}
    if plan.radius is None:
        k = plan.k
        t_prep = time.perf_counter()
        lib.topk_prepare(Q, k)  # scratch + the derived plane copies, before the timed region
        if Q == 1 and hasattr(lib, "query_hint"):
            lib.query_hint(queries[0])  # the device-resident query's plane list (ring / warp count)
        torch.cuda.synchronize()
        prep_ms = (time.perf_counter() - t_prep) * 1e3
        keys = torch.empty((Q, k), dtype=torch.int64, device=dev)
        cnt = torch.empty((Q,), dtype=torch.int32, device=dev)
        if world > 1:
            # per-rank results land in packed blocks (keys, then counts) that
            # go to the collective as they are; rank 0 gathers them into one
            # (world, block) buffer and merges with one kernel. Consecutive
            # steps pipeline as in a serving loop: step i's gather + merge (on
            # a second stream) overlap step i + 1's scan, double-buffered (a
            # scan waits until the gather that last read its block is done).
            # Every step's scan, gather and merge run inside the timed region.
            comm = torch.cuda.Stream(dev)
            blocks = [D.packed_block(Q, k, dev) for _ in range(2)]
            gbufs = [None, None]
            gdone = [None, None]
            state["i"] = 0

        def step(pipelined: bool = False):
            if world == 1:
                lib.topk_async(dq, Q, k, keys, cnt, stream)
                return keys, cnt
            blk, bk, bc = blocks[0]
            if not pipelined:
                lib.topk_async(dq, Q, k, bk, bc, stream)
                return D.gather_topk_packed(blk, Q, k)
            j = state["i"] % 2
            state["i"] += 1
            blk, bk, bc = blocks[j]
            cur = torch.cuda.current_stream(dev)
            if gdone[j] is not None:
                cur.wait_event(gdone[j])
            lib.topk_async(dq, Q, k, bk, bc, stream)
            scanned = torch.cuda.Event()
            scanned.record(cur)
            with torch.cuda.stream(comm):
                comm.wait_event(scanned)
                if gbufs[j] is None and rank == 0:
                    gbufs[j] = torch.empty((world, blk.numel()), dtype=torch.int64, device=dev)
                r = D.gather_topk_packed(blk, Q, k, gbuf=gbufs[j])
                gdone[j] = torch.cuda.Event()
                gdone[j].record(comm)
            return r
    else:
        rad = torch.full((Q,), plan.radius, dtype=torch.uint8, device=dev)
        count_t = torch.zeros((1,), dtype=torch.int64, device=dev)
        t_prep = time.perf_counter()
        if group_devs:
            state["hits"] = lib.range_begin(queries, plan.radius)
        else:
            cap = 1 << 22
            out = torch.empty((cap,), dtype=torch.int64, device=dev)
            lib.range_async(dq, Q, rad, out, cap, count_t, stream)
            torch.cuda.synchronize()
            hits = int(count_t.item())
            if hits > cap:
                cap = hits + 1024
                out = torch.empty((cap,), dtype=torch.int64, device=dev)
            state.update(hits=hits, cap=cap, out=out)
        prep_ms = (time.perf_counter() - t_prep) * 1e3

        def step():
            if group_devs:  # per-shard scans + sorts, root merge; hits stay on the root
                return lib.range_begin(queries, plan.radius)
            lib.range_async(dq, Q, rad, state["out"], state["cap"], count_t, stream)
            lib.sort_keys(state["out"], state["hits"], stream)
            if world > 1:
                return D.gather_range(state["out"][: state["hits"]], D.device_merge_runs)
            return state["out"][: state["hits"]]

    def barrier():
        if world > 1:
            if backend == "nccl":
                dist.barrier(device_ids=[local_rank])
            else:
                dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # Library bytes one scan launch reads: the whole tiled shard, or for the
    # single-query plane scan only the planes of the query (8 popcount planes +
    # min(|q|, 166 - |q|) key planes, 1 bit per entry each).
    kernel = lib.last_kernel
    compact, bpe = lib.layout()
    if kernel == "single-query plane scan":
        bytes_per_launch = float(shard_n) * plane_scan_planes(queries[0]) / 8.0
    else:
        bytes_per_launch = float(bpe) * shard_n
    # Bytes read per step larger than L2 are their own flush: the scans stream
    # with an L2 evict-first policy, so K steps run back to back between one
    # event pair. Smaller ones (C1; C2 on the plane scan) get an explicit flush
    # between steps, outside per-step events.
    policy = l2_policy(plan, queries, world if world > 1 else max(1, len(group_devs or [0])))
    flush = (not args.no_flush) and policy.startswith("flushed")
    if flush:
        flush_buf, clean_buf = {}, {}
        for d in (group_devs or [local_rank]):
            flush_buf[d] = torch.empty(max(2 * l2, 256 << 20), dtype=torch.uint8, device=d)
            clean_buf[d] = torch.ones(max(2 * l2, 256 << 20) // 8, dtype=torch.int64, device=d)
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
        pipelined = world > 1 and plan.radius is None  # (this branch: shards larger than L2, no flush)
        ev0[0].record()
        for i in range(args.steps):
            step(pipelined) if pipelined else step()
        if pipelined:
            torch.cuda.current_stream(dev).wait_stream(comm)
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
    mem = lib.memory()

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
        achieved = Q * shard_n / (scan_avg_ms / 1e3) / 1e9
        naive = sm * POPC_PER_SM_CLK / POPC_PER_CMP_NAIVE * mhz * 1e6 / 1e9
        model = roofline_model(args.workload)
        if kernel == "tensor-core multi-query scan":
            # tcgen05 GEMM: K = 192 elements (3 x 64 bits) per (query, entry)
            # pair, 2 ops per multiply-add. Denominator: the MEASURED dense
            # issue rate of the operand kind the scan ran with, at its
            # accumulator width (tools/microbench/umma_peak.cu,
            # profiles/tensor_peaks.json); nominal rates beside it. The
            # 6-POPC figure of SURVEY §8(d) is obsolete for this kernel.
            mk = lib.last_mma_kind or "i8"
            fam = "i8" if mk == "i8" else "mxf4"
            width = (256 if Q > 128 else 128 if Q > 64 else 64) if fam == "i8" else (
                64 if Q <= 64 else 128 if Q <= 128 else 208)
            tp = tensor_peaks()
            peak = float(tp.get(fam, {}).get(str(width), tp.get("nominal", {}).get(fam, 4500.0)))
            ops = 2.0 * 192 * Q * shard_n
            tops = ops / (scan_avg_ms / 1e3) / 1e12
            tensor = {"bound": "tensor", "achieved": tops, "peak": peak,
                      "unit": f"TOP/s ({'int8' if fam == 'i8' else 'fp4 e2m1, block-scaled'})", "frac": tops / peak,
                      "peak_source": f"measured dense tcgen05 kind::{'i8' if fam == 'i8' else 'mxf4'} rate at N = "
                                     f"{width} (profiles/tensor_peaks.json, tools/microbench/umma_peak.cu); nominal "
                                     f"{tp.get('nominal', {}).get(fam, 0):.0f} TOP/s: "
                                     f"{tops / max(tp.get('nominal', {}).get(fam, 1.0), 1.0):.3f}",
                      "algorithmic_ops_per_launch": ops}
            # the operand stream: the library's tiles (int8: 21 B/entry) or its
            # fp4 operand copy (96 B/entry), read once per pass from HBM (the
            # query chunks of a library range share it through L2); the
            # binding roofline is whichever fraction is higher
            op_bytes = (96.0 if mk == "fp4x" else float(bpe)) * shard_n
            hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
            hbm_gbs = op_bytes / (scan_avg_ms / 1e3) / 1e9
            hbm = {"bound": "hbm", "achieved": hbm_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": hbm_gbs / hbm_peak,
                   "peak_source": peaks["_source"], "algorithmic_bytes_per_launch": op_bytes,
                   "nominal_8tbs_frac": hbm_gbs / 8000.0}
            if hbm["frac"] > 1.0:
                # the measured peak is a COPY (read + write bytes of b.copy_(a)); a
                # read-only stream can run above it, up to the nominal 8 TB/s
                hbm["note"] = ("read-only stream above the copy-measured peak (which moves read + write bytes); "
                               "see nominal_8tbs_frac")
            main, other = (hbm, tensor) if hbm["frac"] > tensor["frac"] else (tensor, hbm)
            roof = dict(main, traffic=traffic_for(f"{args.workload}_{mk}") or traffic_for(args.workload),
                        operand_kind=mk, accumulator_columns=width, comparisons_per_s=achieved * 1e9)
            roof["other_bound"] = other
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
        # bytes the scan streams from HBM per launch: the fp4 operand copy
        # (96 B/entry, read once per pass; the query chunks share it in L2),
        # else the tiled library / bit-plane copy
        src_bpe = 96.0 if (kernel == "tensor-core multi-query scan" and lib.last_mma_kind == "fp4x") else float(bpe)
        roof.update({"naive_6popc_peak": naive, "naive_6popc_frac": achieved / naive,
                     "scan_kernel_ms": scan_avg_ms, "hbm_bytes_per_launch": src_bpe * shard_n,
                     "kernel": kernel})

    n_total = float(plan.n)
    parallel = (f"{n_gpus} GPUs in one process (LibraryGroup, gather {lib.gather})" if group_devs else
                f"{world} ranks (torchrun), {backend} gather to rank 0"
            + (" (test mode: ranks share the visible GPUs)" if share else "") if world > 1 else "1 GPU")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n_gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": dict(plan.describe(), l2=policy if not args.no_flush else "no flush (--no-flush)"),
        "method": {
            "parallelism": parallel,
            "pipelining": (f"pipelined: step i's {backend} gather + rank-0 merge overlap step i+1's scan (second "
                           "stream, double-buffered results); all K steps' scans, gathers and merges are inside the "
                           "timed region" if (world > 1 and plan.radius is None and not flush) else None),
            "l2": "flushed between steps outside the timed events (2xL2 write, then 2xL2 read so no dirty "
                  "lines are left)" if flush else
                  "library larger than L2 and streamed with an L2 evict-first policy: no flush, the K steps "
                  "run back to back between one event pair",
            "layout": (f"plane-major bit planes (1 bit/entry/plane); the query reads "
                       f"{plane_scan_planes(queries[0])} of 174 planes = "
                       f"{plane_scan_planes(queries[0]) / 8:.3f} B/entry"
                       if kernel == "single-query plane scan" else
                       f"tiles of {256 if compact else 128} entries, SoA inside a tile, {bpe} B/entry "
                       f"({'compact: word 2 as u32 + u8' if compact else 'full: 3 x u64'})"),
        },
        "library": {
            "load_ms": load_ms,
            "prepare_ms": prep_ms,
            "derived_build_ms": mem["derived_build_ms"],
            "hbm_bytes_per_entry": {"library": mem["library_bytes"] / n_total,
                                    "derived": mem["derived_bytes"] / n_total,
                                    "scratch": mem["scratch_bytes"] / n_total,
                                    "total": (mem["library_bytes"] + mem["derived_bytes"] + mem["scratch_bytes"])
                                    / n_total},
            "note": "this rank's HBM ÷ this rank's entries" if world > 1 else "all devices of the job ÷ entries",
        },
        "roofline": roof,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_s * 1e3 / e2e_steps, "steps": e2e_steps,
                "l2": "flushed before every call, calls timed one by one" if (flush and world == 1)
                      else "calls back to back"},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if world > 1:
        line["library"]["hbm_bytes_per_entry"] = {key: v * n_total / max(count, 1)
                                                  for key, v in line["library"]["hbm_bytes_per_entry"].items()}
    if rank == 0 and n_gpus == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(plan)
    elif rank == 0:
        line["cpu_baseline"] = None
    # sanity: results are real (first query's best hit; under torchrun the
    # rank-0 merge of every rank's shard)
    if rank == 0 and plan.radius is None and world == 1:
        res = lib.search_batch(qhost[:1], plan.k)
        line["check"] = {"q0_best": list(res.hits(0)[:1][0]) if res.count[0] else None}
    if world > 1 and plan.radius is None:
        r = step()
        if rank == 0:
            kk, cc = r
            kk, cc = kk.cpu().numpy().view(np.uint64), cc.cpu().numpy()
            line["check"] = {"q0_best": [int(kk[0, 0] & np.uint64((1 << 40) - 1)), int(kk[0, 0] >> np.uint64(40))]
                             if cc[0] else None}
    elif world > 1:
        r = step()
        if rank == 0:
            h = r.cpu().numpy().view(np.uint64)
            line["check"] = {"range_hits": int(len(h)),
                             "sorted": bool(np.all(h[1:] > h[:-1])) if len(h) > 1 else True}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    lib.close()
    return 0


def main():
    args = parse_args()
    rank, local_rank, world = dist_env()
    if args.gpus < 1:
        return fail("--gpus must be >= 1")
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, local_rank, world)


if __name__ == "__main__":
    sys.exit(main())
