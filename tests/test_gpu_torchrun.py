"""bench.py's one-process-per-GPU path end to end (needs a B200).

The driver's scaling run launches ``bench.py --gpus N`` under torchrun, one
rank per GPU over NCCL. Only one GPU is available here and NCCL rejects
ranks that share a device, so this runs the same code path with two ranks on
the one GPU and the gloo backend (``FPS_BENCH_SHARE_GPU=1``,
``FPS_BENCH_DIST_BACKEND=gloo``: the collectives take a host round trip; no
kernel waits on another rank). What it pins: contiguous shards with global
indices, the per-step gather + rank-0 merge (pipelined across steps for
shards larger than L2), the range runs merged by rank, the JSON line — and
that the merged answer equals the single-GPU answer on the whole library
(merge_topk semantics, scan.py:225-236; split_sizes, libstore.py:174-179).
"""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

from paper_1906_06170_b200 import synth

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(workload: str, nproc: int = 2) -> dict:
    env = dict(os.environ, FPS_BENCH_SHARE_GPU="1", FPS_BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(nproc),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"),
           "--gpus", str(nproc), "--workload", workload, "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
           "--e2e-steps", "3"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-4000:]  # rank 0 prints one line
    return json.loads(lines[0])


def test_torchrun_topk_pipelined_shards_match_single_gpu():
    """C3 (95.4 M entries) over two ranks: 47.7 M-entry shards (planes larger
    than L2, so the gather of step i overlaps the scan of step i + 1)."""
    line = _torchrun("c3")
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert "pipelin" in (line["method"].get("pipelining") or "")
    plan = synth.make_plan("c3")
    lib, q = synth.build_library(plan)
    try:
        best = lib.search_batch(q[:1], plan.k).hits(0)[0]
    finally:
        lib.close()
    assert line["check"]["q0_best"] == [int(best[0]), int(best[1])]


def test_torchrun_small_shards_flushed_path():
    """C2 (k = 100, planted near-duplicates) over two ranks: shards below L2
    take the flushed, step-by-step path."""
    line = _torchrun("c2")
    assert line["n_gpus"] == 2
    assert line["method"].get("pipelining") is None and "flushed" in line["method"]["l2"]
    plan = synth.make_plan("c2")
    lib, q = synth.build_library(plan)
    try:
        best = lib.search_batch(q[:1], plan.k).hits(0)[0]
    finally:
        lib.close()
    assert line["check"]["q0_best"] == [int(best[0]), int(best[1])]


def test_torchrun_range_runs_merged():
    """C5 over two ranks: per-rank sorted range runs merged by rank on rank 0
    (fps_merge_runs_async) — the hit count equals the single-GPU count."""
    line = _torchrun("c5")
    plan = synth.make_plan("c5")
    lib, q = synth.build_library(plan)
    try:
        n = len(lib.range_search(q, plan.radius))
    finally:
        lib.close()
    assert line["check"]["range_hits"] == n and line["check"]["sorted"]
