"""World-size-2 tests of the multi-GPU plumbing on CPU (gloo backend).

Each rank holds its contiguous shard (libstore.split_sizes semantics) and a
per-shard top-k / range result with global indices; the package's
``gather_topk`` / ``gather_range`` move them to rank 0 exactly as the NCCL
path does. The device merge / sort are replaced by host equivalents built on
the oracle, so what is tested here is the sharding + collective + merge
contract; the CUDA merge kernel itself is covered by the gpu tests
(test_multi_shard_merge_on_one_gpu).
"""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _encode(idx, dist_, cnt, k):
    keys = np.full((len(cnt), k), -1, dtype=np.int64)
    for q in range(len(cnt)):
        c = int(cnt[q])
        keys[q, :c] = ((dist_[q, :c].astype(np.int64) << 40) | idx[q, :c].astype(np.int64))
    return torch.from_numpy(keys), torch.from_numpy(cnt.astype(np.int32))


def _host_merge(in_keys, in_cnt, k):
    import fps_oracle as orc

    G, Q, _ = in_keys.shape
    out = torch.full((Q, k), -1, dtype=torch.int64)
    outc = torch.zeros((Q,), dtype=torch.int32)
    for q in range(Q):
        parts = []
        for g in range(G):
            c = int(in_cnt[g, q])
            kk = in_keys[g, q, :c].numpy().astype(np.uint64)
            parts.append([(int(x & np.uint64((1 << 40) - 1)), int(x >> np.uint64(40))) for x in kk])
        m = orc.merge_topk(parts, k)
        outc[q] = len(m)
        for i, (ident, d) in enumerate(m):
            out[q, i] = (d << 40) | ident
    return out, outc


def _host_merge_runs(runs):
    """Host stand-in for fps_merge_runs_async: every run arrives sorted."""
    for r in runs:
        assert bool(torch.all(r[1:] > r[:-1])) if r.numel() > 1 else True
    return torch.sort(torch.cat(runs)).values


def _worker(rank, world, port, n, k, result_path):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "oracle"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import fps_oracle as orc

        from paper_1906_06170_b200 import distributed as D
        from paper_1906_06170_b200 import synth

        plan = synth.make_plan("c4", seed=77, n=n, Q=6)
        w = orc.generate_words(plan.seed_key, plan.thresholds, 0, n)
        q = synth.planted_after_sources(plan, w)
        start, count = D.shard_range(n, world, rank)
        idx, dd, cnt = orc.c_topk(w[start:start + count], q, k, threads=2)
        idx = np.where(idx == np.iinfo(np.uint64).max, idx, idx + np.uint64(start))
        keys, cnts = _encode(idx, dd, cnt, k)
        merged = D.gather_topk(keys, cnts, k, _host_merge)

        rr = orc.c_range(w[start:start + count], q, 25, threads=2)
        rkeys = torch.from_numpy(((rr[:, 0] << 48) | (rr[:, 2] << 40) | (rr[:, 1] + start)).astype(np.int64))
        rmerged = D.gather_range(rkeys, _host_merge_runs)
        if rank == 0:
            ei, ed, ec = orc.c_topk(w, q, k, threads=2)
            ek, ecn = _encode(ei, ed, ec, k)
            ok_topk = torch.equal(merged[0], ek) and torch.equal(merged[1], ecn)
            er = orc.c_range(w, q, 25, threads=2)
            got = rmerged.numpy().astype(np.uint64)
            ok_range = np.array_equal(orc.range_keys_to_rows(got), er)
            Path(result_path).write_text(f"{int(ok_topk)} {int(ok_range)} {len(er)}")
        else:
            assert merged is None and rmerged is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gather_merge_equals_single_process(tmp_path, world):
    result = tmp_path / "result.txt"
    mp.spawn(_worker, args=(world, _free_port(), 30_011, 17, str(result)), nprocs=world, join=True)
    ok_topk, ok_range, nrange = result.read_text().split()
    assert ok_topk == "1"
    assert ok_range == "1"
    assert int(nrange) > 0
