"""Multi-GPU sharding: one process per GPU, contiguous shards, merge on rank 0.

The reference's only parallelism is whole shards on a thread pool, merged in
process by ``merge_topk`` (scan.py:256-287, :225-236) over contiguous,
balanced shards (libstore.split_sizes, libstore.py:174-179). Here each rank
holds shard ``rank`` of the library in its HBM and reports global indices
(index_base = shard start); per-query top-k lists (k keys of
``distance << 40 | index`` per query, sorted) are gathered to rank 0 over
NCCL (NVLink on a B200 box) and merged there by the device merge kernel.
The top-k of a union equals the top-k of per-shard top-ks under a total
order, and shards are disjoint, so the merge is exact and associative.
Range hits are variable-sized: counts are all-gathered first, then padded
buffers gathered and the per-rank sorted runs merged by rank on rank 0
(``fps_merge_runs_async``; no re-sort of the union).

The collective plumbing is backend-agnostic (NCCL on GPUs, gloo in the CPU
tests); the merge / sort step is injected so the CPU tests can check the
plumbing against the oracle while the GPU path uses libfpsgpu.so.
"""

from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist

from .libstore import split_sizes

MergeFn = Callable[[torch.Tensor, torch.Tensor, int], tuple[torch.Tensor, torch.Tensor]]
MergeRunsFn = Callable[[list[torch.Tensor]], torch.Tensor]


def shard_range(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """(start, count) of this rank's contiguous shard."""
    sizes = split_sizes(n_total, world)
    return sum(sizes[:rank]), sizes[rank]


def _host_collective(t: torch.Tensor, group) -> bool:
    """gloo gathers CPU tensors only: device tensors take a host round trip
    (the CPU tests and the shared-GPU plumbing test; NCCL gathers in HBM)."""
    return t.is_cuda and dist.get_backend(group) != "nccl"


def gather_topk(keys: torch.Tensor, cnt: torch.Tensor, k: int, merge: MergeFn, group=None,
                dst: int = 0) -> tuple[torch.Tensor, torch.Tensor] | None:
    """Gather every rank's (Q, k) sorted key lists and (Q,) counts to ``dst``
    and merge them there. Returns the merged (keys, cnt) on dst, else None."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    keys = keys.contiguous()
    cnt = cnt.contiguous()
    if world == 1:
        return merge(keys.unsqueeze(0), cnt.unsqueeze(0), k)
    # one collective per call: keys and counts travel in a single int64 buffer
    Q = cnt.numel()
    packed = torch.cat([keys.reshape(-1).view(torch.int64), cnt.to(torch.int64)])
    dev = packed.device
    if _host_collective(packed, group):
        packed = packed.cpu()
    if rank == dst:
        bufs = [torch.empty_like(packed) for _ in range(world)]
        dist.gather(packed, bufs, dst=dst, group=group)
        allp = torch.stack(bufs).to(dev)  # (G, Q*k + Q)
        kk = allp[:, :Q * k].reshape(world, *keys.shape).view(keys.dtype)
        cc = allp[:, Q * k:].to(cnt.dtype)
        return merge(kk.contiguous(), cc.contiguous(), k)
    dist.gather(packed, None, dst=dst, group=group)
    return None


def packed_block(Q: int, k: int, device) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """One rank's result block for gather_topk_packed: Q x k keys then Q u32
    counts in one int64 buffer; returns (block, keys view, counts view) --
    the views are what fps_topk_async writes, so the block goes to the
    collective as is (no repacking)."""
    blk = torch.empty((Q * k + Q,), dtype=torch.int64, device=device)
    return blk, blk[: Q * k].view(Q, k), blk[Q * k:].view(torch.int32)[:Q]


def gather_topk_packed(block: torch.Tensor, Q: int, k: int, group=None, dst: int = 0,
                       gbuf: torch.Tensor | None = None) -> tuple[torch.Tensor, torch.Tensor] | None:
    """Gather every rank's packed result block (packed_block) into one
    (world, Q*k + Q) buffer on ``dst`` and merge it there with one kernel
    (fps_merge_packed_async). Returns the merged (keys, counts) on dst."""
    from . import _native as N

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = block.device
    L = block.numel()
    host = _host_collective(block, group)
    src = block.cpu() if host else block
    if rank != dst:
        dist.gather(src, None, dst=dst, group=group)
        return None
    if gbuf is None or gbuf.shape != (world, L) or gbuf.device != src.device:
        gbuf = torch.empty((world, L), dtype=torch.int64, device=src.device)
    dist.gather(src, list(gbuf.unbind(0)), dst=dst, group=group)
    if host:
        gbuf = gbuf.to(dev)
    out_keys = torch.empty((Q, k), dtype=torch.int64, device=dev)
    out_cnt = torch.empty((Q,), dtype=torch.int32, device=dev)
    N.check(N.load().fps_merge_packed_async(gbuf.data_ptr(), L * 8, world, Q, k, out_keys.data_ptr(),
                                            out_cnt.data_ptr(), torch.cuda.current_stream(dev).cuda_stream),
            "fps_merge_packed_async")
    return out_keys, out_cnt


def gather_range(keys: torch.Tensor, merge_runs: MergeRunsFn, group=None, dst: int = 0) -> torch.Tensor | None:
    """Gather every rank's sorted range-key run ((q, d, idx) order) to
    ``dst`` and merge the runs there. Returns the merged keys on dst."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    keys = keys.contiguous()
    if world == 1:
        return keys
    dev = keys.device
    host = _host_collective(keys, group)
    cdev = torch.device("cpu") if host else dev
    n = torch.tensor([keys.numel()], dtype=torch.int64, device=cdev)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(sizes)
    padded = torch.full((max(m, 1),), -1, dtype=keys.dtype, device=cdev)
    padded[: keys.numel()] = keys.to(cdev)
    if rank == dst:
        bufs = [torch.empty_like(padded) for _ in range(world)]
        dist.gather(padded, bufs, dst=dst, group=group)
        return merge_runs([b[:s].to(dev) for b, s in zip(bufs, sizes)])
    dist.gather(padded, None, dst=dst, group=group)
    return None


def device_merge(in_keys: torch.Tensor, in_cnt: torch.Tensor, k: int) -> tuple[torch.Tensor, torch.Tensor]:
    """CUDA merge kernel over (G, Q, k) keys / (G, Q) counts (rank 0)."""
    from .library import merge_async

    G, Q, _ = in_keys.shape
    out_keys = torch.empty((Q, k), dtype=torch.int64, device=in_keys.device)
    out_cnt = torch.empty((Q,), dtype=torch.int32, device=in_keys.device)
    merge_async(in_keys, in_cnt, G, Q, k, out_keys, out_cnt, torch.cuda.current_stream(in_keys.device).cuda_stream)
    return out_keys, out_cnt


def device_merge_runs(runs: list[torch.Tensor]) -> torch.Tensor:
    """Merge sorted runs of unique range keys by rank on the device (rank 0)."""
    import ctypes as C

    from . import _native as N

    dev = runs[0].device
    total = sum(r.numel() for r in runs)
    out = torch.empty((total,), dtype=torch.int64, device=dev)
    if total == 0:
        return out
    ptrs = (C.c_void_p * len(runs))(*[r.data_ptr() for r in runs])
    lens = (C.c_uint64 * len(runs))(*[r.numel() for r in runs])
    N.check(N.load().fps_merge_runs_async(ptrs, lens, len(runs), out.data_ptr(),
                                          torch.cuda.current_stream(dev).cuda_stream), "fps_merge_runs_async")
    return out


class ShardedLibrary:
    """This rank's contiguous shard of a library plus the rank-0 merge."""

    def __init__(self, local, n_total: int, group=None):
        self.local = local
        self.n_total = n_total
        self.group = group

    def topk_device(self, d_queries: torch.Tensor, k: int, stream: int | None = None):
        """Local top-k on this GPU, gathered and merged on rank 0 (device tensors)."""
        Q = d_queries.shape[0]
        dev = d_queries.device
        blk, keys, cnt = packed_block(Q, k, dev)
        s = torch.cuda.current_stream(dev).cuda_stream if stream is None else stream
        self.local.topk_async(d_queries, Q, k, keys, cnt, s)
        return gather_topk_packed(blk, Q, k, self.group)
