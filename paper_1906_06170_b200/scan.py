"""Drop-in replacement for the reference search surface, CUDA-backed.

Same names, argument meaning and error behaviour as
/root/reference/pkg/src/fpscan/scan.py: ``SearchHit`` / ``TopK`` /
``SearchParams`` (scan.py:50-88), ``merge_topk`` (scan.py:225-236),
``scan_shard`` / ``search`` / ``batch_search`` (scan.py:212-318). Results are
a pure function of (library bytes, query, n) under the (distance, cid) total
order, independent of ``parallelism``.

Differences, by design:
* the library is uploaded to HBM once per manifest (cached) instead of
  re-read from the shard files on every search (scan.py:160);
* ``kernel`` selects nothing: "cuda" is the default and "packed" /
  "reference" are accepted as aliases (the reference proves the two kernels
  equal, test_scan.py:217-222); every value runs the CUDA scan;
* progress fires once per shard when the device pass completes (final
  count only, still monotone and ending at record_count); cancellation is
  checked before launch.
"""

from __future__ import annotations

import os
import threading
from dataclasses import dataclass
from pathlib import Path
from typing import Callable, Literal, Sequence

import numpy as np

from .errors import DuplicateCid, LibstoreError, ScanCancelled, ScanError
from .fingerprint import as_query_words
from .library import Library, LibraryGroup

ShardProgressFn = Callable[[int], None]
SearchProgressFn = Callable[[str, int, int], None]
CancelFn = Callable[[], bool]

Kernel = Literal["cuda", "packed", "reference"]
BLOCK_RECORDS = 65536  # the reference's progress granularity (scan.py:29)


@dataclass(frozen=True)
class SearchHit:
    cid: int
    distance: int

    def sort_key(self) -> tuple[int, int]:
        return (self.distance, self.cid)


@dataclass(frozen=True)
class TopK:
    """The K smallest hits of a stream under (distance, cid) order."""

    capacity: int
    hits: tuple[SearchHit, ...]

    def __post_init__(self):
        if self.capacity < 1:
            raise ValueError("capacity must be >= 1")
        if len(self.hits) > self.capacity:
            raise ValueError(f"{len(self.hits)} hits exceed capacity {self.capacity}")
        keys = [h.sort_key() for h in self.hits]
        if any(a >= b for a, b in zip(keys, keys[1:])):
            raise ValueError("hits must be strictly increasing under (distance, cid)")


@dataclass(frozen=True)
class SearchParams:
    n: int = 30
    parallelism: int = 1
    kernel: Kernel = "cuda"

    def __post_init__(self):
        if self.n < 1:
            raise ValueError("n must be >= 1")
        if self.parallelism < 1:
            raise ValueError("parallelism must be >= 1")
        if self.kernel not in ("cuda", "packed", "reference"):
            raise ValueError(f"unknown kernel {self.kernel!r}")


def merge_topk(parts: Sequence[TopK], n: int) -> TopK:
    """The n smallest hits of the union; associative, commutative, duplicate-checking."""
    seen: set[int] = set()
    merged: list[tuple[int, int]] = []
    for part in parts:
        for hit in part.hits:
            if hit.cid in seen:
                raise DuplicateCid(f"cid {hit.cid} appears in more than one part")
            seen.add(hit.cid)
            merged.append((hit.distance, hit.cid))
    merged.sort()
    return TopK(capacity=n, hits=tuple(SearchHit(cid=c, distance=d) for d, c in merged[:n]))


# --------------------------------------------------------------------------
# resident libraries, one per (manifest contents, devices)
# --------------------------------------------------------------------------
@dataclass
class _Resident:
    lib: "Library | LibraryGroup"
    cids: np.ndarray
    cid_monotone: bool
    offsets: list[int]
    users: int = 0        # searches in flight (guarded by _cache_lock)
    evicted: bool = False  # out of the cache: closed when the last user leaves


_cache: dict[tuple, _Resident] = {}
_CACHE_MAX = 8
_cache_lock = threading.Lock()
RECORDS_PER_DEVICE = 8_000_000  # below this a library stays on one GPU (launch cost > scan)


def _manifest_key(manifest) -> tuple:
    parts = []
    for s in manifest.shards:
        p = Path(s.path)
        try:
            st = p.stat()
            parts.append((str(p), s.record_count, st.st_mtime_ns, st.st_size))
        except OSError:
            parts.append((str(p), s.record_count, None, None))
    return tuple(parts)


def search_devices(total_records: int) -> tuple[int, ...] | None:
    """GPUs a resident library is sharded over (the reference's shard fan-out,
    scan.py:256-287, is per process too): ``FPS_DEVICES=0,1,...`` if set,
    else every visible GPU, one per RECORDS_PER_DEVICE records (None: the
    current device only)."""
    env = os.environ.get("FPS_DEVICES")
    if env:
        devs = tuple(int(x) for x in env.replace(" ", "").split(",") if x)
        return devs or None
    from . import _native as N

    n = N.device_count()
    use = min(n, max(1, total_records // RECORDS_PER_DEVICE))
    return tuple(range(use)) if use > 1 else None


def _close(res: _Resident) -> None:
    res.lib.close()


def _acquire(manifest, devices: tuple[int, ...] | None) -> _Resident:
    """The resident library for this manifest, with a use reference taken:
    eviction never closes a library another thread is searching."""
    from . import libstore

    key = (_manifest_key(manifest), devices)
    with _cache_lock:
        hit = _cache.get(key)
        if hit is not None:
            hit.users += 1
            return hit
        # header pre-check in shard order, so the first bad shard is the one reported
        offsets = [0]
        for shard in manifest.shards:
            try:
                with open(shard.path, "rb") as f:
                    offsets.append(offsets[-1] + libstore.read_shard_header(f, shard.path))
            except (OSError, LibstoreError) as exc:
                raise ScanError(f"shard {shard.path}: {exc}") from exc
        paths = [s.path for s in manifest.shards]
        if devices is not None and len(devices) > 1:
            lib = LibraryGroup.from_fps1(paths, devices)
        else:
            lib = Library.from_fps1(paths, device=devices[0] if devices else None)
        cids = lib.cids
        if len(cids) > 1 and not bool(np.all(cids[1:] >= cids[:-1])):
            lib, cids = _cid_ordered(lib, paths, cids, devices)
        res = _Resident(lib=lib, cids=cids, cid_monotone=True, offsets=offsets, users=1)
        _cache[key] = res
        while len(_cache) > _CACHE_MAX:  # bounded HBM use: evict the oldest library
            old = _cache.pop(next(iter(_cache)))
            old.evicted = True
            if old.users == 0:
                _close(old)
        return res


def _fps1_words(paths) -> np.ndarray:
    """Every record's three fingerprint words, in shard order (bytes 8..31 of
    each 32-byte FPS1 record, as scan.py:169 views them)."""
    parts = [np.fromfile(p, dtype="<u8", offset=16).reshape(-1, 4)[:, 1:4] for p in paths]
    return np.ascontiguousarray(np.concatenate(parts) if parts else np.empty((0, 3), np.uint64), dtype=np.uint64)


def _cid_ordered(lib, paths, cids: np.ndarray, devices):
    """The library re-uploaded in CID order (stable; equal CIDs stay adjacent).
    Then (distance, index) order is (distance, cid) order, the reference's
    total order (scan.py:55-56), and the plain top-k is exact under distance
    ties for any CIDs — no range pass over the tied distance is needed."""
    order = np.argsort(cids, kind="stable")
    words = _fps1_words(paths)[order]
    lib.close()
    cids = np.ascontiguousarray(cids[order])
    if devices is not None and len(devices) > 1:
        return LibraryGroup.from_words(words, devices, check_padding=False, cids=cids), cids
    return Library.from_words(words, device=devices[0] if devices else None, check_padding=False, cids=cids), cids


def _release(res: _Resident) -> None:
    with _cache_lock:
        res.users -= 1
        if res.evicted and res.users == 0:
            _close(res)


def clear_cache() -> None:
    """Release every resident library (frees HBM); libraries still being
    searched are closed when their last search returns."""
    with _cache_lock:
        for r in _cache.values():
            r.evicted = True
            if r.users == 0:
                _close(r)
        _cache.clear()


def _hits_by_cid(res: _Resident, idx: np.ndarray, dist: np.ndarray, n: int) -> TopK:
    cids = res.cids[idx.astype(np.int64)]
    if len(np.unique(cids)) != len(cids):
        raise DuplicateCid("a cid appears more than once in the library")
    order = np.lexsort((cids, dist))[:n]
    return TopK(capacity=n, hits=tuple(SearchHit(cid=int(cids[i]), distance=int(dist[i])) for i in order))


def _topk_one(res: _Resident, q: np.ndarray, n: int, minq: bool) -> TopK:
    lib = res.lib
    if minq:
        hits = lib.search_min(q, n)
    else:
        hits = lib.search_batch(q, n).hits(0)
    if not hits:
        return TopK(capacity=n, hits=())
    idx = np.array([h[0] for h in hits], dtype=np.uint64)
    dist = np.array([h[1] for h in hits], dtype=np.int64)
    # the resident library is in CID order (_cid_ordered): (distance, index)
    # order is (distance, cid) order
    return _hits_by_cid(res, idx, dist, n)


def _search_multi(manifest, queries: np.ndarray, params: SearchParams, progress: SearchProgressFn | None,
                  cancel: CancelFn | None, minq: bool, device: int | None = None) -> TopK:
    shards = manifest.shards
    if not shards:
        return TopK(capacity=params.n, hits=())
    if cancel is not None and cancel():
        raise ScanCancelled(str(shards[0].path))
    if device is not None:
        devices = (device,)
    else:
        devices = search_devices(sum(int(s.record_count) for s in shards))
    res = _acquire(manifest, devices)
    try:
        if res.lib.n == 0:
            top = TopK(capacity=params.n, hits=())
        else:
            top = _topk_one(res, queries, params.n, minq)
    finally:
        _release(res)
    if progress is not None:
        for shard, a, b in zip(shards, res.offsets, res.offsets[1:]):
            progress(shard.dataset_label, b - a, shard.record_count)
    return top


def search(manifest, query, params: SearchParams, progress: SearchProgressFn | None = None,
           cancel: CancelFn | None = None) -> TopK:
    """Search the whole library (scan.py:290-303); independent of parallelism."""
    return _search_multi(manifest, as_query_words(query)[:1], params, progress, cancel, minq=False)


def batch_search(manifest, queries, params: SearchParams, progress: SearchProgressFn | None = None,
                 cancel: CancelFn | None = None) -> TopK:
    """Nearest-to-query-set search (scan.py:306-318): min over queries."""
    q = as_query_words(list(queries) if not isinstance(queries, np.ndarray) else queries)
    if len(q) == 0:
        raise ValueError("batch_search requires at least one query")
    if len(q) == 1:
        return _search_multi(manifest, q, params, progress, cancel, minq=False)
    return _search_multi(manifest, q, params, progress, cancel, minq=True)


def scan_shard(shard, query, params: SearchParams, progress: ShardProgressFn | None = None,
               cancel: CancelFn | None = None) -> TopK:
    """Top-K over one shard (scan.py:212-222)."""
    from .libstore import ShardManifest

    manifest = ShardManifest(shards=(shard,), total_records=shard.record_count)
    wrapped = None
    if progress is not None:
        wrapped = lambda label, done, total: progress(done)
    try:
        return _search_multi(manifest, as_query_words(query)[:1], params, wrapped, cancel, minq=False)
    except ScanError as exc:
        cause = exc.__cause__
        if isinstance(cause, (OSError, LibstoreError)):
            raise cause
        raise
