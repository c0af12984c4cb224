"""CPU oracle for the fingerprint-scan hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU reference. The product package (``paper_1906_06170_b200``) never
imports it; its scan path is CUDA-only and fails loudly without the extension.

This is a numpy restatement of the reference ``fpscan`` search path
(``/root/reference/pkg/src/fpscan``), function by function:

* distance semantics — ``fingerprint.py:151-158`` (popcount of XOR over three
  u64 words) with the naive per-key oracle ``fingerprint.py:143-148``;
* the block scan — ``scan.py:137-143`` (``_distances_packed``: min over queries
  of ``bitwise_count(words ^ q).sum(axis=1)`` as uint16), ``scan.py:158-170``
  (65,536-record blocks), ``scan.py:173-209`` (``_scan_shard``: lexsort warm-up,
  then the ``d < wd or (d == wd and cid < wc)`` candidate filter into a bounded
  heap, ``scan.py:91-126``);
* shard fan-out and merge — ``scan.py:225-236`` (``merge_topk``),
  ``scan.py:239-287`` (``_search_multi``, one thread per shard) and
  ``libstore.py:174-179`` (``split_sizes``);
* the FPS1 record view — ``libstore.py:5-16``, ``:28-35``, ``:202-212``.

Orderings use (distance, index); the reference orders by (distance, cid) and
its synthetic libraries use cid = index + 1 (``synth.py:37``), so the two
orders coincide. Where a caller supplies explicit cids, they are used as-is.

Two semantics have no reference op:
per-query batch top-k (== one ``search`` per query) and range search (every
(query, index, distance) with distance <= r, sorted by (query, distance,
index)). Both are restated on top of ``_distances_packed`` and pinned through
it (range results must contain every top-k prefix; see tests).

Parity is pinned: ``tests/golden/make_golden.py`` runs the real reference
(importable in the build container) and commits its outputs; the
``-m "not gpu"`` suite checks this module against them.
"""

from __future__ import annotations

import heapq
import os
from concurrent.futures import ThreadPoolExecutor
from typing import Iterable, Sequence

import numpy as np

NUM_KEYS = 166
WORD_COUNT = 3
BLOCK_RECORDS = 65536  # scan.py:29
RECORD_SIZE = 32  # libstore.py:31
HEADER_SIZE = 16  # libstore.py:30
_M64 = (1 << 64) - 1


# --------------------------------------------------------------------------
# scalar distance contract (fingerprint.py:143-158)
# --------------------------------------------------------------------------
def distance_packed(a: Sequence[int], b: Sequence[int]) -> int:
    """popcount(a XOR b) over the three words (fingerprint.py:151-158)."""
    return sum(((int(x) ^ int(y)) & _M64).bit_count() for x, y in zip(a, b))


def manhattan_reference(a: Sequence[int], b: Sequence[int]) -> int:
    """Key-by-key |a_j - b_j| over keys 1..166 (fingerprint.py:143-148)."""
    va = int(a[0]) | (int(a[1]) << 64) | (int(a[2]) << 128)
    vb = int(b[0]) | (int(b[1]) << 64) | (int(b[2]) << 128)
    return sum(abs(((va >> i) & 1) - ((vb >> i) & 1)) for i in range(NUM_KEYS))


# --------------------------------------------------------------------------
# vectorised distance kernel (scan.py:137-143)
# --------------------------------------------------------------------------
def distances_packed(words: np.ndarray, qwords: np.ndarray) -> np.ndarray:
    """Min over queries of popcount(record XOR query), uint16 per record.

    ``words`` is (n, 3) uint64 (may be a strided view of (n, 4) records, as in
    scan.py:169); ``qwords`` is (Q, 3) uint64.
    """
    qwords = np.atleast_2d(np.asarray(qwords, dtype=np.uint64))
    out = None
    for q in qwords:
        d = np.bitwise_count(words ^ q).sum(axis=1, dtype=np.uint16)
        out = d if out is None else np.minimum(out, d, out=out)
    return out


def distances_one(words: np.ndarray, q: np.ndarray) -> np.ndarray:
    """popcount(record XOR q) for one query, uint16 per record."""
    return np.bitwise_count(words ^ np.asarray(q, dtype=np.uint64)).sum(axis=1, dtype=np.uint16)


# --------------------------------------------------------------------------
# bounded heap and block scan (scan.py:91-126, 173-209)
# --------------------------------------------------------------------------
class TopKAccumulator:
    """Bounded max-heap of (-distance, -id) — restates scan.py:91-126."""

    def __init__(self, capacity: int):
        self.capacity = capacity
        self._heap: list[tuple[int, int]] = []

    @property
    def full(self) -> bool:
        return len(self._heap) >= self.capacity

    def worst(self) -> tuple[int, int]:
        d, c = self._heap[0]
        return (-d, -c)

    def offer(self, ident: int, distance: int) -> None:
        entry = (-distance, -ident)
        if len(self._heap) < self.capacity:
            heapq.heappush(self._heap, entry)
        elif entry > self._heap[0]:
            heapq.heapreplace(self._heap, entry)

    def result(self) -> list[tuple[int, int]]:
        """Sorted [(id, distance)] ascending under (distance, id)."""
        return [(-c, -d) for d, c in sorted(self._heap, reverse=True)]


def iter_blocks(words: np.ndarray, ids: np.ndarray) -> Iterable[tuple[np.ndarray, np.ndarray]]:
    """Fixed 65,536-record blocks (scan.py:158-170), from memory instead of a file."""
    n = len(words)
    for s in range(0, n, BLOCK_RECORDS):
        yield ids[s : s + BLOCK_RECORDS], words[s : s + BLOCK_RECORDS]


def scan_shard(words: np.ndarray, qwords: np.ndarray, k: int, ids: np.ndarray | None = None,
               blocks: Iterable[tuple[np.ndarray, np.ndarray]] | None = None) -> list[tuple[int, int]]:
    """The reference block scan (scan.py:173-209) over one shard.

    Returns [(id, distance)] sorted by (distance, id); ``ids`` default to the
    row index. ``qwords`` may hold several queries (min-over-queries,
    scan.py:137-143), which is the reference ``batch_search`` semantics.
    """
    if k < 1:
        raise ValueError("n must be >= 1")
    if ids is None and blocks is None:
        ids = np.arange(len(words), dtype=np.uint64)
    qwords = np.atleast_2d(np.asarray(qwords, dtype=np.uint64))
    acc = TopKAccumulator(k)
    for bids, bwords in (blocks if blocks is not None else iter_blocks(words, ids)):
        d = distances_packed(bwords, qwords)
        if not acc.full:
            for i in np.lexsort((bids, d))[:k]:
                acc.offer(int(bids[i]), int(d[i]))
        else:
            wd, wc = acc.worst()
            cand = np.flatnonzero((d < wd) | ((d == wd) & (bids < np.uint64(wc))))
            for i in cand:
                acc.offer(int(bids[i]), int(d[i]))
    return acc.result()


def merge_topk(parts: Sequence[Sequence[tuple[int, int]]], k: int) -> list[tuple[int, int]]:
    """Union, duplicate check, sort, truncate (scan.py:225-236)."""
    seen: set[int] = set()
    merged = []
    for part in parts:
        for ident, d in part:
            if ident in seen:
                raise ValueError(f"duplicate id {ident} across parts")
            seen.add(ident)
            merged.append((d, ident))
    merged.sort()
    return [(i, d) for d, i in merged[:k]]


def split_sizes(total: int, shard_count: int) -> list[int]:
    """Contiguous split, sizes differ by <= 1 (libstore.py:174-179)."""
    if shard_count < 1:
        raise ValueError("shard_count must be >= 1")
    base, extra = divmod(total, shard_count)
    return [base + (1 if i < extra else 0) for i in range(shard_count)]


def search(words: np.ndarray, qwords: np.ndarray, k: int, shard_count: int = 1,
           parallelism: int = 1) -> list[tuple[int, int]]:
    """``_search_multi`` restated (scan.py:239-287): contiguous shards, one
    worker per shard (ThreadPoolExecutor, numpy releases the GIL), merged."""
    n = len(words)
    sizes = split_sizes(n, shard_count)
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    ids = np.arange(n, dtype=np.uint64)

    def run(s: int):
        a, b = offs[s], offs[s + 1]
        return scan_shard(words[a:b], qwords, k, ids[a:b])

    if n == 0:
        return []
    if parallelism == 1 or shard_count == 1:
        parts = [run(s) for s in range(shard_count)]
    else:
        with ThreadPoolExecutor(max_workers=min(parallelism, shard_count)) as pool:
            parts = list(pool.map(run, range(shard_count)))
    return merge_topk(parts, k)


# --------------------------------------------------------------------------
# full-sort oracles (test_scan.py:48-58 pattern) and the two non-reference ops
# --------------------------------------------------------------------------
def topk_full_sort(words: np.ndarray, q: np.ndarray, k: int) -> list[tuple[int, int]]:
    """Materialise every distance, sort by (distance, index), truncate."""
    d = distances_one(words, q)
    idx = np.arange(len(words))
    order = np.lexsort((idx, d))[:k]
    return [(int(i), int(d[i])) for i in order]


def batch_topk(words: np.ndarray, queries: np.ndarray, k: int) -> list[list[tuple[int, int]]]:
    """Per-query top-k (config 4): exactly one reference ``search`` per query."""
    return [topk_full_sort(words, q, k) for q in np.atleast_2d(queries)]


def batch_min_topk(words: np.ndarray, queries: np.ndarray, k: int) -> list[tuple[int, int]]:
    """Reference ``batch_search`` semantics (scan.py:306-318): min over queries."""
    d = distances_packed(words, queries)
    idx = np.arange(len(words))
    order = np.lexsort((idx, d))[:k]
    return [(int(i), int(d[i])) for i in order]


def range_search(words: np.ndarray, queries: np.ndarray, radius) -> np.ndarray:
    """All (query, index, distance) with distance <= radius[q], sorted by
    (query, distance, index). Returns an (m, 3) int64 array.

    ``radius`` is a scalar or one value per query. Restated on the reference
    distance kernel (scan.py:137-143); there is no reference range op.
    """
    queries = np.atleast_2d(np.asarray(queries, dtype=np.uint64))
    radii = np.broadcast_to(np.asarray(radius, dtype=np.int64), (len(queries),))
    out = []
    for qi, q in enumerate(queries):
        rows = []
        for s in range(0, len(words), BLOCK_RECORDS):
            d = distances_one(words[s : s + BLOCK_RECORDS], q)
            hit = np.flatnonzero(d <= radii[qi])
            if len(hit):
                rows.append(np.stack([np.full(len(hit), qi), hit + s, d[hit]], axis=1))
        if rows:
            r = np.concatenate(rows).astype(np.int64)
            r = r[np.lexsort((r[:, 1], r[:, 2]))]
            out.append(r)
    return np.concatenate(out) if out else np.zeros((0, 3), dtype=np.int64)


# --------------------------------------------------------------------------
# FPS1 records (libstore.py:5-16, :158-164, :202-212) and synthetic words
# --------------------------------------------------------------------------
def records_from_words(words: np.ndarray, cids: np.ndarray | None = None) -> np.ndarray:
    """(n, 4) '<u8' record view: col 0 CID, cols 1..3 the fingerprint words.

    Bytes 8..28 of a record are the 21 packed fingerprint bytes and bytes
    29..31 are zero, so cols 1..3 equal ``Fingerprint.words`` for any valid
    fingerprint (libstore.py:158-164, scan.py:169).
    """
    n = len(words)
    rec = np.zeros((n, 4), dtype="<u8")
    rec[:, 0] = np.arange(1, n + 1, dtype=np.uint64) if cids is None else cids
    rec[:, 1:4] = words
    return rec


def read_fps1(path) -> np.ndarray:
    """Read an FPS1 shard into its (n, 4) record view (libstore.py:202-212)."""
    raw = np.fromfile(path, dtype=np.uint8)
    if len(raw) < HEADER_SIZE or bytes(raw[:4]) != b"FPS1":
        raise ValueError(f"{path}: bad FPS1 header")
    count = int(raw[8:16].view("<u8")[0])
    body = raw[HEADER_SIZE : HEADER_SIZE + count * RECORD_SIZE]
    if len(body) != count * RECORD_SIZE:
        raise ValueError(f"{path}: truncated")
    return body.view("<u8").reshape(count, 4)


_GOLDEN = 0x9E3779B97F4A7C15


def _splitmix64_finalize(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def generate_words(seed_key: int, thresholds: np.ndarray, start: int, count: int) -> np.ndarray:
    """numpy twin of the device generator ``fps_generate`` (csrc/fps_gen.cu).

    Entry i, key j (1-based) is set iff u32(i, j) < thresholds[j-1], where
    u32 is half of h(i, c) = splitmix64(seed_key + (i*83 + c) * golden),
    c = (j-1) >> 1 (low half for odd j, high half for even j).
    """
    thr = np.asarray(thresholds, dtype=np.uint64)
    i = np.arange(start, start + count, dtype=np.uint64)[:, None]
    c = np.arange(83, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        ctr = i * np.uint64(83) + c
        z = np.uint64(seed_key) + (ctr + np.uint64(1)) * np.uint64(_GOLDEN)
        h = _splitmix64_finalize(z)
    lo = h & np.uint64(0xFFFFFFFF)
    hi = h >> np.uint64(32)
    u = np.empty((count, 166), dtype=np.uint64)
    u[:, 0::2] = lo
    u[:, 1::2] = hi
    bits = (u < thr[None, :]).astype(np.uint64)
    words = np.zeros((count, 3), dtype=np.uint64)
    for w in range(3):
        seg = bits[:, 64 * w : 64 * (w + 1)]
        sh = np.arange(seg.shape[1], dtype=np.uint64)
        words[:, w] = np.bitwise_or.reduce(seg << sh[None, :], axis=1)
    return words


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# --------------------------------------------------------------------------
# C restatement (oracle/fps_oracle.c -> oracle/_ref/libfps_oracle.so)
# --------------------------------------------------------------------------
import ctypes as _C
import json as _json
import subprocess as _sp
from pathlib import Path as _Path

_ORACLE_DIR = _Path(__file__).resolve().parent
_ORACLE_SO = _ORACLE_DIR / "_ref" / "libfps_oracle.so"
_clib = None


def build_c() -> _Path:
    """Compile the C restatement with the committed Makefile."""
    src = _ORACLE_DIR / "fps_oracle.c"
    if not _ORACLE_SO.exists() or _ORACLE_SO.stat().st_mtime < src.stat().st_mtime:
        _sp.run(["make", "-s", "-C", str(_ORACLE_DIR)], check=True)
    return _ORACLE_SO


def _lib():
    global _clib
    if _clib is None:
        build_c()
        lib = _C.CDLL(str(_ORACLE_SO))
        vp = _C.c_void_p
        lib.orc_topk.argtypes = [vp, vp, vp, _C.c_int64, _C.c_uint64, vp, _C.c_uint32, _C.c_uint32, _C.c_int,
                                 vp, vp, vp]
        lib.orc_range.argtypes = [vp, vp, vp, _C.c_int64, _C.c_uint64, vp, _C.c_uint32, vp, _C.c_int,
                                  _C.POINTER(vp), _C.POINTER(_C.c_uint64)]
        lib.orc_free.argtypes = [vp]
        lib.orc_fnv1a_64.argtypes = [vp, _C.c_uint64, _C.c_uint64]
        lib.orc_fnv1a_64.restype = _C.c_uint64
        lib.orc_generate.argtypes = [_C.c_uint64, vp, _C.c_uint64, _C.c_uint64, _C.c_int, vp]
        _clib = lib
    return _clib


def _planes(words):
    """(w0, w1, w2, stride) pointers for an (n, 3) / (n, 4)-record array or a
    tuple of three plane arrays."""
    if isinstance(words, tuple):
        a, b, c = (np.ascontiguousarray(x, dtype=np.uint64) for x in words)
        return (a, b, c), a.ctypes.data, b.ctypes.data, c.ctypes.data, 1, len(a)
    w = np.asarray(words)
    if w.dtype != np.uint64 and w.dtype != np.dtype("<u8"):
        w = w.astype(np.uint64)
    if not w.flags.c_contiguous:
        w = np.ascontiguousarray(w)
    base = w.ctypes.data
    if w.shape[1] == 3:
        return (w,), base, base + 8, base + 16, 3, len(w)
    if w.shape[1] == 4:  # FPS1 record view: col 0 is the cid
        return (w,), base + 8, base + 16, base + 24, 4, len(w)
    raise ValueError(f"words must be (n, 3) or (n, 4), got {w.shape}")


def c_topk(words, queries, k: int, threads: int | None = None):
    """Exact per-query top-k in C: returns (idx (Q,k) uint64, dist (Q,k) uint16, cnt (Q,))."""
    keep, p0, p1, p2, stride, n = _planes(words)
    q = np.ascontiguousarray(np.atleast_2d(np.asarray(queries, dtype=np.uint64)))
    Q = len(q)
    idx = np.full((Q, k), np.iinfo(np.uint64).max, dtype=np.uint64)
    dist = np.full((Q, k), 0xFFFF, dtype=np.uint16)
    cnt = np.zeros(Q, dtype=np.uint32)
    rc = _lib().orc_topk(p0, p1, p2, stride, n, q.ctypes.data, Q, k, threads or cpu_threads(), idx.ctypes.data,
                         dist.ctypes.data, cnt.ctypes.data)
    if rc:
        raise RuntimeError(f"orc_topk failed: {rc}")
    del keep
    return idx, dist, cnt


def c_range(words, queries, radius, threads: int | None = None) -> np.ndarray:
    """Range search in C: (m, 3) int64 rows (query, index, distance), sorted."""
    keep, p0, p1, p2, stride, n = _planes(words)
    q = np.ascontiguousarray(np.atleast_2d(np.asarray(queries, dtype=np.uint64)))
    rad = np.ascontiguousarray(np.broadcast_to(np.asarray(radius, dtype=np.uint8), (len(q),)))
    out = _C.c_void_p()
    m = _C.c_uint64()
    rc = _lib().orc_range(p0, p1, p2, stride, n, q.ctypes.data, len(q), rad.ctypes.data, threads or cpu_threads(),
                          _C.byref(out), _C.byref(m))
    if rc:
        raise RuntimeError(f"orc_range failed: {rc}")
    try:
        keys = np.ctypeslib.as_array(_C.cast(out, _C.POINTER(_C.c_uint64)), shape=(m.value,)).copy() \
            if m.value else np.zeros(0, np.uint64)
    finally:
        _lib().orc_free(out)
    del keep
    return range_keys_to_rows(keys)


def range_keys_to_rows(keys: np.ndarray) -> np.ndarray:
    keys = np.asarray(keys, dtype=np.uint64)
    return np.stack([(keys >> np.uint64(48)).astype(np.int64),
                     (keys & np.uint64((1 << 40) - 1)).astype(np.int64),
                     ((keys >> np.uint64(40)) & np.uint64(0xFF)).astype(np.int64)], axis=1)


def fnv1a_64(data: bytes | np.ndarray, value: int = 0xCBF29CE484222325) -> int:
    """64-bit FNV-1a (libstore.py:93-98), in C for library-sized inputs."""
    buf = np.frombuffer(data, dtype=np.uint8) if isinstance(data, (bytes, bytearray)) else \
        np.ascontiguousarray(data).view(np.uint8).reshape(-1)
    return int(_lib().orc_fnv1a_64(buf.ctypes.data, buf.size, value))


def write_fps1_library(out_dir, words: np.ndarray, shard_count: int, cids: np.ndarray | None = None):
    """Write FPS1 shards + manifest.json that the unmodified reference
    ``fpscan.libstore.load_manifest`` / ``scan.search`` read (libstore.py:5-16,
    :182-199, :279-300). Returns the manifest path."""
    out_dir = _Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    rec = records_from_words(words, cids)
    shards = []
    off = 0
    for i, size in enumerate(split_sizes(len(rec), shard_count)):
        name = f"shard-{i:03d}.fps"
        region = rec[off:off + size]
        header = b"FPS1" + (1).to_bytes(2, "little") + b"\0\0" + int(size).to_bytes(8, "little")
        with open(out_dir / name, "wb") as f:
            f.write(header)
            region.tofile(f)
        letter = chr(ord("A") + i % 26)
        label = letter if i < 26 else f"{letter}{i // 26}"
        shards.append({"path": name, "dataset_label": label, "record_count": int(size),
                       "checksum": f"{fnv1a_64(region):016x}"})
        off += size
    doc = {"format_version": 1, "total_records": int(len(rec)), "shards": shards}
    path = out_dir / "manifest.json"
    path.write_text(_json.dumps(doc, indent=2) + "\n", encoding="utf-8")
    return path


# --------------------------------------------------------------------------
# file-streaming restatement: the reference reads FPS1 shards per search
# (scan.py:158-170) with one worker thread per shard (scan.py:256-287)
# --------------------------------------------------------------------------
def iter_fps1_blocks(path):
    """(ids, words) blocks of 65,536 records read with f.read, as scan.py:158-170."""
    with open(path, "rb") as f:
        head = f.read(HEADER_SIZE)
        if len(head) < HEADER_SIZE or head[:4] != b"FPS1":
            raise ValueError(f"{path}: bad FPS1 header")
        count = int.from_bytes(head[8:16], "little")
        remaining = count
        while remaining > 0:
            n = min(remaining, BLOCK_RECORDS)
            buf = f.read(n * RECORD_SIZE)
            if len(buf) < n * RECORD_SIZE:
                raise ValueError(f"{path}: truncated")
            block = np.frombuffer(buf, dtype="<u8").reshape(n, 4)
            yield block[:, 0], block[:, 1:4]
            remaining -= n


def search_fps1(manifest_path, qwords, k: int, parallelism: int = 1) -> list[tuple[int, int]]:
    """The reference ``search`` restated over FPS1 files: per-shard block scan
    (ids are the stored CIDs) on a thread pool, then merge_topk."""
    doc = _json.loads(_Path(manifest_path).read_text())
    base = _Path(manifest_path).parent
    paths = [base / s["path"] for s in doc["shards"]]

    def run(p):
        return scan_shard(None, qwords, k, blocks=iter_fps1_blocks(p))

    if not paths:
        return []
    if parallelism == 1 or len(paths) == 1:
        parts = [run(p) for p in paths]
    else:
        with ThreadPoolExecutor(max_workers=min(parallelism, len(paths))) as pool:
            parts = list(pool.map(run, paths))
    return merge_topk(parts, k)


def generate_words_parallel(seed_key: int, thresholds: np.ndarray, start: int, count: int,
                            threads: int | None = None, chunk: int = 1 << 18) -> np.ndarray:
    """generate_words for a whole library: the C twin (orc_generate) on all
    host threads; same words as the numpy generate_words (pinned by tests)."""
    out = np.empty((count, 3), dtype=np.uint64)
    thr = np.ascontiguousarray(np.asarray(thresholds, dtype=np.uint64))
    if count:
        rc = _lib().orc_generate(seed_key & _M64, thr.ctypes.data, start, count, threads or cpu_threads(),
                                 out.ctypes.data)
        if rc:
            raise RuntimeError("orc_generate failed")
    return out
