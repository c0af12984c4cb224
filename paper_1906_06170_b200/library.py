"""The north-star search surface: an HBM-resident library and its queries.

``load_library(source) -> Library`` uploads once; ``Library.search``,
``search_batch`` and ``range_search`` return (index, distance) results in the
reference total order (distance, then index; scan.py:55-56). Every scan runs
in libfpsgpu.so (CUDA, sm_100a) through the C ABI of include/fps.h.

Replaces, for the hot path, the reference's per-search shard streaming and
numpy kernel (/root/reference/pkg/src/fpscan/scan.py:137-209, :239-318).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path
from typing import Sequence

import numpy as np

from . import _native as N
from .fingerprint import as_query_words

_U64_MAX = np.uint64(0xFFFFFFFFFFFFFFFF)
IDX_MASK = (1 << 40) - 1


@dataclass(frozen=True)
class RangeResult:
    """Range hits sorted by (query, distance, index)."""

    query: np.ndarray     # uint32
    index: np.ndarray     # uint64 (global library index)
    distance: np.ndarray  # uint16

    def __len__(self) -> int:
        return len(self.index)

    @staticmethod
    def from_keys(keys: np.ndarray) -> "RangeResult":
        keys = np.asarray(keys, dtype=np.uint64)
        return RangeResult(
            query=(keys >> np.uint64(48)).astype(np.uint32),
            index=keys & np.uint64(IDX_MASK),
            distance=((keys >> np.uint64(40)) & np.uint64(0xFF)).astype(np.uint16),
        )

    def rows(self) -> np.ndarray:
        """(m, 3) int64 array of (query, index, distance)."""
        return np.stack([self.query.astype(np.int64), self.index.astype(np.int64),
                         self.distance.astype(np.int64)], axis=1)


_U64 = np.dtype(np.uint64)
_topk = None


def _topk_fn():
    global _topk
    if _topk is None:
        _topk = N.load().fps_topk
    return _topk


@dataclass(slots=True)
class TopKResult:
    """Per-query top-k: row q holds count[q] valid (index, distance) pairs."""

    index: np.ndarray     # (Q, k) uint64, UINT64_MAX in unused slots
    distance: np.ndarray  # (Q, k) uint16, 0xFFFF in unused slots
    count: np.ndarray     # (Q,) uint32

    def hits(self, q: int) -> list[tuple[int, int]]:
        c = int(self.count[q])
        return [(int(i), int(d)) for i, d in zip(self.index[q, :c], self.distance[q, :c])]


class Library:
    """A fingerprint library resident in one GPU's HBM as three u64 planes."""

    def __init__(self, handle: int, cids: np.ndarray | None = None, borrowed: bool = False):
        self._h = C.c_void_p(handle)
        self._borrowed = borrowed  # a shard of a LibraryGroup: closed by the group
        n, base, dev = C.c_uint64(), C.c_uint64(), C.c_int()
        N.check(N.load().fps_info(self._h, C.byref(n), C.byref(base), C.byref(dev)), "fps_info")
        self.n = n.value
        self.index_base = base.value
        self.device = dev.value
        self.cids = cids
        self._cids_monotone = None

    # ---- construction -------------------------------------------------
    @staticmethod
    def _device(device: int | None) -> int:
        N.require_device()
        if device is None:
            try:
                import torch

                return torch.cuda.current_device()
            except Exception:  # pragma: no cover - torch missing
                return 0
        return int(device)

    @classmethod
    def from_words(cls, words, device: int | None = None, index_base: int = 0, check_padding: bool = True,
                   cids: np.ndarray | None = None) -> "Library":
        """Upload an (n, 3) uint64 word array (Fingerprint.words per row)."""
        arr = np.ascontiguousarray(np.asarray(words, dtype=np.uint64).reshape(-1, 3))
        h = C.c_void_p()
        N.check(N.load().fps_open(arr.ctypes.data, len(arr), N.LAYOUT_ROWS3, cls._device(device), index_base,
                                  int(check_padding), C.byref(h)), "fps_open")
        return cls(h.value, cids)

    @classmethod
    def from_records(cls, records: np.ndarray, device: int | None = None, index_base: int = 0) -> "Library":
        """Upload an (n, 4) '<u8' FPS1 record view (cid, w0, w1, w2) — scan.py:169.

        Words are scanned exactly as stored (the reference scan does not
        validate padding, so neither does this)."""
        rec = np.ascontiguousarray(np.asarray(records, dtype=np.uint64).reshape(-1, 4))
        h = C.c_void_p()
        N.check(N.load().fps_open(rec.ctypes.data, len(rec), N.LAYOUT_FPS1, cls._device(device), index_base, 0,
                                  C.byref(h)), "fps_open")
        return cls(h.value, rec[:, 0].copy())

    @classmethod
    def from_fps1(cls, paths, start: int = 0, count: int | None = None, device: int | None = None,
                  with_cids: bool = True) -> "Library":
        """Stream FPS1 shard files (in order) into HBM; only records
        [start, start + count) of their concatenation are loaded (one rank's
        slice). Headers are validated first: a bad shard raises ScanError
        naming its path (scan.py:283-284)."""
        paths = [str(p) for p in paths]
        arr = (C.c_char_p * max(1, len(paths)))(*[p.encode() for p in paths])
        total = None
        if with_cids or count is None:
            total = sum(_fps1_count(p) for p in paths)
        n = (total - start) if count is None else count
        if total is not None:
            n = max(0, min(n, total - start))
        cids = np.empty(n, dtype=np.uint64) if with_cids else None
        h = C.c_void_p()
        dev = cls._device(device) if paths else cls._device(device)
        N.check(N.load().fps_open_fps1(arr, len(paths), start, n if count is not None or total is not None
                                       else (1 << 64) - 1, dev, cids.ctypes.data if cids is not None else None,
                                       C.byref(h)), "fps_open_fps1")
        return cls(h.value, cids)

    @classmethod
    def from_device_planes(cls, w0, w1, w2, device: int | None = None, index_base: int = 0) -> "Library":
        """Copy three device planes (torch int64/uint64 tensors or pointers)."""
        n = int(w0.numel()) if hasattr(w0, "numel") else None
        if n is None:
            raise ValueError("from_device_planes needs tensors")
        h = C.c_void_p()
        dev = w0.device.index if hasattr(w0, "device") and w0.device.index is not None else cls._device(device)
        N.check(N.load().fps_open_device(N.ptr(w0), N.ptr(w1), N.ptr(w2), n, dev, index_base, C.byref(h)),
                "fps_open_device")
        return cls(h.value)

    @classmethod
    def generate(cls, n: int, seed_key: int, thresholds: np.ndarray, device: int | None = None, start: int = 0,
                 index_base: int | None = None) -> "Library":
        """Synthetic library generated on the device (see synth.py)."""
        thr = np.asarray(thresholds, dtype=np.uint64)
        thr32 = np.minimum(thr, np.uint64(0xFFFFFFFF)).astype(np.uint32)
        allset = (thr > np.uint64(0xFFFFFFFF)).astype(np.uint8)
        h = C.c_void_p()
        N.check(N.load().fps_open_generated(n, start, seed_key & ((1 << 64) - 1), thr32.ctypes.data,
                                            allset.ctypes.data, cls._device(device),
                                            start if index_base is None else index_base, C.byref(h)),
                "fps_open_generated")
        return cls(h.value)

    def close(self) -> None:
        if self._h and self._h.value:
            if not self._borrowed:
                N.load().fps_close(self._h)
            self._h = C.c_void_p()

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---- data access ----------------------------------------------------
    def layout(self) -> tuple[bool, int]:
        """(compact, bytes per entry) of the HBM planes."""
        c, b = C.c_int(), C.c_uint64()
        N.check(N.load().fps_layout(self._h, C.byref(c), C.byref(b)), "fps_layout")
        return bool(c.value), int(b.value)

    def read_entries(self, start: int = 0, count: int | None = None) -> np.ndarray:
        """Copy entries back as (count, 3) uint64 rows (checking / export)."""
        count = self.n - start if count is None else count
        rows = np.empty((count, 3), dtype=np.uint64)
        if count:
            N.check(N.load().fps_read_entries(self._h, start, count, rows.ctypes.data), "fps_read_entries")
        return rows

    def words_host(self) -> np.ndarray:
        """The whole library as (n, 3) uint64 (for checking only)."""
        return self.read_entries()

    def write_entries(self, index: np.ndarray, words: np.ndarray) -> None:
        """Overwrite local entries ``index`` with rows of ``words``."""
        idx = np.ascontiguousarray(np.asarray(index, dtype=np.uint64))
        w = np.ascontiguousarray(np.asarray(words, dtype=np.uint64).reshape(-1, 3))
        if len(idx) != len(w):
            raise ValueError("index and words differ in length")
        N.check(N.load().fps_write_entries(self._h, idx.ctypes.data, w.ctypes.data, len(idx)), "fps_write_entries")

    def memory(self) -> dict:
        """HBM bytes held (library tiles, derived copies, scratch) and the
        host time spent building the derived copies."""
        a, b, c, t = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_double()
        N.check(N.load().fps_memory(self._h, C.byref(a), C.byref(b), C.byref(c), C.byref(t)), "fps_memory")
        return {"library_bytes": a.value, "derived_bytes": b.value, "scratch_bytes": c.value,
                "derived_build_ms": t.value}

    def release_derived(self) -> None:
        """Free the derived plane copies (rebuilt on next use)."""
        N.check(N.load().fps_release_derived(self._h), "fps_release_derived")

    def timing(self, enable: bool) -> None:
        N.check(N.load().fps_timing(self._h, int(enable)), "fps_timing")

    def timing_read(self) -> tuple[float, int]:
        """(summed scan-kernel ms, launches) since the last read."""
        t, c = C.c_double(), C.c_uint64()
        N.check(N.load().fps_timing_read(self._h, C.byref(t), C.byref(c)), "fps_timing_read")
        return t.value, c.value

    KERNELS = {0: "none", 1: "single-query HBM scan", 2: "multi-query POPC scan", 3: "bit-sliced multi-query scan",
               4: "large-k histogram/range/sort", 5: "single-query plane scan",
               6: "tensor-core multi-query scan"}

    @property
    def last_kernel(self) -> str:
        return self.KERNELS.get(int(N.load().fps_last_kernel(self._h)), "unknown")

    MMA_KINDS = {0: None, 1: "i8", 2: "fp4", 3: "fp4x"}

    @property
    def last_mma_kind(self) -> str | None:
        """Operand kind of the last tensor-core scan: "i8", "fp4" or "fp4x"."""
        return self.MMA_KINDS.get(int(N.load().fps_last_mma_kind(self._h)))

    @property
    def mma_overflowed(self) -> bool:
        """True if the last tensor-core top-k overflowed a candidate list and ran
        its exact fallback pass (diagnostic; synchronises the device)."""
        f = C.c_int(0)
        N.check(N.load().fps_mma_overflowed(self._h, C.byref(f)), "fps_mma_overflowed")
        return bool(f.value)

    @property
    def launches(self) -> int:
        return int(N.load().fps_launch_count(self._h))

    # ---- queries ----------------------------------------------------------
    def search_batch(self, queries, k: int) -> TopKResult:
        """Per-query top-k, one independent search per query (config 4)."""
        if (type(queries) is np.ndarray and queries.dtype == _U64 and queries.ndim == 2
                and queries.shape[1] == 3 and queries.flags.c_contiguous):
            q = queries  # fast path: padding bits are validated by fps_topk (FPS_EPADDING)
        else:
            q = as_query_words(queries)
        if k < 1:
            raise ValueError("n must be >= 1")
        Q = len(q)
        # one host block for the three outputs: a single allocation and one
        # address lookup per call (this is on the latency-critical path)
        blk = np.empty(Q * k * 10 + Q * 4 + 8, dtype=np.uint8)
        base = C.addressof(C.c_char.from_buffer(blk))
        idx = np.ndarray((Q, k), np.uint64, blk, 0)
        dist = np.ndarray((Q, k), np.uint16, blk, Q * k * 8)
        cnt = np.ndarray((Q,), np.uint32, blk, Q * k * 10)
        if Q:
            try:
                qp = C.addressof(C.c_char.from_buffer(q))
            except (TypeError, ValueError):  # read-only query array
                qp = q.ctypes.data
            rc = _topk_fn()(self._h, qp, Q, k, base, base + Q * k * 8, base + Q * k * 10)
            if rc:
                N.check(rc, "fps_topk")
        else:
            cnt[:] = 0
        return TopKResult(idx, dist, cnt)

    def search(self, query, k: int) -> list[tuple[int, int]]:
        """Top-k [(index, distance)] for one query (reference ``search``)."""
        return self.search_batch(query, k).hits(0)

    def search_min(self, queries, k: int) -> list[tuple[int, int]]:
        """Reference ``batch_search``: min over queries, one top-k."""
        q = as_query_words(queries)
        if len(q) == 0:
            raise ValueError("batch_search requires at least one query")
        idx = np.empty((1, k), dtype=np.uint64)
        dist = np.empty((1, k), dtype=np.uint16)
        cnt = np.zeros(1, dtype=np.uint32)
        N.check(N.load().fps_topk_min(self._h, q.ctypes.data, len(q), k, idx.ctypes.data, dist.ctypes.data,
                                      cnt.ctypes.data), "fps_topk_min")
        return TopKResult(idx, dist, cnt).hits(0)

    def range_begin(self, queries, radius) -> int:
        """Scan + device sort of the range hits, left on the device (their
        count is returned); ``range_search`` also fetches them."""
        q = as_query_words(queries)
        rad = np.ascontiguousarray(np.minimum(np.broadcast_to(np.asarray(radius, dtype=np.int64), (len(q),)),
                                              254).astype(np.uint8))
        n_out = C.c_uint64()
        N.check(N.load().fps_range_begin(self._h, q.ctypes.data, len(q), rad.ctypes.data, C.byref(n_out)),
                "fps_range_begin")
        return n_out.value

    def range_search(self, queries, radius) -> RangeResult:
        """Every (query, index, distance) with distance <= radius (scalar or per query)."""
        q = as_query_words(queries)
        Q = len(q)
        r = np.broadcast_to(np.asarray(radius, dtype=np.int64), (Q,))
        if np.any(r < 0):
            raise ValueError("radius must be >= 0")
        rad = np.ascontiguousarray(np.minimum(r, 254).astype(np.uint8))
        n_out = C.c_uint64()
        if Q == 0:
            return RangeResult.from_keys(np.zeros(0, np.uint64))
        lib = N.load()
        # scan + device sort, then the sorted hits straight into the result
        # columns through a pinned double buffer (no intermediate key array)
        N.check(lib.fps_range_begin(self._h, q.ctypes.data, Q, rad.ctypes.data, C.byref(n_out)), "fps_range_begin")
        m = n_out.value
        query = np.empty(m, np.uint32)
        index = np.empty(m, np.uint64)
        distance = np.empty(m, np.uint16)
        N.check(lib.fps_range_fetch(self._h, query.ctypes.data, index.ctypes.data, distance.ctypes.data, m),
                "fps_range_fetch")
        return RangeResult(query=query, index=index, distance=distance)

    # ---- stream-ordered device API --------------------------------------
    def topk_prepare(self, Q: int, k: int) -> None:
        N.check(N.load().fps_topk_prepare(self._h, Q, k), "fps_topk_prepare")

    def topk_async(self, d_queries, Q: int, k: int, d_keys, d_cnt, stream: int) -> None:
        N.check(N.load().fps_topk_async(self._h, N.ptr(d_queries), Q, k, N.ptr(d_keys), N.ptr(d_cnt), stream),
                "fps_topk_async")

    def query_hint(self, query=None) -> None:
        """Host copy of the single device-resident query the next ``topk_async``
        calls scan (sizes the plane scan to its plane list); None forgets it."""
        if query is None:
            N.check(N.load().fps_query_hint(self._h, None), "fps_query_hint")
            return
        q = np.ascontiguousarray(as_query_words(query)[:1])
        N.check(N.load().fps_query_hint(self._h, q.ctypes.data), "fps_query_hint")

    def range_async(self, d_queries, Q: int, d_radius, d_out, cap: int, d_count, stream: int) -> None:
        N.check(N.load().fps_range_async(self._h, N.ptr(d_queries), Q, N.ptr(d_radius), N.ptr(d_out), cap,
                                         N.ptr(d_count), stream), "fps_range_async")

    def sort_keys(self, d_keys, n: int, stream: int) -> None:
        N.check(N.load().fps_sort_keys(self._h, N.ptr(d_keys), n, stream), "fps_sort_keys")


class LibraryGroup:
    """One library over several GPUs of this process (include/fps.h fps_group_*).

    Contiguous shards (``split_sizes``, libstore.py:174-179), shard i on
    ``devices[i]`` with global indices; every shard scans concurrently on its
    own device and the root (devices[0]) gathers and merges — the merge kernel
    reads the shard results straight from peer HBM (``gather="p2p"``), or
    after an NCCL send/recv (``"nccl"``) or peer copies (``"copy"``). Results
    equal a single Library over the whole library (merge_topk semantics,
    scan.py:225-236). Same query methods as Library.
    """

    GATHERS = {v: k for k, v in N.GATHER_NAMES.items()}

    def __init__(self, handle: int, cids: np.ndarray | None = None):
        self._h = C.c_void_p(handle)
        n, ns, root, gather = C.c_uint64(), C.c_uint32(), C.c_int(), C.c_int()
        N.check(N.load().fps_group_info(self._h, C.byref(n), C.byref(ns), C.byref(root), C.byref(gather)),
                "fps_group_info")
        self.n = n.value
        self.device = root.value
        self.gather = self.GATHERS.get(gather.value, str(gather.value))
        self.cids = cids
        self.shards: list[Library] = []
        for i in range(ns.value):
            h = C.c_void_p()
            N.check(N.load().fps_group_shard(self._h, i, C.byref(h)), "fps_group_shard")
            self.shards.append(Library(h.value, borrowed=True))
        self.index_base = self.shards[0].index_base
        self.devices = [s.device for s in self.shards]

    # ---- construction -------------------------------------------------
    @staticmethod
    def _gather(gather) -> int:
        if isinstance(gather, int):
            return gather
        try:
            return N.GATHER_NAMES[gather]
        except KeyError:
            raise ValueError(f"unknown gather mode {gather!r} (auto, p2p, nccl, copy)") from None

    @classmethod
    def from_shards(cls, shards: Sequence[Library], gather="auto", cids: np.ndarray | None = None) -> "LibraryGroup":
        """Bind already-open contiguous shard Libraries; the group takes them over."""
        arr = (C.c_void_p * len(shards))(*[s._h.value for s in shards])
        h = C.c_void_p()
        N.check(N.load().fps_group_open(arr, len(shards), cls._gather(gather), C.byref(h)), "fps_group_open")
        for s in shards:  # now owned by the group
            s._borrowed = True
        return cls(h.value, cids)

    @classmethod
    def from_words(cls, words, devices: Sequence[int], check_padding: bool = True, gather="auto",
                   cids: np.ndarray | None = None) -> "LibraryGroup":
        from .libstore import split_sizes

        arr = np.ascontiguousarray(np.asarray(words, dtype=np.uint64).reshape(-1, 3))
        return cls._split(lambda a, b, dev: Library.from_words(arr[a:b], dev, a, check_padding),
                          len(arr), devices, gather, cids, split_sizes)

    @classmethod
    def from_records(cls, records: np.ndarray, devices: Sequence[int], gather="auto") -> "LibraryGroup":
        from .libstore import split_sizes

        rec = np.ascontiguousarray(np.asarray(records, dtype=np.uint64).reshape(-1, 4))
        return cls._split(lambda a, b, dev: Library.from_records(rec[a:b], dev, a), len(rec), devices, gather,
                          rec[:, 0].copy(), split_sizes)

    @classmethod
    def from_fps1(cls, paths, devices: Sequence[int], gather="auto", with_cids: bool = True) -> "LibraryGroup":
        """Stream FPS1 shard files into one contiguous slice per device (all
        devices load concurrently); headers are validated first."""
        N.require_device()
        paths = [str(p) for p in paths]
        arr = (C.c_char_p * max(1, len(paths)))(*[p.encode() for p in paths])
        devs = (C.c_int * len(devices))(*[int(d) for d in devices])
        cids = np.empty(sum(_fps1_count(p) for p in paths), dtype=np.uint64) if with_cids else None
        h = C.c_void_p()
        N.check(N.load().fps_group_open_fps1(arr, len(paths), devs, len(devices), cls._gather(gather),
                                             cids.ctypes.data if cids is not None else None, C.byref(h)),
                "fps_group_open_fps1")
        return cls(h.value, cids)

    @classmethod
    def generate(cls, n: int, seed_key: int, thresholds: np.ndarray, devices: Sequence[int], start: int = 0,
                 gather="auto") -> "LibraryGroup":
        """Synthetic library [start, start + n) generated shard by shard on its device."""
        from .libstore import split_sizes

        return cls._split(lambda a, b, dev: Library.generate(b - a, seed_key, thresholds, dev, start + a, start + a),
                          n, devices, gather, None, split_sizes)

    @classmethod
    def _split(cls, open_one, n: int, devices: Sequence[int], gather, cids, split_sizes) -> "LibraryGroup":
        N.require_device()
        if not devices:
            raise ValueError("at least one device")
        libs: list[Library] = []
        a = 0
        try:
            for dev, size in zip(devices, split_sizes(n, len(devices))):
                libs.append(open_one(a, a + size, int(dev)))
                a += size
            return cls.from_shards(libs, gather, cids)
        except BaseException:
            for lib in libs:
                lib.close()
            raise

    def close(self) -> None:
        if self._h and self._h.value:
            for s in self.shards:
                s._h = C.c_void_p()
            N.load().fps_group_close(self._h)
            self._h = C.c_void_p()

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---- reporting ------------------------------------------------------
    @property
    def last_kernel(self) -> str:
        return self.shards[0].last_kernel

    @property
    def last_mma_kind(self) -> str | None:
        return self.shards[0].last_mma_kind

    @property
    def launches(self) -> int:
        return int(N.load().fps_group_launch_count(self._h))

    def layout(self) -> tuple[bool, int]:
        return self.shards[0].layout()

    def memory(self) -> dict:
        out: dict = {}
        for s in self.shards:
            for key, v in s.memory().items():
                out[key] = out.get(key, 0) + v
        return out

    def read_entries(self, start: int = 0, count: int | None = None) -> np.ndarray:
        count = self.n - start if count is None else count
        parts = []
        for s in self.shards:
            lo, hi = max(start, s.index_base), min(start + count, s.index_base + s.n)
            if lo < hi:
                parts.append(s.read_entries(lo - s.index_base, hi - lo))
        return np.concatenate(parts) if parts else np.zeros((0, 3), np.uint64)

    def words_host(self) -> np.ndarray:
        return self.read_entries()

    def timing(self, enable: bool) -> None:
        for s in self.shards:
            s.timing(enable)

    def timing_read(self) -> tuple[float, int]:
        """(max over shards of the summed scan-kernel ms, launches of shard 0)."""
        reads = [s.timing_read() for s in self.shards]
        return max(r[0] for r in reads), reads[0][1]

    # ---- queries ----------------------------------------------------------
    def search_batch(self, queries, k: int) -> TopKResult:
        q = as_query_words(queries)
        if k < 1:
            raise ValueError("n must be >= 1")
        Q = len(q)
        idx = np.empty((Q, k), np.uint64)
        dist = np.empty((Q, k), np.uint16)
        cnt = np.zeros((Q,), np.uint32)
        if Q:
            N.check(N.load().fps_group_topk(self._h, q.ctypes.data, Q, k, idx.ctypes.data, dist.ctypes.data,
                                            cnt.ctypes.data), "fps_group_topk")
        return TopKResult(idx, dist, cnt)

    def search(self, query, k: int) -> list[tuple[int, int]]:
        return self.search_batch(query, k).hits(0)

    def search_min(self, queries, k: int) -> list[tuple[int, int]]:
        q = as_query_words(queries)
        if len(q) == 0:
            raise ValueError("batch_search requires at least one query")
        idx = np.empty((1, k), dtype=np.uint64)
        dist = np.empty((1, k), dtype=np.uint16)
        cnt = np.zeros(1, dtype=np.uint32)
        N.check(N.load().fps_group_topk_min(self._h, q.ctypes.data, len(q), k, idx.ctypes.data, dist.ctypes.data,
                                            cnt.ctypes.data), "fps_group_topk_min")
        return TopKResult(idx, dist, cnt).hits(0)

    def range_begin(self, queries, radius) -> int:
        """Per-shard scans + the root merge of the range hits, left on the root
        device (their count is returned); ``range_search`` also fetches them."""
        q = as_query_words(queries)
        rad = np.ascontiguousarray(np.minimum(np.broadcast_to(np.asarray(radius, dtype=np.int64), (len(q),)),
                                              254).astype(np.uint8))
        n_out = C.c_uint64()
        N.check(N.load().fps_group_range_begin(self._h, q.ctypes.data, len(q), rad.ctypes.data, C.byref(n_out)),
                "fps_group_range_begin")
        return n_out.value

    def range_search(self, queries, radius) -> RangeResult:
        q = as_query_words(queries)
        Q = len(q)
        r = np.broadcast_to(np.asarray(radius, dtype=np.int64), (Q,))
        if np.any(r < 0):
            raise ValueError("radius must be >= 0")
        if Q == 0:
            return RangeResult.from_keys(np.zeros(0, np.uint64))
        rad = np.ascontiguousarray(np.minimum(r, 254).astype(np.uint8))
        n_out = C.c_uint64()
        lib = N.load()
        N.check(lib.fps_group_range_begin(self._h, q.ctypes.data, Q, rad.ctypes.data, C.byref(n_out)),
                "fps_group_range_begin")
        m = n_out.value
        query, index, distance = np.empty(m, np.uint32), np.empty(m, np.uint64), np.empty(m, np.uint16)
        N.check(lib.fps_group_range_fetch(self._h, query.ctypes.data, index.ctypes.data, distance.ctypes.data, m),
                "fps_group_range_fetch")
        return RangeResult(query=query, index=index, distance=distance)

    # ---- stream-ordered device API (root device) ---------------------------
    def topk_prepare(self, Q: int, k: int) -> None:
        N.check(N.load().fps_group_topk_prepare(self._h, Q, k), "fps_group_topk_prepare")

    def topk_async(self, d_queries, Q: int, k: int, d_keys, d_cnt, stream: int) -> None:
        N.check(N.load().fps_group_topk_async(self._h, N.ptr(d_queries), Q, k, N.ptr(d_keys), N.ptr(d_cnt), stream),
                "fps_group_topk_async")


def merge_async(d_in_keys, d_in_cnt, G: int, Q: int, k: int, d_out_keys, d_out_cnt, stream: int) -> None:
    """Device merge of G per-shard sorted top-k lists (merge_topk semantics)."""
    N.check(N.load().fps_merge_async(N.ptr(d_in_keys), N.ptr(d_in_cnt), G, Q, k, N.ptr(d_out_keys),
                                     N.ptr(d_out_cnt), stream), "fps_merge_async")


def keys_to_hits(keys: np.ndarray, cnt: np.ndarray) -> TopKResult:
    """Decode device (distance << 40 | index) keys into a TopKResult."""
    keys = np.asarray(keys, dtype=np.uint64)
    cnt = np.asarray(cnt, dtype=np.uint32)
    Q, k = keys.shape
    valid = np.arange(k)[None, :] < cnt[:, None]
    idx = np.where(valid, keys & np.uint64(IDX_MASK), _U64_MAX)
    dist = np.where(valid, (keys >> np.uint64(40)) & np.uint64(0xFF), 0xFFFF).astype(np.uint16)
    return TopKResult(idx.astype(np.uint64), dist, cnt)


def _fps1_count(path) -> int:
    """Record count declared by an FPS1 header (validated again by the C loader)."""
    with open(path, "rb") as f:
        head = f.read(16)
    if len(head) < 16 or head[:4] != b"FPS1":
        return 0  # the loader reports the precise error
    return int.from_bytes(head[8:16], "little")


def load_library(source, device: int | None = None, index_base: int = 0, devices: Sequence[int] | None = None,
                 gather: str = "auto"):
    """Upload a library once: an (n, 3) word array, an (n, 4) FPS1 record
    array, a ShardManifest / library directory (FPS1 shards), or a Library.

    ``devices=[d0, d1, ...]`` (two or more) shards it contiguously over those
    GPUs and returns a LibraryGroup (same query methods); a device may repeat
    (several shards on one GPU)."""
    if isinstance(source, (Library, LibraryGroup)):
        return source
    if devices is not None and len(devices) > 1:
        if isinstance(source, np.ndarray):
            if source.ndim == 2 and source.shape[1] == 4:
                return LibraryGroup.from_records(source, devices, gather)
            return LibraryGroup.from_words(source, devices, gather=gather)
        from . import libstore

        manifest = source if hasattr(source, "shards") else libstore.load_manifest(Path(source))
        return LibraryGroup.from_fps1([s.path for s in manifest.shards], devices, gather)
    if devices is not None and len(devices) == 1:
        device = devices[0]
    if isinstance(source, np.ndarray):
        if source.ndim == 2 and source.shape[1] == 4:
            return Library.from_records(source, device, index_base)
        return Library.from_words(source, device, index_base)
    from . import libstore

    manifest = source if hasattr(source, "shards") else libstore.load_manifest(Path(source))
    return Library.from_fps1([s.path for s in manifest.shards], device=device)


def load_libraries(sources: Sequence, device: int | None = None) -> list[Library]:
    return [load_library(s, device) for s in sources]
