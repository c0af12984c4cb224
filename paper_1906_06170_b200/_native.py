"""ctypes binding of libfpsgpu.so (include/fps.h) and status -> exception mapping.

The shared library is built in-tree (``build.py``) and loaded from this
package directory. There is no CPU fallback: if the library or a CUDA device
is missing, every scan entry point raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import FingerprintError, NativeUnavailable, ScanCancelled, ScanError

LIB_NAME = "libfpsgpu.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

FPS_OK = 0
FPS_EINVAL = 1
FPS_ENOMEM = 2
FPS_ECUDA = 3
FPS_EPADDING = 4
FPS_ECANCELLED = 5
FPS_ENODEV = 6
FPS_EIO = 7

LAYOUT_ROWS3 = 0
LAYOUT_FPS1 = 1
LAYOUT_PLANES = 2

_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_u16p = C.POINTER(C.c_uint16)
_u8p = C.POINTER(C.c_uint8)
_vp = C.c_void_p

# name -> (restype, argtypes); every symbol declared in include/fps.h
SIGNATURES = {
    "fps_version": (C.c_int, []),
    "fps_last_error": (C.c_char_p, []),
    "fps_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "fps_open": (C.c_int, [_vp, C.c_uint64, C.c_int, C.c_int, C.c_uint64, C.c_int, C.POINTER(_vp)]),
    "fps_open_device": (C.c_int, [_vp, _vp, _vp, C.c_uint64, C.c_int, C.c_uint64, C.POINTER(_vp)]),
    "fps_open_fps1": (C.c_int, [C.POINTER(C.c_char_p), C.c_uint32, C.c_uint64, C.c_uint64, C.c_int, _vp,
                                C.POINTER(_vp)]),
    "fps_open_generated": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, _vp, _vp, C.c_int, C.c_uint64,
                                     C.POINTER(_vp)]),
    "fps_close": (C.c_int, [_vp]),
    "fps_info": (C.c_int, [_vp, _u64p, _u64p, C.POINTER(C.c_int)]),
    "fps_layout": (C.c_int, [_vp, C.POINTER(C.c_int), _u64p]),
    "fps_read_entries": (C.c_int, [_vp, C.c_uint64, C.c_uint64, _vp]),
    "fps_write_entries": (C.c_int, [_vp, _vp, _vp, C.c_uint64]),
    "fps_topk": (C.c_int, [_vp, _vp, C.c_uint32, C.c_uint32, _vp, _vp, _vp]),
    "fps_topk_min": (C.c_int, [_vp, _vp, C.c_uint32, C.c_uint32, _vp, _vp, _vp]),
    "fps_range": (C.c_int, [_vp, _vp, C.c_uint32, _vp, C.POINTER(_vp), _u64p]),
    "fps_free": (None, [_vp]),
    "fps_range_unpack": (None, [_vp, C.c_uint64, _vp, _vp, _vp]),
    "fps_range_begin": (C.c_int, [_vp, _vp, C.c_uint32, _vp, _u64p]),
    "fps_range_fetch": (C.c_int, [_vp, _vp, _vp, _vp, C.c_uint64]),
    "fps_fnv1a64": (C.c_uint64, [_vp, C.c_uint64, C.c_uint64]),
    "fps_fnv1a64_file": (C.c_int, [C.c_char_p, C.c_uint64, _u64p]),
    "fps_build_shards": (C.c_int, [_vp, C.c_uint64, _vp, C.c_uint64, C.c_char_p, C.c_uint32, C.c_char_p, C.c_int,
                                   _vp, _vp, _u64p, _u64p, _u64p, _u64p]),
    "fps_topk_prepare": (C.c_int, [_vp, C.c_uint32, C.c_uint32]),
    "fps_topk_async": (C.c_int, [_vp, _vp, C.c_uint32, C.c_uint32, _vp, _vp, _vp]),
    "fps_range_async": (C.c_int, [_vp, _vp, C.c_uint32, _vp, _vp, C.c_uint64, _vp, _vp]),
    "fps_sort_keys": (C.c_int, [_vp, _vp, C.c_uint64, _vp]),
    "fps_merge_async": (C.c_int, [_vp, _vp, C.c_uint32, C.c_uint32, C.c_uint32, _vp, _vp, _vp]),
    "fps_merge_runs_async": (C.c_int, [_vp, _vp, C.c_uint32, _vp, _vp]),
    "fps_merge_packed_async": (C.c_int, [_vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, _vp, _vp, _vp]),
    "fps_launch_count": (C.c_uint64, [_vp]),
    "fps_last_kernel": (C.c_int, [_vp]),
    "fps_last_mma_kind": (C.c_int, [_vp]),
    "fps_mma_overflowed": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "fps_query_hint": (C.c_int, [_vp, _vp]),
    "fps_timing": (C.c_int, [_vp, C.c_int]),
    "fps_timing_read": (C.c_int, [_vp, C.POINTER(C.c_double), _u64p]),
    "fps_memory": (C.c_int, [_vp, _u64p, _u64p, _u64p, C.POINTER(C.c_double)]),
    "fps_release_derived": (C.c_int, [_vp]),
    "fps_group_open": (C.c_int, [C.POINTER(_vp), C.c_uint32, C.c_int, C.POINTER(_vp)]),
    "fps_group_open_fps1": (C.c_int, [C.POINTER(C.c_char_p), C.c_uint32, C.POINTER(C.c_int), C.c_uint32, C.c_int,
                                      _vp, C.POINTER(_vp)]),
    "fps_group_close": (C.c_int, [_vp]),
    "fps_group_info": (C.c_int, [_vp, _u64p, _u32p, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "fps_group_shard": (C.c_int, [_vp, C.c_uint32, C.POINTER(_vp)]),
    "fps_group_launch_count": (C.c_uint64, [_vp]),
    "fps_group_topk": (C.c_int, [_vp, _vp, C.c_uint32, C.c_uint32, _vp, _vp, _vp]),
    "fps_group_topk_min": (C.c_int, [_vp, _vp, C.c_uint32, C.c_uint32, _vp, _vp, _vp]),
    "fps_group_range_begin": (C.c_int, [_vp, _vp, C.c_uint32, _vp, _u64p]),
    "fps_group_range_fetch": (C.c_int, [_vp, _vp, _vp, _vp, C.c_uint64]),
    "fps_group_topk_prepare": (C.c_int, [_vp, C.c_uint32, C.c_uint32]),
    "fps_group_topk_async": (C.c_int, [_vp, _vp, C.c_uint32, C.c_uint32, _vp, _vp, _vp]),
}

GATHER_AUTO = 0
GATHER_P2P = 1
GATHER_NCCL = 2
GATHER_COPY = 3
GATHER_NAMES = {"auto": GATHER_AUTO, "p2p": GATHER_P2P, "nccl": GATHER_NCCL, "copy": GATHER_COPY}

_lib = None
_lock = threading.Lock()


def load(path: str | os.PathLike | None = None) -> C.CDLL:
    """Load libfpsgpu.so (once) and declare every exported signature."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise NativeUnavailable(
                f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = C.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.fps_version() != 1:
            raise NativeUnavailable(f"{p}: unexpected ABI version {lib.fps_version()}")
        if path is None:
            _lib = lib
        return lib


def last_error() -> str:
    msg = load().fps_last_error()
    return msg.decode(errors="replace") if msg else ""


def check(rc: int, what: str) -> None:
    """Map an fps_status to the reference's exception types."""
    if rc == FPS_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == FPS_EINVAL:
        raise ValueError(msg)
    if rc == FPS_EPADDING:
        raise FingerprintError(msg)
    if rc == FPS_ENOMEM:
        raise MemoryError(msg)
    if rc == FPS_ECANCELLED:
        raise ScanCancelled(msg)
    if rc == FPS_ENODEV:
        raise NativeUnavailable(msg)
    if rc == FPS_EIO:
        raise ScanError(last_error())  # "shard <path>: ..." like scan.py:283-284
    raise ScanError(msg)


def device_count() -> int:
    n = C.c_int(0)
    load().fps_device_count(C.byref(n))
    return n.value


def require_device() -> None:
    if device_count() < 1:
        raise NativeUnavailable("no CUDA device visible: the fingerprint scan has no CPU fallback")


def ptr(a) -> int:
    """Address of a numpy array's data or a torch tensor's storage."""
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data
