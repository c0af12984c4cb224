"""The C ABI library builds, loads, and exports every symbol include/fps.h declares.

CPU only: no compute call is made; without a GPU the scan must fail loudly
(NativeUnavailable), never fall back to a CPU path.
"""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "fps.h").read_text()
    return sorted(set(re.findall(r"\b(fps_[a-z_0-9]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_1906_06170_b200 import build

    build.build()
    from paper_1906_06170_b200 import _native

    return _native.load()


def test_exports_every_declared_symbol(lib):
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s


def test_python_binding_covers_header():
    from paper_1906_06170_b200 import _native

    assert sorted(_native.SIGNATURES) == declared_symbols()


def test_version_and_last_error(lib):
    assert lib.fps_version() == 1
    assert isinstance(lib.fps_last_error(), bytes)


def test_built_for_sm100a():
    import subprocess

    so = ROOT / "paper_1906_06170_b200" / "libfpsgpu.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device(lib):
    import torch

    from paper_1906_06170_b200 import NativeUnavailable, _native
    from paper_1906_06170_b200.library import Library

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible; covered by the gpu tests")
    assert _native.device_count() == 0
    with pytest.raises(NativeUnavailable):
        Library.from_words(np.zeros((4, 3), dtype=np.uint64))
    h = ctypes.c_void_p()
    w = np.zeros((4, 3), dtype=np.uint64)
    rc = lib.fps_open(w.ctypes.data, 4, 0, 0, 0, 1, ctypes.byref(h))
    assert rc == _native.FPS_ENODEV


def test_null_handle_rejected(lib):
    from paper_1906_06170_b200 import _native

    cnt = np.zeros(1, dtype=np.uint32)
    q = np.zeros((1, 3), dtype=np.uint64)
    assert lib.fps_topk(None, q.ctypes.data, 1, 5, None, None, cnt.ctypes.data) == _native.FPS_EINVAL
    assert b"null" in lib.fps_last_error()


def test_fps1_loader_reports_bad_shards_without_a_gpu(lib, tmp_path):
    """Shard headers are validated before any device work: bad magic, wrong
    version and truncation come back as FPS_EIO naming the path (the
    reference's ScanError("shard <path>: ...") contract, scan.py:283-284)."""
    import ctypes

    from paper_1906_06170_b200 import _native

    good = tmp_path / "good.fps"
    good.write_bytes(b"FPS1" + (1).to_bytes(2, "little") + b"\0\0" + (2).to_bytes(8, "little") + b"\0" * 64)
    cases = {
        "magic.fps": b"NOPE" + b"\0" * 12,
        "version.fps": b"FPS1" + (2).to_bytes(2, "little") + b"\0\0" + (0).to_bytes(8, "little"),
        "trunc.fps": b"FPS1" + (1).to_bytes(2, "little") + b"\0\0" + (5).to_bytes(8, "little") + b"\0" * 40,
        "short.fps": b"FPS1",
    }
    for name, data in cases.items():
        p = tmp_path / name
        p.write_bytes(data)
        arr = (ctypes.c_char_p * 2)(str(good).encode(), str(p).encode())
        h = ctypes.c_void_p()
        rc = lib.fps_open_fps1(arr, 2, 0, 2**64 - 1, 0, None, ctypes.byref(h))
        assert rc == _native.FPS_EIO, name
        msg = lib.fps_last_error().decode()
        assert msg.startswith("shard ") and name in msg, msg
    arr = (ctypes.c_char_p * 1)(str(tmp_path / "missing.fps").encode())
    assert lib.fps_open_fps1(arr, 1, 0, 2**64 - 1, 0, None, ctypes.byref(ctypes.c_void_p())) == _native.FPS_EIO


def test_range_unpack_matches_key_layout(lib):
    """fps_range_unpack (host code, no GPU) splits (q << 48 | d << 40 | idx)
    keys exactly like RangeResult.from_keys."""
    from paper_1906_06170_b200.library import RangeResult

    rng = np.random.default_rng(3)
    n = 10_001
    q = rng.integers(0, 65535, n, dtype=np.uint64)
    d = rng.integers(0, 167, n, dtype=np.uint64)
    idx = rng.integers(0, 1 << 40, n, dtype=np.uint64)
    keys = (q << np.uint64(48)) | (d << np.uint64(40)) | idx
    oq, oi, od = np.empty(n, np.uint32), np.empty(n, np.uint64), np.empty(n, np.uint16)
    lib.fps_range_unpack(keys.ctypes.data, n, oq.ctypes.data, oi.ctypes.data, od.ctypes.data)
    ref = RangeResult.from_keys(keys)
    assert np.array_equal(oq, ref.query) and np.array_equal(oi, ref.index) and np.array_equal(od, ref.distance)
    assert np.array_equal(oq, q.astype(np.uint32)) and np.array_equal(od, d.astype(np.uint16))
