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
