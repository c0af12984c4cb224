"""Test configuration: the `gpu` marker and import paths.

`-m "not gpu"` runs the oracle-vs-golden pins, host logic, C-ABI load/export
checks and the world_size-2 gloo tests on CPU; `-m gpu` runs the CUDA parity
tests (they call libfpsgpu.so through its C ABI).
"""

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
for p in (ROOT, ROOT / "oracle"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libfpsgpu.so")


@pytest.fixture(scope="session")
def golden():
    import json

    return json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())
