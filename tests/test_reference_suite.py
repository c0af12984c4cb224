"""The reference's own search tests, run through the CUDA adapter.

``tests/reference_suite/fpscan_cuda.py`` patches the installed reference
(``baseline/_ref``, tools/install_reference.sh) so that ``search``,
``batch_search``, ``scan_shard`` — and through them the JobQueue and the HTTP
server — run on libfpsgpu.so; the reference's test files then run unchanged:

* ``test_scan.py`` — all of it (scan_shard / search / batch_search against
  the brute-force oracles, ties by CID, progress, cancel, shard errors,
  merge_topk, the accumulator);
* ``test_acceptance.py`` criteria 1-4, 7 and 10 (kernel equivalence, oracle
  top-N under every parallelism and kernel, determinism, self-retrieval with
  CID tie order, batch search, HTTP API conformance end to end).

Not run: criterion 5 (CPU-throughput claim of the numpy kernel), 6 and 8
(library round trips, molfile keys: off the scan path), 9 (its cancel-mid-scan
step assumes a scan longer than 0.15 s; a GPU scan of its library finishes
first — INTEGRATION.md §3).
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"
REF_TESTS = REF / "fpscan_tests"
ACCEPTANCE = ["criterion_01", "criterion_02", "criterion_03", "criterion_04", "criterion_07", "criterion_10"]


def _run(tmp_path, files, kexpr=None):
    ini = tmp_path / "pytest.ini"
    ini.write_text("[pytest]\nfilterwarnings =\n    ignore:Using `httpx` with `starlette.testclient` is deprecated\n")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF), str(ROOT / "tests" / "reference_suite"), str(ROOT),
                                         str(REF_TESTS), env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-q", "-c", str(ini), "--rootdir", str(REF_TESTS), "-p", "fpscan_cuda",
           "-p", "no:cacheprovider", *[str(REF_TESTS / f) for f in files]]
    if kexpr:
        cmd += ["-k", kexpr]
    return subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=1800)


def _needs_reference():
    if not (REF / "fpscan" / "scan.py").exists() or not (REF_TESTS / "test_scan.py").exists():
        pytest.skip("baseline/_ref is missing: __graft_entry__.build() / tools/install_reference.sh installs it in the build container")


@pytest.mark.gpu
def test_reference_test_scan(tmp_path):
    _needs_reference()
    r = _run(tmp_path, ["test_scan.py"])
    tail = (r.stdout + r.stderr)[-6000:]
    assert r.returncode == 0, tail
    assert "failed" not in r.stdout.splitlines()[-1], tail
    assert "calls routed to libfpsgpu.so" in r.stdout, tail


@pytest.mark.gpu
def test_reference_acceptance(tmp_path):
    _needs_reference()
    r = _run(tmp_path, ["test_acceptance.py"], " or ".join(ACCEPTANCE))
    tail = (r.stdout + r.stderr)[-6000:]
    assert r.returncode == 0, tail
    for c in ACCEPTANCE:
        assert any(line.startswith("PASS") and c in line for line in r.stdout.splitlines()), (c, tail)
