"""pytest plugin: run the reference's own fpscan tests against the CUDA scan.

Loaded with ``-p fpscan_cuda`` before the reference test modules are
collected, it applies the reference-side patch INTEGRATION.md §2 describes:
``fpscan.scan._search_multi`` (scan.py:239-287, behind ``search`` and
``batch_search``, and so behind the JobQueue / HTTP server) and
``fpscan.scan.scan_shard`` (scan.py:212-222) are routed to
``paper_1906_06170_b200.scan`` — the HBM-resident library and the sm_100a
kernels in libfpsgpu.so — for every ``kernel`` value the tests pass
("packed" and "reference" both run the CUDA scan). Results come back as the
reference's own ``TopK`` / ``SearchHit`` objects and errors as its own
exception classes, so the reference's assertions run unchanged.

Test infrastructure only: the reference package comes from ``baseline/_ref``
(tools/install_reference.sh); nothing in the product imports this file.
"""

from __future__ import annotations

import functools

import fpscan.scan as ref

from paper_1906_06170_b200 import errors as gerr
from paper_1906_06170_b200 import scan as gpu

CALLS = {"search_multi": 0, "scan_shard": 0}


def _to_ref(top) -> ref.TopK:
    return ref.TopK(capacity=top.capacity,
                    hits=tuple(ref.SearchHit(cid=h.cid, distance=h.distance) for h in top.hits))


def _params(params: ref.SearchParams) -> gpu.SearchParams:
    return gpu.SearchParams(n=params.n, parallelism=params.parallelism, kernel="cuda")


def _translated(fn):
    """Map the package's exception classes onto the reference's (same names,
    same messages: scan.py:38-48)."""

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        try:
            return fn(*args, **kwargs)
        except gerr.ScanCancelled as exc:
            raise ref.ScanCancelled(str(exc)) from exc
        except gerr.DuplicateCid as exc:
            raise ref.DuplicateCid(str(exc)) from exc
        except gerr.ScanError as exc:
            raise ref.ScanError(str(exc)) from exc

    return wrapper


@_translated
def _search_multi(manifest, queries, params, progress=None, cancel=None):
    CALLS["search_multi"] += 1
    queries = tuple(queries)
    if len(queries) == 1:
        top = gpu.search(manifest, queries[0], _params(params), progress, cancel)
    else:
        top = gpu.batch_search(manifest, queries, _params(params), progress, cancel)
    return _to_ref(top)


@_translated
def scan_shard(shard, query, params, progress=None, cancel=None):
    CALLS["scan_shard"] += 1
    return _to_ref(gpu.scan_shard(shard, query, _params(params), progress, cancel))


# the patch: module attributes replaced before any test module imports them
ref._search_multi = _search_multi
ref.scan_shard = scan_shard


def pytest_terminal_summary(terminalreporter):
    terminalreporter.section("fpscan -> CUDA adapter")
    terminalreporter.write_line(f"calls routed to libfpsgpu.so: {CALLS}")
