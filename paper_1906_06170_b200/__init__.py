"""paper_1906_06170_b200 — B200-native MACCS-166 fingerprint similarity scan.

The hot path of FPScreen (arXiv 1906.06170) / the reference ``fpscan``
package — per-query Hamming distance over every library entry plus top-k or
range selection — as hand-written sm_100a CUDA behind a C ABI
(include/fps.h, libfpsgpu.so), bound here with ctypes. There is no CPU
fallback: without libfpsgpu.so and a CUDA device the scan raises.

* ``load_library`` / ``Library``: the library resident in HBM (SoA planes);
  ``search``, ``search_batch``, ``range_search`` return (index, distance).
* ``scan``: drop-in ``search`` / ``batch_search`` / ``scan_shard`` /
  ``merge_topk`` with the reference's types (TopK of (cid, distance)).
* ``LibraryGroup`` (``load_library(..., devices=[...])``): one library over
  several GPUs of this process, merged on the root device (peer reads over
  NVLink, NCCL, or peer copies).
* ``distributed``: contiguous shards, one process per GPU (torchrun), merge
  on rank 0.
"""

from .errors import (
    DuplicateCid,
    FingerprintError,
    InvalidCharacter,
    NativeUnavailable,
    ScanCancelled,
    ScanError,
    WrongLength,
)
from .fingerprint import NUM_KEYS, Fingerprint, distance_packed, parse_bitstring, to_bitstring
from .library import Library, LibraryGroup, RangeResult, TopKResult, load_library

__all__ = [
    "NUM_KEYS",
    "Fingerprint",
    "FingerprintError",
    "InvalidCharacter",
    "WrongLength",
    "DuplicateCid",
    "ScanCancelled",
    "ScanError",
    "NativeUnavailable",
    "distance_packed",
    "parse_bitstring",
    "to_bitstring",
    "Library",
    "LibraryGroup",
    "RangeResult",
    "TopKResult",
    "load_library",
]

__version__ = "0.1.0"
