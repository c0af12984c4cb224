"""Read side of the reference's FPS1 shard format and manifest (library input).

Mirrors /root/reference/pkg/src/fpscan/libstore.py: 16-byte header "FPS1" |
u16 version (1) | 2 zero bytes | u64 record_count (libstore.py:5-16, :28-35,
:202-212); 32-byte records u64 cid | 21 fingerprint bytes | 3 zero bytes
(libstore.py:158-164), which the scan views as (n, 4) little-endian u64
(scan.py:169); manifest.json with shard paths relative to it
(libstore.py:279-326); contiguous balanced splits (libstore.py:174-179).
Writing libraries (text ingestion, FNV-1a checksums) is out of scope here.
"""

from __future__ import annotations

import json
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import BadMagic, IoFailure, LibstoreError, TruncatedFile, VersionMismatch

MAGIC = b"FPS1"
FORMAT_VERSION = 1
HEADER_SIZE = 16
RECORD_SIZE = 32
_HEADER = struct.Struct("<4sHHQ")


@dataclass(frozen=True)
class Shard:
    path: Path
    record_count: int
    dataset_label: str
    checksum: int


@dataclass(frozen=True)
class ShardManifest:
    shards: tuple[Shard, ...]
    total_records: int
    format_version: int = FORMAT_VERSION

    def __post_init__(self):
        if self.total_records != sum(s.record_count for s in self.shards):
            raise LibstoreError(
                f"total_records {self.total_records} != sum of shard counts "
                f"{sum(s.record_count for s in self.shards)}"
            )


def split_sizes(total: int, shard_count: int) -> list[int]:
    """Contiguous split into shard_count parts whose sizes differ by at most 1."""
    if shard_count < 1:
        raise ValueError("shard_count must be >= 1")
    base, extra = divmod(total, shard_count)
    return [base + (1 if i < extra else 0) for i in range(shard_count)]


def shard_offsets(total: int, shard_count: int) -> list[int]:
    """Start index of every contiguous shard (plus the end)."""
    offs = [0]
    for s in split_sizes(total, shard_count):
        offs.append(offs[-1] + s)
    return offs


def manifest_path(library_dir) -> Path:
    return Path(library_dir) / "manifest.json"


def load_manifest(library_dir) -> ShardManifest:
    """Load manifest.json from a library directory, resolving shard paths."""
    library_dir = Path(library_dir)
    if library_dir.is_file():
        library_dir = library_dir.parent
    path = manifest_path(library_dir)
    try:
        doc = json.loads(path.read_text(encoding="utf-8"))
    except FileNotFoundError as exc:
        raise IoFailure(f"no manifest at {path}") from exc
    except (OSError, json.JSONDecodeError) as exc:
        raise IoFailure(f"reading {path}: {exc}") from exc
    shards = tuple(
        Shard(path=library_dir / s["path"], record_count=int(s["record_count"]),
              dataset_label=s["dataset_label"], checksum=int(s["checksum"], 16))
        for s in doc["shards"]
    )
    return ShardManifest(shards=shards, total_records=int(doc["total_records"]),
                         format_version=int(doc["format_version"]))


def read_shard_header(f, path) -> int:
    """Validate the 16-byte header and return the record count it declares."""
    raw = f.read(HEADER_SIZE)
    if len(raw) < HEADER_SIZE:
        raise TruncatedFile(path, f"header is {len(raw)} bytes, expected {HEADER_SIZE}")
    magic, version, _, count = _HEADER.unpack(raw)
    if magic != MAGIC:
        raise BadMagic(path, f"magic {magic!r}, expected {MAGIC!r}")
    if version != FORMAT_VERSION:
        raise VersionMismatch(path, f"format version {version}, expected {FORMAT_VERSION}")
    return count


def read_shard_records(shard) -> np.ndarray:
    """The whole record region of one shard as an (n, 4) '<u8' array."""
    path = Path(shard.path)
    with open(path, "rb") as f:
        count = read_shard_header(f, path)
        buf = f.read(count * RECORD_SIZE)
    if len(buf) < count * RECORD_SIZE:
        raise TruncatedFile(path, f"holds {len(buf) // RECORD_SIZE} records, header declares {count}")
    return np.frombuffer(buf, dtype="<u8").reshape(count, 4)


def read_manifest_records(manifest) -> np.ndarray:
    """All shards of a manifest, concatenated in manifest order."""
    parts = [read_shard_records(s) for s in manifest.shards]
    if not parts:
        return np.zeros((0, 4), dtype="<u8")
    return np.concatenate(parts) if len(parts) > 1 else parts[0]
