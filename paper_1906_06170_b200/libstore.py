"""Read side of the reference's FPS1 shard format and manifest (library input).

Mirrors /root/reference/pkg/src/fpscan/libstore.py: 16-byte header "FPS1" |
u16 version (1) | 2 zero bytes | u64 record_count (libstore.py:5-16, :28-35,
:202-212); 32-byte records u64 cid | 21 fingerprint bytes | 3 zero bytes
(libstore.py:158-164), which the scan views as (n, 4) little-endian u64
(scan.py:169); manifest.json with shard paths relative to it
(libstore.py:279-326); contiguous balanced splits (libstore.py:174-179).

The write side -- text-line ingestion, FNV-1a checksums, shard files,
manifest, validation (libstore.py:93-98, :136-155, :243-290, :339-398) -- runs
in the native builder (csrc/fps_ingest.cpp, multi-threaded, no GPU needed):
``build_shards`` / ``build_shards_from_file`` / ``fnv1a_64`` /
``validate_manifest``. Only a rejected line is re-parsed here, to raise the
reference's exact exception.
"""

from __future__ import annotations

import json
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import (BadCid, BadMagic, ChecksumMismatch, FingerprintError, InvalidCharacter, IoFailure,
                     LibstoreError, LineFormatError, MissingTab, ShardFileError, TruncatedFile, VersionMismatch,
                     WrongLength)

MAGIC = b"FPS1"
FORMAT_VERSION = 1
HEADER_SIZE = 16
RECORD_SIZE = 32
_HEADER = struct.Struct("<4sHHQ")
CID_MAX = (1 << 64) - 1
NUM_KEYS = 166
FNV64_OFFSET = 0xCBF29CE484222325


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


# --------------------------------------------------------------------------
# write side (native builder)
# --------------------------------------------------------------------------
def _lib():
    from . import _native

    return _native.load()


def fnv1a_64(data: bytes, value: int = FNV64_OFFSET) -> int:
    """64-bit FNV-1a over `data`, resumable (libstore.py:93-98); native loop."""
    buf = bytes(data)
    return int(_lib().fps_fnv1a64(buf, len(buf), value))


def shard_label(index: int) -> str:
    """Labels A, B, ... Z, then A1, B1, ... Z1, A2, ... (libstore.py:166-171)."""
    letter = chr(ord("A") + index % 26)
    cycle = index // 26
    return letter if cycle == 0 else f"{letter}{cycle}"


def _parse_bits(text: str) -> None:
    """Validation half of parse_bitstring (fingerprint.py:112-134): raises the
    reference's WrongLength / InvalidCharacter."""
    if len(text) in (NUM_KEYS, NUM_KEYS + 1):
        for i, c in enumerate(text):
            if c not in "01":
                raise InvalidCharacter(c, i)
    else:
        raise WrongLength(len(text))


def parse_library_line(line: str, line_number: int | None = None) -> int:
    """Check one `<CID><TAB><bitstring>` line like libstore.py:136-155 and
    return its CID; raises MissingTab / BadCid / LineFormatError. (The
    native builder parses the records; this restatement only turns a rejected
    line into the reference's exact exception.)"""
    line = line.rstrip("\r\n")
    cid_text, sep, bits = line.partition("\t")
    if not sep:
        raise MissingTab(line_number)
    if not (cid_text.isascii() and cid_text.isdigit()):
        raise BadCid(cid_text, line_number)
    cid = int(cid_text)
    if cid == 0 or cid > CID_MAX:
        raise BadCid(cid_text, line_number)
    try:
        _parse_bits(bits)
    except FingerprintError as exc:
        raise LineFormatError(str(exc), line_number) from exc
    return cid


def _raise_line_error(raw: bytes, line_number: int):
    text = raw.decode("utf-8")  # UnicodeDecodeError for undecodable bytes, as text-mode reading raises
    parse_library_line(text, line_number)
    raise LineFormatError("malformed library line", line_number)  # not reached for native-rejected lines


def save_manifest(manifest: ShardManifest, library_dir) -> Path:
    """Write manifest.json, shard paths relative to the library dir (libstore.py:279-300)."""
    library_dir = Path(library_dir)
    doc = {
        "format_version": manifest.format_version,
        "total_records": manifest.total_records,
        "shards": [
            {
                "path": Path(s.path).name,
                "dataset_label": s.dataset_label,
                "record_count": s.record_count,
                "checksum": f"{s.checksum:016x}",
            }
            for s in manifest.shards
        ],
    }
    path = manifest_path(library_dir)
    try:
        path.write_text(json.dumps(doc, indent=2) + "\n", encoding="utf-8")
    except OSError as exc:
        raise IoFailure(f"writing {path}: {exc}") from exc
    return path


def _build(text: bytes | None, offsets, n_lines: int, text_path, shard_count: int, out_dir,
           threads: int) -> ShardManifest:
    import ctypes as C

    from . import _native

    if shard_count < 1:
        raise ValueError("shard_count must be >= 1")
    out_dir = Path(out_dir)  # created by the builder once every line parsed
    counts = np.zeros(shard_count, np.uint64)
    sums = np.zeros(shard_count, np.uint64)
    total, el, eo, en = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
    rc = _lib().fps_build_shards(text, len(text) if text is not None else 0,
                                 offsets.ctypes.data if offsets is not None else None, n_lines,
                                 str(text_path).encode() if text_path is not None else None, shard_count,
                                 str(out_dir).encode(), threads, counts.ctypes.data, sums.ctypes.data,
                                 C.byref(total), C.byref(el), C.byref(eo), C.byref(en))
    if rc == _native.FPS_EINVAL and el.value:
        if text_path is not None:
            with open(text_path, "rb") as f:
                f.seek(eo.value)
                raw = f.read(en.value)
        else:
            raw = text[eo.value:eo.value + en.value]
        _raise_line_error(raw, int(el.value))
    if rc == _native.FPS_EIO:
        raise IoFailure(_native.last_error())
    _native.check(rc, "fps_build_shards")
    shards = tuple(
        Shard(path=out_dir / f"shard-{i:03d}.fps", record_count=int(counts[i]), dataset_label=shard_label(i),
              checksum=int(sums[i]))
        for i in range(shard_count)
    )
    manifest = ShardManifest(shards=shards, total_records=int(total.value))
    save_manifest(manifest, out_dir)
    return manifest


def build_shards(lines, shard_count: int, out_dir, threads: int = 0) -> ShardManifest:
    """libstore.build_shards (libstore.py:243-272): pack text library lines
    into `shard_count` balanced FPS1 shards + manifest.json. Same records,
    bytes, checksums, labels and errors as the reference; parsing, packing,
    FNV-1a and the file writes run natively in parallel. A text file object
    opened like the reference CLI does (utf-8, default newlines) is read
    whole by the native builder."""
    import io

    if isinstance(lines, io.TextIOWrapper) and lines.encoding.lower().replace("-", "") == "utf8" \
            and getattr(lines, "name", None) and lines.seekable() and lines.tell() == 0:
        return build_shards_from_file(lines.name, shard_count, out_dir, threads)
    items = [ln.encode("utf-8") for ln in lines]
    offsets = np.zeros(len(items) + 1, np.uint64)
    if items:
        np.cumsum([len(b) for b in items], out=offsets[1:])
    return _build(b"".join(items), offsets, len(items), None, shard_count, out_dir, threads)


def build_shards_from_file(path, shard_count: int, out_dir, threads: int = 0) -> ShardManifest:
    """Build shards from a text library file (the reference CLI's
    `build` path, cli.py:69-70), read with Python text-mode line splitting."""
    return _build(None, None, 0, Path(path), shard_count, out_dir, threads)


@dataclass(frozen=True)
class Violation:
    kind: str
    path: str
    message: str

    def __str__(self) -> str:
        return f"[{self.kind}] {self.path}: {self.message}"


def validate_manifest(manifest: ShardManifest) -> list[Violation]:
    """Check every shard against the manifest (libstore.py:339-398);
    violations are data, not exceptions. Checksums by the native FNV-1a."""
    import ctypes as C

    violations: list[Violation] = []
    declared_total = sum(s.record_count for s in manifest.shards)
    if manifest.total_records != declared_total:
        violations.append(Violation("sum-mismatch", "manifest",
                                    f"total_records {manifest.total_records} != shard sum {declared_total}"))
    seen: set[str] = set()
    for shard in manifest.shards:
        spath = str(shard.path)
        if spath in seen:
            violations.append(Violation("duplicate-path", spath, "shard path repeated"))
        seen.add(spath)
        p = Path(shard.path)
        if not p.exists():
            violations.append(Violation("missing-file", spath, "shard file does not exist"))
            continue
        try:
            with open(p, "rb") as f:
                header_count = read_shard_header(f, p)
        except ShardFileError as exc:
            violations.append(Violation("bad-header", spath, str(exc)))
            continue
        if header_count != shard.record_count:
            violations.append(Violation("count-mismatch", spath,
                                        f"header declares {header_count} records, manifest says "
                                        f"{shard.record_count}"))
            continue
        size = p.stat().st_size
        expected = HEADER_SIZE + shard.record_count * RECORD_SIZE
        if size != expected:
            violations.append(Violation("size-mismatch", spath, f"file is {size} bytes, expected {expected}"))
            continue
        out = C.c_uint64()
        rc = _lib().fps_fnv1a64_file(str(p).encode(), HEADER_SIZE, C.byref(out))
        if rc != 0:
            from . import _native

            raise IoFailure(_native.last_error())
        if out.value != shard.checksum:
            violations.append(Violation("checksum-mismatch", spath,
                                        f"record region hashes to {out.value:016x}, manifest says "
                                        f"{shard.checksum:016x}"))
    return violations
