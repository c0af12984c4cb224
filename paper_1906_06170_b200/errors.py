"""Exception types, named and layered like the reference's.

``FingerprintError`` / ``WrongLength`` / ``InvalidCharacter`` mirror
fingerprint.py:30-44; ``ScanError`` / ``DuplicateCid`` / ``ScanCancelled``
mirror scan.py:38-48; the shard-file errors mirror libstore.py:42-90.
"""

from __future__ import annotations

from pathlib import Path


class FingerprintError(ValueError):
    """Base class for fingerprint parsing and validation failures."""


class WrongLength(FingerprintError):
    def __init__(self, length: int):
        super().__init__(f"bitstring must be 166 or 167 characters, got {length}")
        self.length = length


class InvalidCharacter(FingerprintError):
    def __init__(self, char: str, position: int):
        super().__init__(f"invalid character {char!r} at position {position}; only '0'/'1' allowed")
        self.char = char
        self.position = position


class ScanError(Exception):
    """A scan failed; message names the shard or device."""


class DuplicateCid(ScanError):
    """Two merged parts contained the same CID, which means sharding is broken."""


class ScanCancelled(Exception):
    """Raised when the cancellation signal is observed."""


class NativeUnavailable(RuntimeError):
    """libfpsgpu.so or a CUDA device is missing; there is no CPU fallback."""


class LibstoreError(Exception):
    """Base class for library storage failures."""


class LineFormatError(LibstoreError):
    """A text library line is malformed; carries the 1-based line number when known."""

    def __init__(self, message: str, line_number: int | None = None):
        self.line_number = line_number
        prefix = f"line {line_number}: " if line_number is not None else ""
        super().__init__(prefix + message)


class MissingTab(LineFormatError):
    def __init__(self, line_number: int | None = None):
        super().__init__("expected `<CID>\\t<bitstring>`, no tab found", line_number)


class BadCid(LineFormatError):
    def __init__(self, raw: str, line_number: int | None = None):
        super().__init__(f"bad CID {raw!r}: must be a decimal integer in 1..2^64-1", line_number)


class ShardFileError(LibstoreError):
    """A shard file failed structural validation; carries the offending path."""

    def __init__(self, path, message: str):
        self.path = Path(path)
        super().__init__(f"{path}: {message}")


class BadMagic(ShardFileError):
    pass


class VersionMismatch(ShardFileError):
    pass


class ChecksumMismatch(ShardFileError):
    pass


class TruncatedFile(ShardFileError):
    pass


class IoFailure(LibstoreError):
    pass
