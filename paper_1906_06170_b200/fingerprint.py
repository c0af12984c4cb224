"""Query-side fingerprint value type (host plumbing for the scan's inputs).

Mirrors the reference L0 surface (/root/reference/pkg/src/fpscan/fingerprint.py):
166 keys packed into three little-endian u64 words, key j (1-based) at word
(j-1)//64, bit (j-1)%64 (fingerprint.py:3-5); the 26 bits above key 166 must
be zero (fingerprint.py:60-61); 166- and 167-character bitstrings
(fingerprint.py:112-133). The scan itself never runs here — distances over a
library are computed only by the CUDA path (libfpsgpu.so).
"""

from __future__ import annotations

import operator
from dataclasses import dataclass
from typing import Iterable

import numpy as np

from .errors import FingerprintError, InvalidCharacter, WrongLength

NUM_KEYS = 166
WORD_COUNT = 3
PACKED_BYTES = 21

_WORD_MASK = (1 << 64) - 1
_LAST_WORD_MASK = (1 << (NUM_KEYS - 128)) - 1


@dataclass(frozen=True)
class Fingerprint:
    """Immutable 166-key fingerprint packed into three little-endian 64-bit words."""

    words: tuple[int, int, int]

    def __post_init__(self):
        if len(self.words) != WORD_COUNT:
            raise FingerprintError(f"expected {WORD_COUNT} words, got {len(self.words)}")
        for i, w in enumerate(self.words):
            if not 0 <= w <= _WORD_MASK:
                raise FingerprintError(f"word {i} out of 64-bit range: {w:#x}")
        if self.words[2] & ~_LAST_WORD_MASK:
            raise FingerprintError("padding bits above key 166 must be zero")

    @classmethod
    def zero(cls) -> "Fingerprint":
        return cls((0, 0, 0))

    @classmethod
    def from_keys(cls, keys: Iterable[int]) -> "Fingerprint":
        words = [0, 0, 0]
        for j in keys:
            j = operator.index(j)
            if not 1 <= j <= NUM_KEYS:
                raise FingerprintError(f"key index {j} outside 1..{NUM_KEYS}")
            words[(j - 1) // 64] |= 1 << ((j - 1) % 64)
        return cls(tuple(words))

    @classmethod
    def from_packed(cls, data: bytes) -> "Fingerprint":
        if len(data) != PACKED_BYTES:
            raise FingerprintError(f"packed fingerprint must be {PACKED_BYTES} bytes, got {len(data)}")
        return cls((int.from_bytes(data[0:8], "little"), int.from_bytes(data[8:16], "little"),
                    int.from_bytes(data[16:21], "little")))

    def to_packed(self) -> bytes:
        w0, w1, w2 = self.words
        return w0.to_bytes(8, "little") + w1.to_bytes(8, "little") + w2.to_bytes(5, "little")

    def key(self, j: int) -> bool:
        if not 1 <= j <= NUM_KEYS:
            raise FingerprintError(f"key index {j} outside 1..{NUM_KEYS}")
        return bool(self.words[(j - 1) // 64] >> ((j - 1) % 64) & 1)

    def keys(self) -> frozenset[int]:
        return frozenset(j for j in range(1, NUM_KEYS + 1) if self.key(j))

    def popcount(self) -> int:
        return sum(w.bit_count() for w in self.words)


def parse_bitstring(text: str) -> Fingerprint:
    """166 chars: char i -> key i+1; 167 chars: the leading char is dropped."""
    if len(text) not in (NUM_KEYS, NUM_KEYS + 1):
        raise WrongLength(len(text))
    for i, c in enumerate(text):
        if c not in "01":
            raise InvalidCharacter(c, i)
    if len(text) == NUM_KEYS + 1:
        text = text[1:]
    value = int(text[::-1], 2)
    return Fingerprint((value & _WORD_MASK, (value >> 64) & _WORD_MASK, value >> 128))


def to_bitstring(fp: Fingerprint) -> str:
    w0, w1, w2 = fp.words
    return format(w0 | (w1 << 64) | (w2 << 128), f"0{NUM_KEYS}b")[::-1]


def distance_packed(a: Fingerprint, b: Fingerprint) -> int:
    """Scalar distance contract between two fingerprints (popcount of XOR)."""
    return sum((x ^ y).bit_count() for x, y in zip(a.words, b.words))


def as_query_words(queries) -> np.ndarray:
    """Normalise queries to a C-contiguous (Q, 3) uint64 array.

    Accepts Fingerprint objects (ours or the reference's — anything with
    ``.words``), 3-tuples of ints, or a (Q, 3) / (3,) integer array. Padding
    bits are validated like the Fingerprint constructor.
    """
    if isinstance(queries, np.ndarray):
        arr = np.ascontiguousarray(np.atleast_2d(queries).astype(np.uint64, copy=False))
    else:
        if hasattr(queries, "words") or (isinstance(queries, tuple) and len(queries) == 3
                                         and all(isinstance(x, (int, np.integer)) for x in queries)):
            queries = [queries]
        rows = [tuple(getattr(q, "words", q)) for q in queries]
        arr = np.array(rows, dtype=np.uint64).reshape(-1, 3) if rows else np.zeros((0, 3), np.uint64)
    if arr.ndim != 2 or arr.shape[1] != 3:
        raise FingerprintError(f"queries must be (Q, 3) words, got shape {arr.shape}")
    if np.any(arr[:, 2] >> np.uint64(38)):
        raise FingerprintError("padding bits above key 166 must be zero")
    return arr
