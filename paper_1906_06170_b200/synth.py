"""Seeded synthetic workloads for the five BASELINE.json configurations.

The real PubChem MACCS library (95,417,114 entries) is not
available; these stand in with its sizes:

* per seed, p_j ~ Beta(0.6, 2.0) for keys j = 1..166 (numpy PCG64), with
  p_1 = 0 ("bit 0 always 0" read as key 1, word 0 bit 0 — the reference's
  key j <-> bit j-1 mapping, fingerprint.py:3-5);
* entry i, key j is set iff u32(i, j) < floor(p_j * 2^32), u32 taken from a
  counter-based splitmix64 stream, so any chunk is reproducible on the GPU
  (gen_kernel) and in numpy (oracle twin) — the chunk-determinism pattern of
  the reference's synth.py:28-39 with its CID = index + 1 convention;
* queries are library entries with distinct key flips drawn from keys
  2..166; planted near-duplicates (C2, C5) are the query with 0..m flips at
  distinct random indices that exclude the query sources.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

NUM_KEYS = 166
_M64 = (1 << 64) - 1

CONFIGS = {
    # name: (entries, queries, k, radius, query flips (lo, hi), planted (count per query, lo, hi))
    "c1": dict(n=1_000_000, Q=1, k=10, radius=None, flips=(3, 3), planted=None),
    "c2": dict(n=10_000_000, Q=1, k=100, radius=None, flips=(3, 3), planted=(1000, 0, 4)),
    "c3": dict(n=95_417_114, Q=1, k=10, radius=None, flips=(3, 3), planted=None),
    "c4": dict(n=95_417_114, Q=1024, k=10, radius=None, flips=(0, 8), planted=None),
    "c5": dict(n=95_417_114, Q=64, k=None, radius=6, flips=(0, 6), planted=(10000, 0, 6)),
}


def splitmix64(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def seed_key(seed: int) -> int:
    return splitmix64(seed & _M64)


def beta_thresholds(seed: int) -> np.ndarray:
    """166 thresholds in [0, 2^32]: key j set iff u32 < thr[j-1]."""
    p = np.random.Generator(np.random.PCG64(seed)).beta(0.6, 2.0, size=NUM_KEYS)
    p[0] = 0.0
    return np.floor(p * 2.0**32).astype(np.uint64)


def flip_mask(keys) -> np.ndarray:
    """Words with the given 1-based keys set."""
    w = [0, 0, 0]
    for j in keys:
        j = int(j)
        w[(j - 1) // 64] |= 1 << ((j - 1) % 64)
    return np.array(w, dtype=np.uint64)


@dataclass
class Plan:
    name: str
    n: int
    Q: int
    k: int | None
    radius: int | None
    seed: int
    seed_key: int
    thresholds: np.ndarray
    source_idx: np.ndarray                 # (Q,) library entries the queries start from
    query_flips: list                      # per query: array of flipped keys
    planted_idx: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    planted_query: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    planted_flips: list = field(default_factory=list)

    def queries_from_sources(self, source_words: np.ndarray) -> np.ndarray:
        q = np.asarray(source_words, dtype=np.uint64).reshape(self.Q, 3).copy()
        for i, f in enumerate(self.query_flips):
            q[i] ^= flip_mask(f)
        return q

    def planted_words(self, queries: np.ndarray) -> np.ndarray:
        out = np.empty((len(self.planted_idx), 3), dtype=np.uint64)
        for i, (qi, f) in enumerate(zip(self.planted_query, self.planted_flips)):
            out[i] = queries[qi] ^ flip_mask(f)
        return out

    def describe(self) -> dict:
        return {"workload": self.name, "entries": self.n, "queries": self.Q, "k": self.k,
                "radius": self.radius, "seed": self.seed, "planted": int(len(self.planted_idx))}


def _flips(rng: np.random.Generator, lo: int, hi: int) -> np.ndarray:
    f = int(rng.integers(lo, hi + 1))
    return np.sort(rng.choice(NUM_KEYS - 1, size=f, replace=False) + 2)


def _distinct_indices(rng: np.random.Generator, n: int, m: int, exclude: np.ndarray) -> np.ndarray:
    if m + len(exclude) > n:
        raise ValueError(f"cannot place {m} entries in a library of {n}")
    excl = set(int(x) for x in exclude)
    out: list[int] = []
    seen = set(excl)
    while len(out) < m:
        cand = rng.integers(0, n, size=2 * (m - len(out)) + 16)
        for c in cand:
            c = int(c)
            if c not in seen:
                seen.add(c)
                out.append(c)
                if len(out) == m:
                    break
    return np.array(out, dtype=np.int64)


def make_plan(name: str, seed: int = 20240808, n: int | None = None, planted_per_query: int | None = None,
              Q: int | None = None) -> Plan:
    """The workload of config ``name`` (c1..c5); ``n`` / ``Q`` / planted counts
    may be scaled down for parity tests."""
    cfg = CONFIGS[name]
    n = cfg["n"] if n is None else n
    Q = cfg["Q"] if Q is None else Q
    rng = np.random.Generator(np.random.PCG64(seed + 1))
    src = _distinct_indices(rng, n, Q, np.zeros(0, np.int64))
    qflips = [_flips(rng, *cfg["flips"]) for _ in range(Q)]
    plan = Plan(name=name, n=n, Q=Q, k=cfg["k"], radius=cfg["radius"], seed=seed, seed_key=seed_key(seed),
                thresholds=beta_thresholds(seed), source_idx=src, query_flips=qflips)
    if cfg["planted"] is not None:
        per, lo, hi = cfg["planted"]
        if planted_per_query is not None:
            per = planted_per_query
        per = min(per, max(0, (n - Q) // max(Q, 1)))
        idx = _distinct_indices(rng, n, per * Q, src)
        plan.planted_idx = idx
        plan.planted_query = np.repeat(np.arange(Q), per)
        plan.planted_flips = [_flips(rng, lo, hi) for _ in range(per * Q)]
    return plan


def build_library(plan: Plan, device: int | None = None, index_base: int = 0, start: int = 0,
                  count: int | None = None, devices=None):
    """Generate the plan's library on the GPU (this rank's contiguous slice
    [start, start + count)), apply planted entries, and return (library, queries).

    ``devices=[d0, d1, ...]`` generates the slice as a LibraryGroup sharded
    over those GPUs (one process). Queries need the source entries' words;
    they are regenerated on the host from the same counter-based stream
    (cheap: Q entries)."""
    from .library import Library, LibraryGroup

    count = plan.n - start if count is None else count
    if devices is not None and len(devices) > 1:
        lib = LibraryGroup.generate(count, plan.seed_key, plan.thresholds, devices, start=start)
        shards = lib.shards
    else:
        dev = devices[0] if devices else device
        lib = Library.generate(count, plan.seed_key, plan.thresholds, device=dev, start=start,
                               index_base=start if index_base == 0 else index_base)
        shards = [lib]
    src_words = generate_rows(plan.seed_key, plan.thresholds, plan.source_idx)
    queries = plan.queries_from_sources(src_words)
    if len(plan.planted_idx):
        words = plan.planted_words(queries)
        for sh in shards:  # global index of a shard's entry 0 is its index_base (== start for one shard)
            lo = sh.index_base if len(shards) > 1 else start
            mine = (plan.planted_idx >= lo) & (plan.planted_idx < lo + sh.n)
            if np.any(mine):
                sh.write_entries(plan.planted_idx[mine] - lo, words[mine])
    return lib, queries


def generate_rows(seed_key_: int, thresholds: np.ndarray, indices: np.ndarray) -> np.ndarray:
    """Host evaluation of the counter-based generator for a few entries
    (query sources). Same definition as the device gen_kernel."""
    thr = np.asarray(thresholds, dtype=np.uint64)
    out = np.zeros((len(indices), 3), dtype=np.uint64)
    for r, i in enumerate(np.asarray(indices, dtype=np.uint64)):
        w = [0, 0, 0]
        for c in range(83):
            z = (seed_key_ + ((int(i) * 83 + c + 1) * 0x9E3779B97F4A7C15)) & _M64
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
            h = z ^ (z >> 31)
            for half, j in ((h & 0xFFFFFFFF, 2 * c), (h >> 32, 2 * c + 1)):
                if half < int(thr[j]):
                    w[j >> 6] |= 1 << (j & 63)
        out[r] = w
    return out


def planted_after_sources(plan: Plan, words_host: np.ndarray) -> np.ndarray:
    """Apply the plan's planted entries to a host copy of the library (oracle side)."""
    src = words_host[plan.source_idx]
    queries = plan.queries_from_sources(src)
    if len(plan.planted_idx):
        words_host[plan.planted_idx] = plan.planted_words(queries)
    return queries
