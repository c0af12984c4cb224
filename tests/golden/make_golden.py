"""Generate tests/golden/ fixtures by running the REAL reference fpscan.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``fpscan`` from /root/reference/pkg/src, builds FPS1 libraries
with the reference's own writer (``libstore.build_shards`` /
``libstore.write_shard_file`` + ``save_manifest``) and records what the
reference's ``scan.search`` / ``batch_search`` / ``merge_topk`` /
``distance_packed`` / ``manhattan_reference`` return. The GPU box never reads
/root/reference; tests only read the committed JSON / npy outputs.
"""

from __future__ import annotations

import hashlib
import itertools
import json
import random
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT))

from fpscan import libstore, scan  # noqa: E402  (the reference)
from fpscan.fingerprint import NUM_KEYS, Fingerprint, distance_packed, manhattan_reference  # noqa: E402

import fps_oracle as orc  # noqa: E402
from paper_1906_06170_b200 import synth  # noqa: E402


def words_sha(words: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(words, dtype="<u8").tobytes()).hexdigest()


def ref_manifest(tmp: Path, words: np.ndarray, shard_count: int, cids=None):
    """Write the library with the reference's own FPS1 writer."""
    tmp.mkdir(parents=True, exist_ok=True)
    n = len(words)
    cids = np.arange(1, n + 1) if cids is None else cids
    payload = b"".join(
        libstore.pack_record(libstore.LibraryRecord(cid=int(c), fp=Fingerprint(tuple(int(x) for x in w))))
        for c, w in zip(cids, words)
    )
    shards = []
    off = 0
    for i, size in enumerate(libstore.split_sizes(n, shard_count)):
        path = tmp / f"shard-{i:03d}.fps"
        region = payload[off * 32:(off + size) * 32]
        checksum = libstore.write_shard_file(path, region, size)
        shards.append(libstore.Shard(path=path, record_count=size, dataset_label=libstore.shard_label(i),
                                     checksum=checksum))
        off += size
    manifest = libstore.ShardManifest(shards=tuple(shards), total_records=n)
    libstore.save_manifest(manifest, tmp)
    return manifest


def hits(top) -> list[list[int]]:
    return [[h.cid, h.distance] for h in top.hits]


def kat_pairs():
    single = [Fingerprint.from_keys({j}) for j in range(1, NUM_KEYS + 1)]
    boundary = [
        Fingerprint.zero(),
        Fingerprint.from_keys(range(1, NUM_KEYS + 1)),
        Fingerprint.from_keys({1}),
        Fingerprint.from_keys({166}),
        Fingerprint.from_keys({1, 166}),
        Fingerprint.from_keys({64, 65, 128, 129}),
        Fingerprint.from_keys({1, 2, 3}),
        Fingerprint.from_keys({2, 3, 4}),
    ]
    rng = random.Random(20240808)
    rand = [Fingerprint((rng.getrandbits(64), rng.getrandbits(64), rng.getrandbits(38))) for _ in range(64)]
    out = []
    for a, b in itertools.product(single[::11] + boundary + rand[:16], boundary + rand[16:32]):
        d = distance_packed(a, b)
        assert d == manhattan_reference(a, b)
        out.append([list(a.words), list(b.words), d])
    return out


def main() -> None:
    golden: dict = {"generator": [], "search": [], "batch_min": [], "per_query": [], "range": [], "merge": [],
                    "kat": kat_pairs(), "split_sizes": [], "fps1": []}

    for total, count in [(10, 3), (0, 2), (7, 7), (100, 8), (95_417_114, 8), (95_417_114, 3)]:
        golden["split_sizes"].append([total, count, libstore.split_sizes(total, count)])

    with tempfile.TemporaryDirectory() as td:
        td = Path(td)
        # --- generator pin + FPS1 writer identity ------------------------------
        for seed, n in [(7, 1000), (20240808, 5000)]:
            thr = synth.beta_thresholds(seed)
            w = orc.generate_words(synth.seed_key(seed), thr, 0, n)
            golden["generator"].append({"seed": seed, "n": n, "sha256": words_sha(w),
                                        "first": [[int(x) for x in r] for r in w[:4]]})
            m = ref_manifest(td / f"gen{seed}", w, 3)
            shas = [hashlib.sha256(Path(s.path).read_bytes()).hexdigest() for s in m.shards]
            golden["fps1"].append({"seed": seed, "n": n, "shards": 3, "sha256": shas,
                                   "checksums": [f"{s.checksum:016x}" for s in m.shards]})

        # --- search (configs 1-3 shapes, scaled down) ---------------------------
        cases = [
            ("c1", 20240808, 20_000, 1, [10, 1, 30]),
            ("c2", 20240809, 50_000, 1, [100, 7]),
            ("c3", 20240810, 40_000, 3, [10]),
        ]
        for name, seed, n, shards, ks in cases:
            plan = synth.make_plan(name, seed=seed, n=n, planted_per_query=200 if name == "c2" else None)
            w = orc.generate_words(plan.seed_key, plan.thresholds, 0, n)
            sha_plain = words_sha(w)
            q = synth.planted_after_sources(plan, w)
            m = ref_manifest(td / f"{name}_{seed}", w, shards)
            for k in ks:
                for par in (1, shards):
                    top = scan.search(m, Fingerprint(tuple(int(x) for x in q[0])), scan.SearchParams(n=k,
                                                                                                   parallelism=par))
                    golden["search"].append({"case": name, "seed": seed, "n": n, "shards": shards, "k": k,
                                             "parallelism": par, "sha256_unplanted": sha_plain,
                                             "sha256": words_sha(w), "query": [int(x) for x in q[0]],
                                             "hits": hits(top)})

        # --- per-query batch top-k (config 4 semantics = one search per query) --
        plan = synth.make_plan("c4", seed=20240811, n=30_000, Q=12)
        w = orc.generate_words(plan.seed_key, plan.thresholds, 0, plan.n)
        q = synth.planted_after_sources(plan, w)
        m = ref_manifest(td / "c4", w, 2)
        golden["per_query"].append({
            "case": "c4", "seed": 20240811, "n": plan.n, "Q": plan.Q, "k": 10, "sha256": words_sha(w),
            "queries": [[int(x) for x in r] for r in q],
            "hits": [hits(scan.search(m, Fingerprint(tuple(int(x) for x in r)), scan.SearchParams(n=10)))
                     for r in q],
        })

        # --- reference batch_search (min over queries) --------------------------
        bq = q[:5]
        top = scan.batch_search(m, [Fingerprint(tuple(int(x) for x in r)) for r in bq], scan.SearchParams(n=30))
        golden["batch_min"].append({"case": "c4", "seed": 20240811, "n": plan.n, "k": 30,
                                    "queries": [[int(x) for x in r] for r in bq], "hits": hits(top)})

        # --- range (config 5 semantics) via the reference distance kernel --------
        plan = synth.make_plan("c5", seed=20240812, n=30_000, Q=4, planted_per_query=50)
        w = orc.generate_words(plan.seed_key, plan.thresholds, 0, plan.n)
        q = synth.planted_after_sources(plan, w)
        rows = []
        for qi, qq in enumerate(q):
            d = scan._distances_packed(w, np.asarray([qq], dtype=np.uint64))
            hit = np.flatnonzero(d <= 6)
            for i in sorted(hit, key=lambda i: (int(d[i]), int(i))):
                rows.append([qi, int(i), int(d[i])])
        golden["range"].append({"case": "c5", "seed": 20240812, "n": plan.n, "Q": plan.Q, "radius": 6,
                                "sha256": words_sha(w), "queries": [[int(x) for x in r] for r in q],
                                "rows": rows})

        # --- tensor-core shapes: >= 192 queries (the default kernel for large
        #     batches, tcgen05 int8 GEMM) -- per-query top-k and range --------
        plan = synth.make_plan("c4", seed=20240813, n=40_000, Q=256)
        w = orc.generate_words(plan.seed_key, plan.thresholds, 0, plan.n)
        q = synth.planted_after_sources(plan, w)
        m = ref_manifest(td / "c4tc", w, 2)
        golden["per_query_tc"] = {
            "case": "c4", "seed": 20240813, "n": plan.n, "Q": plan.Q, "k": 10, "sha256": words_sha(w),
            "queries": [[int(x) for x in r] for r in q],
            "hits": [hits(scan.search(m, Fingerprint(tuple(int(x) for x in r)), scan.SearchParams(n=10)))
                     for r in q],
        }
        # reference batch_search for n > 1024 (any n >= 1 is valid: scan.py:82-84)
        golden["batch_min_large"] = []
        for k in (1025, 4000):
            bq = q[:3]
            top = scan.batch_search(m, [Fingerprint(tuple(int(x) for x in r)) for r in bq], scan.SearchParams(n=k))
            golden["batch_min_large"].append({"seed": 20240813, "n": plan.n, "k": k,
                                              "queries": [[int(x) for x in r] for r in bq], "hits": hits(top)})
        plan = synth.make_plan("c5", seed=20240814, n=40_000, Q=200, planted_per_query=10)
        w = orc.generate_words(plan.seed_key, plan.thresholds, 0, plan.n)
        q = synth.planted_after_sources(plan, w)
        rows = []
        for qi, qq in enumerate(q):
            d = scan._distances_packed(w, np.asarray([qq], dtype=np.uint64))
            hit = np.flatnonzero(d <= 5)
            for i in sorted(hit, key=lambda i: (int(d[i]), int(i))):
                rows.append([qi, int(i), int(d[i])])
        golden["range_tc"] = {"case": "c5", "seed": 20240814, "n": plan.n, "Q": plan.Q, "radius": 5,
                              "planted_per_query": 10, "sha256": words_sha(w),
                              "queries": [[int(x) for x in r] for r in q], "rows": rows}

        # --- random-CID library with distance ties (test_scan.py:28-40 pattern) ---
        rng = random.Random(9)
        cids = rng.sample(range(1, 2**40), 3000)
        pool = []
        recs = []
        for c in cids:
            if pool and rng.random() < 0.2:
                fp = rng.choice(pool)
            else:
                fp = Fingerprint.from_keys(rng.sample(range(1, NUM_KEYS + 1), rng.randint(0, 80)))
                pool.append(fp)
            recs.append((c, fp))
        rec_arr = np.array([[c, *fp.words] for c, fp in recs], dtype=np.uint64)
        np.save(HERE / "cid_library.npy", rec_arr)
        m = ref_manifest(td / "cids", rec_arr[:, 1:], 3, cids=rec_arr[:, 0])
        qs = [pool[3].words, Fingerprint.from_keys(rng.sample(range(1, NUM_KEYS + 1), 40)).words]
        golden["cid_search"] = [
            {"query": list(qq), "k": k, "hits": hits(scan.search(m, Fingerprint(tuple(qq)), scan.SearchParams(n=k)))}
            for qq in qs for k in (1, 5, 30, 100)
        ]
        golden["cid_batch_min"] = {
            "queries": [list(qq) for qq in qs], "k": 30,
            "hits": hits(scan.batch_search(m, [Fingerprint(tuple(qq)) for qq in qs], scan.SearchParams(n=30))),
        }

    # --- merge_topk --------------------------------------------------------------
    rng = random.Random(6)
    ids = iter(rng.sample(range(1, 10**6), 600))
    parts = []
    for _ in range(6):
        pairs = sorted(((rng.randint(0, 166), next(ids)) for _ in range(50)))
        parts.append(scan.TopK(capacity=50, hits=tuple(scan.SearchHit(cid=c, distance=d) for d, c in pairs)))
    for n in (1, 25, 100, 400):
        golden["merge"].append({"parts": [hits(p) for p in parts], "n": n, "hits": hits(scan.merge_topk(parts, n))})

    (HERE / "golden.json").write_text(json.dumps(golden, separators=(",", ":")) + "\n")
    print("wrote", HERE / "golden.json", (HERE / "golden.json").stat().st_size, "bytes")


if __name__ == "__main__":
    main()
