"""Generate tests/golden/ingest*.{json,txt} by running the REAL reference
library builder (fpscan.libstore) in the build container:

    python tests/golden/make_ingest_golden.py

Records, for a text corpus with the edge cases the reference handles (blank
and whitespace-only lines, 167-character bitstrings, CRLF / lone-CR line ends,
leading-zero and maximal CIDs), what ``libstore.build_shards`` writes (shard
bytes as sha256, manifest document) for several shard counts, both from a
list of lines and from a text file opened like the reference CLI does
(cli.py:69-70); the exception class and message for malformed inputs; FNV-1a
vectors; and ``validate_manifest`` violations for damaged libraries. The GPU
box never reads /root/reference; tests only read the committed outputs.
"""

from __future__ import annotations

import hashlib
import json
import random
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from fpscan import libstore  # noqa: E402  (the reference)

NUM_KEYS = 166


def bits(rng: random.Random, n: int = NUM_KEYS) -> str:
    return "".join("1" if rng.random() < 0.25 else "0" for _ in range(n))


def corpus() -> str:
    """Text library with every line shape build_shards accepts."""
    rng = random.Random(1906)
    out = []
    for i in range(1, 301):
        kind = i % 11
        if kind == 3:
            out.append(f"{i}\t{bits(rng, NUM_KEYS + 1)}\n")  # 167-char form
        elif kind == 5:
            out.append(f"{i}\t{bits(rng)}\r\n")  # CRLF
        elif kind == 7:
            out.append("\n")  # blank
            out.append(f"{i}\t{bits(rng)}\n")
        elif kind == 8:
            out.append(" \t \n")  # whitespace only
            out.append(f"{i:08d}\t{bits(rng)}\n")  # leading zeros
        elif kind == 9:
            out.append("\u00a0\u2003\n")  # unicode whitespace only
            out.append(f"{i}\t{bits(rng)}\r")  # lone CR ends the line in text mode
        else:
            out.append(f"{i}\t{bits(rng)}\n")
    out.append(f"{(1 << 64) - 1}\t{'1' * NUM_KEYS}\n")
    out.append(f"1\t{'0' * NUM_KEYS}")  # no final newline
    return "".join(out)


def shard_shas(manifest) -> list[str]:
    return [hashlib.sha256(Path(s.path).read_bytes()).hexdigest() for s in manifest.shards]


def manifest_doc(d: Path) -> dict:
    return json.loads((d / "manifest.json").read_text())


def err(fn):
    try:
        fn()
    except Exception as exc:  # noqa: BLE001 - recorded as data
        return [type(exc).__name__, str(exc)]
    return None


def main() -> None:
    text = corpus()
    (HERE / "ingest_lines.txt").write_bytes(text.encode("utf-8"))
    good = {"list": {}, "file": {}}
    with tempfile.TemporaryDirectory() as td:
        td = Path(td)
        # list-of-lines input: the items are exactly what text-mode iteration yields
        with open(HERE / "ingest_lines.txt", encoding="utf-8") as f:
            lines = list(f)
        for sc in (1, 3, 7, 400):
            d = td / f"list{sc}"
            m = libstore.build_shards(lines, sc, d)
            good["list"][str(sc)] = {"shas": shard_shas(m), "manifest": manifest_doc(d)}
        # items carrying their own "\r\n" / "\r" ends (rstrip("\r\n") per item)
        rng = random.Random(11)
        raw = [f"{i}\t{bits(rng)}" + ("\r\n", "\r", "\n", "", "\r\r\n")[i % 5] for i in range(1, 41)]
        d = td / "raw"
        m = libstore.build_shards(raw, 3, d)
        good["raw"] = {"lines": raw, "shas": shard_shas(m), "manifest": manifest_doc(d)}
        for sc in (1, 4):
            d = td / f"file{sc}"
            with open(HERE / "ingest_lines.txt", encoding="utf-8") as f:
                m = libstore.build_shards(f, sc, d)
            good["file"][str(sc)] = {"shas": shard_shas(m), "manifest": manifest_doc(d)}

        ok = "1\t" + "0" * NUM_KEYS
        cases = {
            "missing_tab": [ok, "2 " + "0" * NUM_KEYS],
            "bad_cid_alpha": ["x1\t" + "0" * NUM_KEYS],
            "bad_cid_zero": ["", "0\t" + "0" * NUM_KEYS],
            "bad_cid_empty": ["\t" + "0" * NUM_KEYS],
            "bad_cid_overflow": [f"{1 << 64}\t" + "0" * NUM_KEYS],
            "bad_cid_unicode_digit": ["١\t" + "0" * NUM_KEYS],
            "wrong_length": [ok, ok, "3\t" + "0" * 165],
            "wrong_length_trailing_space": ["3\t" + "0" * NUM_KEYS + " "],
            "invalid_char": ["4\t" + "0" * 100 + "2" + "0" * 65],
            "invalid_char_167": ["4\t" + "x" + "0" * NUM_KEYS],
            "second_tab": ["5\t" + "0" * 80 + "\t" + "0" * 85],
            "error_after_blanks": ["\n", "  \n", ok + "\n", "7\tzz\n"],
            "first_of_two_errors": ["9\t01\n", "abc\n"],
            "unicode_in_bits": ["6\t" + "0" * 165 + "é"],
        }
        errors = {}
        for name, ls in cases.items():
            errors[name] = {"lines": ls, "error": err(lambda: libstore.build_shards(ls, 2, td / ("e_" + name)))}
            # the reference parses everything before writing: no directory on error
            errors[name]["wrote"] = (td / ("e_" + name)).exists()

        fnv = []
        rng = random.Random(7)
        for n in (0, 1, 2, 31, 32, 1000):
            data = bytes(rng.randrange(256) for _ in range(n))
            fnv.append([data.hex(), libstore.fnv1a_64(data)])
        data = bytes(range(256)) * 3
        fnv.append(["resume", libstore.fnv1a_64(data[300:], libstore.fnv1a_64(data[:300])), data.hex()])

        # validate_manifest on damaged copies of a 3-shard library
        base = td / "val"
        with open(HERE / "ingest_lines.txt", encoding="utf-8") as f:
            m = libstore.build_shards(f, 3, base)
        viol = {}

        def run(name, mutate):
            d = td / ("v_" + name)
            d.mkdir()
            for s in m.shards:
                (d / Path(s.path).name).write_bytes(Path(s.path).read_bytes())
            (d / "manifest.json").write_text((base / "manifest.json").read_text())
            mutate(d)
            mm = libstore.load_manifest(d)
            viol[name] = [[v.kind, Path(v.path).name if v.path != "manifest" else "manifest",
                           v.message.replace(str(d) + "/", "")] for v in libstore.validate_manifest(mm)]

        def flip_byte(d):
            p = d / "shard-001.fps"
            b = bytearray(p.read_bytes())
            b[100] ^= 1
            p.write_bytes(bytes(b))

        def truncate(d):
            p = d / "shard-002.fps"
            p.write_bytes(p.read_bytes()[:-32])

        def bad_magic(d):
            p = d / "shard-000.fps"
            b = bytearray(p.read_bytes())
            b[0:4] = b"NOPE"
            p.write_bytes(bytes(b))

        def missing(d):
            (d / "shard-001.fps").unlink()

        def count(d):
            doc = json.loads((d / "manifest.json").read_text())
            doc["shards"][0]["record_count"] += 1
            doc["total_records"] += 1
            (d / "manifest.json").write_text(json.dumps(doc))

        run("clean", lambda d: None)
        run("flip_byte", flip_byte)
        run("truncate", truncate)
        run("bad_magic", bad_magic)
        run("missing", missing)
        run("count", count)

    out = {"good": good, "errors": errors, "fnv": fnv, "validate": viol}
    (HERE / "ingest.json").write_text(json.dumps(out, indent=1) + "\n")
    print("wrote", HERE / "ingest.json")


if __name__ == "__main__":
    main()
