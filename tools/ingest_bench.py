"""Library build throughput: native builder vs the reference's build_shards.

Writes a synthetic text library with the reference's own writer
(fpscan.synth.write_text_library, needs /root/reference) and times
    reference: fpscan.libstore.build_shards(open(path), S, out)   (cli.py:69-70)
    native:    paper_1906_06170_b200.libstore.build_shards(open(path), S, out)
and checks the two libraries are byte-identical.
"""
import hashlib, os, sys, tempfile, time
from pathlib import Path
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from fpscan import libstore as R, synth as RS
from paper_1906_06170_b200 import libstore as L

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
S = int(sys.argv[2]) if len(sys.argv) > 2 else 16
with tempfile.TemporaryDirectory(dir="/dev/shm") as td:
    td = Path(td)
    txt = td / "lib.txt"
    RS.write_text_library(txt, n, seed=5)
    mb = txt.stat().st_size / 1e6
    t0 = time.perf_counter()
    with open(txt, encoding="utf-8") as f:
        L.build_shards(f, S, td / "native")
    tn = time.perf_counter() - t0
    t0 = time.perf_counter()
    with open(txt, encoding="utf-8") as f:
        R.build_shards(f, S, td / "ref")
    tr = time.perf_counter() - t0
    same = all(hashlib.sha256((td / "native" / p.name).read_bytes()).digest() == hashlib.sha256(p.read_bytes()).digest()
               for p in (td / "ref").glob("*.fps")) and (td / "native" / "manifest.json").read_text() == (td / "ref" / "manifest.json").read_text()
    print(f"{n} lines ({mb:.0f} MB text), {S} shards: reference {tr:.2f} s ({n / tr / 1e6:.2f} M lines/s), "
          f"native {tn:.3f} s ({n / tn / 1e6:.1f} M lines/s, {os.cpu_count()} threads) -> {tr / tn:.0f}x; identical={same}")
