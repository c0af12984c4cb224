import os, sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1906_06170_b200.library import Library
w = np.tile(np.array([[0x1234, 0x5678, 0x9]], dtype=np.uint64), (300_000, 1))
q = np.tile(np.array([[0x1234, 0x5678, 0x8]], dtype=np.uint64), (300, 1))
for seq in sys.argv[1:]:
    lib = Library.from_words(w)
    out = []
    for mode in seq.split(","):
        env, val = mode.split("=")
        os.environ[env] = val
        res = lib.search_batch(q, 10)
        bad = [i for i in range(300) if res.hits(i) != [(j, 1) for j in range(10)]]
        out.append(f"{mode}:{lib.last_kernel}:bad={len(bad)} first={bad[:3]} {res.hits(bad[0])[:3] if bad else ''}")
    print(seq, "|", " ; ".join(out), flush=True)
    for mode in seq.split(","):
        os.environ.pop(mode.split("=")[0], None)
