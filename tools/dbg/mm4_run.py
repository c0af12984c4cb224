"""One C4-shaped batch (1,024 queries) on a 20 M-entry library: the fp4 tensor-core scan (ncu target)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from paper_1906_06170_b200 import synth  # noqa: E402

plan = synth.make_plan("c4", n=int(os.environ.get("N", 20_000_000)))
lib, q = synth.build_library(plan)
for _ in range(2):
    res = lib.search_batch(q, 10)
print("kernel", lib.last_kernel, res.hits(0)[:2])
