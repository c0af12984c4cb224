import sys
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import numpy as np
import fps_oracle as orc
from paper_1906_06170_b200.library import Library
w = orc.generate_words(777, np.full(166, 2**31, np.uint64), 0, 150_000)
lib = Library.from_words(w)
res = lib.search_batch(w[:3].copy(), int(sys.argv[1]) if len(sys.argv) > 1 else 1025)
print(res.hits(0)[:5])
