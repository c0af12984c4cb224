"""Print select_kernel phase timestamps (FPS_DEBUG=1) for each config's shape."""
import os, sys
os.environ["FPS_DEBUG"] = "1"
sys.path.insert(0, ".")
import numpy as np
from paper_1906_06170_b200 import synth
for wl in sys.argv[1:] or ["c2"]:
    plan = synth.make_plan(wl)
    lib, q = synth.build_library(plan)
    for _ in range(3):
        lib.search_batch(np.ascontiguousarray(q[:1]), plan.k)
    print(wl, "done", flush=True)
    lib.close()
