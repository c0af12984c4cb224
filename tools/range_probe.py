"""Where the C5 end-to-end range call spends its time (host side)."""
import sys, time, ctypes as C
sys.path.insert(0, ".")
import numpy as np
from paper_1906_06170_b200 import synth, _native as N
from paper_1906_06170_b200.library import RangeResult
plan = synth.make_plan("c5")
lib, q = synth.build_library(plan)
L = N.load()
rad = np.full(len(q), plan.radius, np.uint8)
qa = np.ascontiguousarray(q)
for _ in range(3):
    r = lib.range_search(qa, plan.radius)
def t(f, n=10):
    t0 = time.perf_counter()
    for _ in range(n): f()
    return (time.perf_counter() - t0) / n * 1e3
out = C.c_void_p(); n_out = C.c_uint64()
def raw():
    L.fps_range(lib._h, qa.ctypes.data, len(qa), rad.ctypes.data, C.byref(out), C.byref(n_out))
    L.fps_free(out)
print("hits", len(r))
print("range_search ms", t(lambda: lib.range_search(qa, plan.radius)))
print("raw fps_range+free ms", t(raw))
L.fps_range(lib._h, qa.ctypes.data, len(qa), rad.ctypes.data, C.byref(out), C.byref(n_out))
m = n_out.value
print("as_array.copy ms", t(lambda: np.ctypeslib.as_array(C.cast(out, C.POINTER(C.c_uint64)), shape=(m,)).copy()))
keys = np.ctypeslib.as_array(C.cast(out, C.POINTER(C.c_uint64)), shape=(m,)).copy()
print("from_keys ms", t(lambda: RangeResult.from_keys(keys)))
