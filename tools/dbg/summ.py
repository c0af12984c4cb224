"""One-line summary of a bench.py JSON line (stdin)."""
import json
import sys

d = json.loads(sys.stdin.read().strip().splitlines()[-1])
r = d["roofline"]
print("step_ms=%.3f scan_ms=%.3f frac=%.3f %s e2e_ms=%.3f derived_ms=%.0f B/entry=%.1f best=%s mhz=%s" % (
    d["ms_per_step"], r.get("scan_kernel_ms", 0), r.get("frac", 0), r.get("kernel"), d["e2e"]["ms_per_step"],
    d["library"]["derived_build_ms"], d["library"]["hbm_bytes_per_entry"]["total"], d.get("check"),
    d["clocks"]["sm_mhz"]))
