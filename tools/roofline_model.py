"""Derive the bit-sliced kernel's ALU instructions per comparison from ncu
captures (gpurun_out/prof_bs_<wl>.ncu-rep) -> profiles/roofline_model.json.

ALU warp-instructions = pipe-ALU busy fraction x 2 warp-instructions/clk x
active SM cycles (summed over SMs)."""
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CMP = {"c4": 1024 * 95_417_114, "c5": 64 * 95_417_114}
out = {}
for wl, ncmp in CMP.items():
    rep = ROOT / "gpurun_out" / f"prof_bs_{wl}.ncu-rep"
    if not rep.exists():
        continue
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    v = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    util = float(v["sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"]) / 100.0
    cyc = float(v["sm__cycles_active.sum"])
    alu = util * 2.0 * cyc
    out[wl] = {"alu_warp_instr_per_cmp": alu / ncmp, "alu_pipe_util": util,
               "ncu_duration": f'{v["gpu__time_duration.sum"]} {u["gpu__time_duration.sum"]}',
               "source": f"ncu --set full, {rep.name}"}
p = ROOT / "profiles" / "roofline_model.json"
doc = json.loads(p.read_text()) if p.exists() else {}
doc.update(out)
doc["_doc"] = ("bit-sliced multi-query kernel: ALU warp-instructions per comparison (ncu: pipe-ALU busy x 2 x "
               "active SM cycles / comparisons); bench.py's ALU roofline divides by it")
p.write_text(json.dumps(doc, indent=2) + "\n")
print(json.dumps(out, indent=2))
