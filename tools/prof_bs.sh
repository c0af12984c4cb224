#!/bin/bash
# ncu --set full of the bit-sliced kernel for C4 and C5 (one launch each)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for w in c4 c5; do
  CMD="python bench.py --workload $w --steps 2 --warmup 1 --no-cpu-baseline"
  $CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"bs_scan_kernel" -s 1 -c 1 -o gpurun_out/prof_bs2_$w $CMD > gpurun_out/ncu_bs2_$w.log 2>&1; echo "ncu $w rc=$?"
done
