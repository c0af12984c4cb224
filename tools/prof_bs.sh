#!/bin/bash
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" || exit 1
CMD="python bench.py --workload c4 --steps 2 --warmup 1 --no-cpu-baseline"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"bs_scan_kernel" -s 1 -c 1 -o gpurun_out/prof_bs_c4 $CMD > gpurun_out/ncu_bs_c4.log 2>&1; echo rc=$?
CMD5="python bench.py --workload c5 --steps 2 --warmup 1 --no-cpu-baseline"
$CMD5 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"bs_scan_kernel" -s 1 -c 1 -o gpurun_out/prof_bs_c5 $CMD5 > gpurun_out/ncu_bs_c5.log 2>&1; echo rc=$?
