#!/bin/bash
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" || exit 1
WL=c2 ./tools/launches.sh
CMD="python bench.py --workload c2 --steps 3 --warmup 2 --no-cpu-baseline"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:select_kernel -s 2 -c 1 -o gpurun_out/prof_sel $CMD > /dev/null 2>&1; echo rc=$?
