#!/bin/bash
# usage: WL=c2 TAG=r01 tools/prof.sh  -> gpurun_out/prof_${TAG}_${WL}.ncu-rep + launches csv
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
WL=${WL:-c2}; TAG=${TAG:-r01}
CMD="python bench.py --workload $WL --steps 3 --warmup 2 --no-cpu-baseline"
$CMD > gpurun_out/plain_$WL.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_$WL.csv $CMD > gpurun_out/ncu_launch_$WL.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"scan_kernel|select_kernel" -s 6 -c 2 -o gpurun_out/prof_${TAG}_$WL $CMD > gpurun_out/ncu_full_$WL.log 2>&1
echo "prof rc=$?"
