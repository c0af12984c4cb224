#!/bin/bash
# usage: WL=c3 TAG=pq1 tools/prof_pq.sh -> gpurun_out/prof_${TAG}_${WL}.ncu-rep (plane scan, one launch)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
WL=${WL:-c3}; TAG=${TAG:-pq1}
CMD="python bench.py --workload $WL --steps 3 --warmup 2 --no-cpu-baseline"
$CMD > gpurun_out/plain_$WL.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pq_scan_kernel" -s 3 -c 1 -o gpurun_out/prof_${TAG}_$WL $CMD > gpurun_out/ncu_full_${TAG}_$WL.log 2>&1
echo "prof rc=$?"
