#!/bin/bash
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" || exit 1
FPS_DEBUG=1 FPS_SCAN_FLAGS=4 python bench.py --workload c2 --steps 3 --warmup 1 --no-cpu-baseline 2>&1 | grep "\[fps\]" | sort | uniq -c | head
FPS_DEBUG=1 FPS_SCAN_FLAGS=4 python bench.py --workload c1 --steps 3 --warmup 1 --no-cpu-baseline 2>&1 | grep "\[fps\]" | sort | uniq -c | head
FPS_DEBUG=1 FPS_SCAN_FLAGS=4 python bench.py --workload c3 --steps 3 --warmup 1 --no-cpu-baseline 2>&1 | grep "\[fps\]" | sort | uniq -c | head
CMD="python bench.py --workload c2 --steps 3 --warmup 2 --no-cpu-baseline"
FPS_SCAN_FLAGS=4 $CMD > /dev/null 2>&1 && FPS_SCAN_FLAGS=4 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2b.csv $CMD > /dev/null 2>&1
grep -E "scan_kernel|select_kernel" gpurun_out/launches_c2b.csv | awk -F'","' '{print $5, $NF}' | sort | uniq -c | head -20
