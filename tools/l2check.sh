#!/bin/bash
# DRAM bytes per scan launch when steps run back to back (no ncu cache flush):
# checks that the evict-first streaming leaves no reuse across steps.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
W=${WL:-c2}
FPS_SCAN_FLAGS=${FLAGS:-0} ncu --cache-control none --clock-control none -k regex:scan_kernel -s 6 -c 3 --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --csv \
  python bench.py --workload $W --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/l2check_$W.csv 2>gpurun_out/l2check_$W.err
grep -E "dram__bytes_read|hit_rate|duration" gpurun_out/l2check_$W.csv | cut -d, -f12- | head -12
