#!/bin/bash
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" || exit 1
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('flags=$FPS_SCAN_FLAGS $*', 'ms/step=%.4f scan_ms=%.4f e2e=%.4f'%(d['ms_per_step'], r['scan_kernel_ms'], d['e2e']['ms_per_step']))"; }
FPS_SCAN_FLAGS=0 run --workload c2
FPS_SCAN_FLAGS=0 run --workload c2 --radius 0
FPS_SCAN_FLAGS=0 run --workload c2 --k 1
FPS_SCAN_FLAGS=3 run --workload c2 --k 1
FPS_SCAN_FLAGS=0 run --workload c3 --radius 0
