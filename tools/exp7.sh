#!/bin/bash
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" || exit 1
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$FPS_SCAN_FLAGS $*', 'ms/step=%.4f scan_ms=%.4f frac=%.3f e2e=%.4f'%(d['ms_per_step'], r['scan_kernel_ms'], r['frac'], d['e2e']['ms_per_step']))"; }
for w in c1 c2; do FPS_SCAN_FLAGS=0 run --workload $w; FPS_SCAN_FLAGS=32 run --workload $w; done
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
