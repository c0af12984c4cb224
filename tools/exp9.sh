#!/bin/bash
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" || exit 1
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('flags=$FPS_SCAN_FLAGS chunk=$FPS_CHUNK $*', 'ms/step=%.4f scan_ms=%.4f frac=%.3f e2e=%.4f best=%s'%(d['ms_per_step'], r['scan_kernel_ms'], r['frac'], d['e2e']['ms_per_step'], d.get('check')))"; }
for w in c2 c3; do
 FPS_SCAN_FLAGS=0 run --workload $w
 for c in 2 4 8 16; do FPS_CHUNK=$c FPS_SCAN_FLAGS=68 run --workload $w; done
done
