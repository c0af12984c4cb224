#!/bin/bash
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$FPS_LAYOUT $*', 'ms/step=%.4f scan_ms=%.4f ach=%.0f frac=%.3f e2e=%.4f'%(d['ms_per_step'], r['scan_kernel_ms'], r['achieved'], r['frac'], d['e2e']['ms_per_step']))"; }
for L in compact full; do for w in c1 c2 c3; do FPS_LAYOUT=$L run --workload $w; done; done
