#!/bin/bash
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" || exit 1
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$*', 'ms/step=%.4f scan_ms=%.4f frac=%.3f'%(d['ms_per_step'], r['scan_kernel_ms'], r['frac']))"; }
for w in c2 c3; do
echo "static"; FPS_SCAN_FLAGS=4 run --workload $w
for c in 4 8 32 128; do echo "chunk $c"; FPS_CHUNK=$c run --workload $w; done
done
