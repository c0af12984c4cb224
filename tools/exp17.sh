#!/bin/bash
# bulk-copy scan: full (24 B) vs compact (21 B) tiles
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for lay in full compact; do
  for w in c2 c3 c1; do
    FPS_LAYOUT=$lay timeout 300 python bench.py --workload $w --steps 30 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$lay $w ms/step=%.4f scan_ms=%.4f e2e=%.4f %s frac=%.3f check=%s'%(d['ms_per_step'], r['scan_kernel_ms'], d['e2e']['ms_per_step'], r['bound'], r['frac'], d.get('check')))"
  done
done
FPS_LAYOUT=compact timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "single_query or schedules" 2>&1 | tail -2
