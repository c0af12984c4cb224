#!/bin/bash
# A/B of scan flags: CFGS="0;128" WLS="c2 c3" tools/ab.sh
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
IFS=";" read -ra CL <<< "${CFGS:-0;128}"
for rep in 1 2; do
for f in "${CL[@]}"; do
  for w in ${WLS:-c2 c3}; do
    FPS_SCAN_FLAGS=$f timeout 300 python bench.py --workload $w --steps ${STEPS:-30} --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('rep=$rep flags=$f $w ms/step=%.4f scan_ms=%.4f e2e=%.4f'%(d['ms_per_step'], r['scan_kernel_ms'], d['e2e']['ms_per_step']))"
  done
done
done
