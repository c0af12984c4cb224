#!/bin/bash
# A/B of scan flags on the batched configs: CFGS="0;1024" tools/ab_bs.sh
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
IFS=";" read -ra CL <<< "${CFGS:-0;1024}"
for rep in 1 2; do
for f in "${CL[@]}"; do
  for w in ${WLS:-c4 c5}; do
    FPS_SCAN_FLAGS=$f timeout 600 python bench.py --workload $w --steps ${STEPS:-3} --warmup 1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('rep=$rep flags=$f $w ms/step=%.3f scan_ms=%.3f e2e=%.3f'%(d['ms_per_step'], r['scan_kernel_ms'], d['e2e']['ms_per_step']))"
  done
done
done
