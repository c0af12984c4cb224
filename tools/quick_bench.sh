#!/bin/bash
# quick: build + benches (no tests), summary lines
mkdir -p gpurun_out; rm -f gpurun_out/quick.txt
python -c "import __graft_entry__ as g; g.build()" || exit 1
for w in ${WORKLOADS:-c1 c2 c3}; do
  FPS_SCAN_FLAGS=${FLAGS:-0} timeout 300 python bench.py --workload $w --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline > gpurun_out/q_$w.json 2>gpurun_out/q_$w.err
  python -c "
import json; d=json.loads(open('gpurun_out/q_$w.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$w value=%.3e ms/step=%.4f scan_ms=%.4f %s frac=%.3f e2e_ms=%.4f launches=%d best=%s clk=%s'%(d['value'], d['ms_per_step'], r['scan_kernel_ms'], r['bound'], r['frac'], d['e2e']['ms_per_step'], d['gpu_launches'], d.get('check'), d['clocks']['sm_mhz']))" >> gpurun_out/quick.txt 2>&1 || tail -3 gpurun_out/q_$w.err >> gpurun_out/quick.txt
done
cat gpurun_out/quick.txt
