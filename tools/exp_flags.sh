#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/exp.txt
python -c "import __graft_entry__ as g; g.build()"
for f in 0 1 3; do for w in c1 c2 c3; do
  FPS_SCAN_FLAGS=$f timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/exp_${w}_$f.json 2>gpurun_out/exp_${w}_$f.err
  python -c "
import json; d=json.loads(open('gpurun_out/exp_${w}_$f.json').read().strip().splitlines()[-1]); r=d['roofline']
print('flags=$f $w ms/step=%.4f scan_ms=%.4f frac=%.3f e2e_ms=%.4f best=%s'%(d['ms_per_step'], r['scan_kernel_ms'], r['frac'], d['e2e']['ms_per_step'], d.get('check')))" >> gpurun_out/exp.txt 2>&1
done; done
cat gpurun_out/exp.txt
python bench.py --workload c2 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 3 -c 1 -o gpurun_out/prof_c2 python bench.py --workload c2 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_c2.log 2>&1
echo ncu rc=$?
